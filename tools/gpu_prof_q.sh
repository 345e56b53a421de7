#!/bin/bash
# ncu --set full (with source) of one config-3 Q-update launch and one window-kernel launch,
# summarised on the box (raw metrics + the hottest source lines), after a plain run.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-profq}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
CMD="python bench.py --config 3 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 $CMD > $O/plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:'panel_tma_kernel<.int.256, .int.2' -s 300 -c 1 -o $O/q $CMD > $O/ncu_q.log 2>&1; echo "ncu q rc=$?"
ncu -i $O/q.ncu-rep --page raw --csv > $O/q_raw.csv 2>&1
ncu -i $O/q.ncu-rep --page source --csv --print-source sass > $O/q_source_sass.csv 2>&1
python tools/ncu_summary.py $O/q.ncu-rep > $O/q_summary.txt 2>&1
rm -f $O/q.ncu-rep
ls -la $O
