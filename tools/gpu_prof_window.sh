#!/bin/bash
# ncu --set full (with source) of one config-2 window-kernel launch at HEAD, summarised on the
# box (raw metrics, the hottest SASS lines with stall reasons), after a plain run of the command.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-profw}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
CMD="python bench.py --config 2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 900 $CMD > $O/plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:'window_kernel' -s 40 -c 1 -o $O/w $CMD > $O/ncu_w.log 2>&1; echo "ncu w rc=$?"
ncu -i $O/w.ncu-rep --page raw --csv > $O/w_raw.csv 2>&1
ncu -i $O/w.ncu-rep --page source --csv --print-source sass > $O/w_source_sass.csv 2>&1
python tools/ncu_summary.py $O/w.ncu-rep > $O/w_summary.txt 2>&1
python tools/ncu_hot_sass.py $O/w_source_sass.csv 30 > $O/w_hot_sass.txt 2>&1
rm -f $O/w.ncu-rep $O/w_source_sass.csv
ls -la $O
cat $O/w_summary.txt | head -60
