#!/bin/bash
# ncu --set full of one config-3 Q-update launch (the bench's dominant kernel), after a plain
# run of the same command: DRAM traffic per launch for bench.py's roofline.traffic.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-traffic}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 1500 ncu --set full --clock-control none --kernel-name-base demangled \
  -k regex:"panel_tma_kernel<.int.256, .int.2" -s 300 -c 1 -o $O/prof_q3 $CMD > $O/ncu_q3.log 2>&1
echo "rc=$?" >> $O/ncu_q3.log
