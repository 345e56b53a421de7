#!/bin/bash
# Round record: GPU tests, smoke, the default bench line (with cpu_baseline and e2e), the
# reference arm, the launch list of the bench command, and ncu --set full captures of the
# window kernel and the left-update kernel (config 2).  Outputs under gpurun_out/$TAG.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
bash tools/gpu_check.sh $TAG
CMD="python bench.py --config 2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > $O/plain_c2.log 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:window_kernel -s 60 -c 1 \
  -o $O/prof_window $CMD > $O/ncu_window.log 2>&1; echo "w rc=$?" >> $O/ncu_window.log
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"panel_tma_kernel<.int.256, .int.0" -s 200 -c 1 -o $O/prof_left $CMD > $O/ncu_left.log 2>&1
echo "l rc=$?" >> $O/ncu_left.log
