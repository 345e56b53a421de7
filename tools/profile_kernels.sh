#!/bin/bash
# ncu captures of the panel and window kernels (config 2), after a plain run of the same command.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-r01b}
CMD="python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_$TAG.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 400 -c 4 -o gpurun_out/prof_panel_$TAG $CMD > gpurun_out/ncu_panel_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:window_kernel -s 100 -c 1 -o gpurun_out/prof_window_$TAG $CMD > gpurun_out/ncu_window_$TAG.log 2>&1
echo done
