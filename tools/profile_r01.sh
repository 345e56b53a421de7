#!/bin/bash
# Round-1 measurement on the GPU box: bench line, launch list, ncu full captures.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_r01.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_r01.log
CMD="python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0"
$CMD > gpurun_out/plain_c2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $CMD > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_launch.log
ncu --set full --clock-control none --import-source on -k regex:panel_kernel -s 300 -c 3 -o gpurun_out/prof_panel $CMD > gpurun_out/ncu_panel.log 2>&1
echo "panel rc=$?" >> gpurun_out/ncu_panel.log
ncu --set full --clock-control none --import-source on -k regex:window_kernel -s 60 -c 1 -o gpurun_out/prof_window $CMD > gpurun_out/ncu_window.log 2>&1
echo "window rc=$?" >> gpurun_out/ncu_window.log
