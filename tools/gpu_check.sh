#!/bin/bash
# One GPU-box pass: build, GPU tests, smoke, the default bench line, the reference arm and
# the ncu launch list of the bench command (config 3).  Outputs under gpurun_out/$TAG.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-chk}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 600 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
if [ "${LAUNCHES:-1}" = 1 ]; then
  CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"panel|window|scan" --csv \
    --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "launch rc=$?" >> $O/ncu_launch.log
fi
