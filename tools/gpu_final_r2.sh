#!/bin/bash
# Round-2 record: build, the whole GPU test suite (durations), smoke, the default bench line
# (config 3, cpu_baseline and e2e), the reference arm, the bench command's ncu launch list, the
# config-2 pencil and rows f3/f4 timings.  Outputs under gpurun_out/$TAG.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-final_r2}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -rA --durations=25 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 600 python bench.py --impl reference > $O/bench_ref.log 2>&1; echo "ref rc=$?" >> $O/bench_ref.log
timeout 600 python tools/bench_pencil.py --config 2 --steps 2 --warmup 1 > $O/pencil_c2.log 2>&1
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"panel|window|scan" --csv \
  --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "launch rc=$?" >> $O/ncu_launch.log
tail -4 $O/pytest_gpu.log; tail -2 $O/smoke.log; grep -h '^{' $O/bench.log | cut -c1-400; grep -h '^{' $O/pencil_c2.log
