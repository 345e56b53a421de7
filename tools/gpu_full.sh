#!/bin/bash
# The round-end sequence: build, every GPU test, smoke, the default bench line, the reference
# arm, and the ncu launch list of the bench command.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-full}
mkdir -p $O
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; free -g; nproc; } > $O/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
start=$(date +%s)
timeout 3000 python -m pytest tests -m gpu -q -rA > $O/pytest_gpu.log 2>&1; echo "pytest rc=$? in $(( $(date +%s) - start )) s"
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -5 $O/smoke.log
timeout 1200 python bench.py > $O/bench.jsonl 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference > $O/bench_ref.jsonl 2> $O/bench_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"panel|window|scan" --csv \
  --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1; echo "launch rc=$?"
