#!/bin/bash
# Sharded path on one GPU: parity tests, then the emulated-ranks bench (config 2) vs one GPU.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-dist}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
SN_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -s > $O/pytest_dist.log 2>&1; echo "pytest rc=$?" >> $O/pytest_dist.log
for P in 1 2 4 8; do
  SN_DEBUG=1 timeout 600 python bench.py --config 2 --steps 2 --warmup 3 --emulate-ranks $P >> $O/bench_emu.log 2>&1; echo "emu P=$P rc=$?" >> $O/bench_emu.log
done
timeout 600 python bench.py --config 2 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline >> $O/bench_emu.log 2>&1; echo "single rc=$?" >> $O/bench_emu.log
