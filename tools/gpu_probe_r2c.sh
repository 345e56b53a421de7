#!/bin/bash
# Round-2 probe call c: pencil GPU tests (cluster split, host buffers, threaded oracle), the
# pencil phase timing with the per-type warp tasks and the cluster-split transforms, the
# config-3 bench after the panel revert.  Outputs under gpurun_out/$TAG.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-r2c}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_pencil.py -x -q --durations=12 > $O/pytest_pencil.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pencil.log
for c in 1 2; do
  for cl in 1 0; do
    SN_PPROF=1 timeout 600 python tools/bench_pencil.py --config $c --steps 2 --warmup 1 --cluster $cl > $O/pencil_c${c}_cl$cl.log 2>&1
  done
done
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/bench_c3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config1_parity or prefix_parity_config2" --durations=5 > $O/pytest_parity.log 2>&1; echo "pytest rc=$?" >> $O/pytest_parity.log
tail -18 $O/pytest_pencil.log; grep -h '^{' $O/pencil_*.log; tail -8 $O/pytest_parity.log
grep -h '^{' $O/bench_c3.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["kernel_ms_isolated"])'
