#!/bin/bash
# Round-2 probe call: (1) A/B of the config-3 bench, base library vs current, alternating;
# (2) Q-kernel SN_TMA_DBG timing variants; (3) pencil window phases and the cluster split;
# (4) the panel / pencil GPU tests touched by the change.  Outputs under gpurun_out/$TAG.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-r2b}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
B="--config 3 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
for r in 1 2; do
  SN_LIB_PATH=paper_1905_04975_b200/libsn_b200_base.so timeout 600 python bench.py $B > $O/ab_base_$r.log 2>&1
  timeout 600 python bench.py $B > $O/ab_new_$r.log 2>&1
done
for f in $O/ab_*.log; do echo "$f $(grep -h '^{' $f | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["kernel_ms_isolated"])')"; done > $O/ab_summary.txt
for c in 1 2; do
  for cl in 1 0; do
    SN_PPROF=1 timeout 600 python tools/bench_pencil.py --config $c --steps 2 --warmup 1 --cluster $cl > $O/pencil_c${c}_cl$cl.log 2>&1
  done
done
timeout 1200 python -m pytest tests/test_gpu_pencil.py tests/test_gpu_parity.py -x -q --durations=30 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
VARIANTS="0 2 32 8 64" bash tools/gpu_q_probe.sh $TAG/qprobe > /dev/null 2>&1
cat $O/ab_summary.txt; grep -h '^{' $O/pencil_*.log; tail -3 $O/pytest.log; cat $O/qprobe/summary.jsonl
