#!/bin/bash
# Bench lines of the other BASELINE configs and the N-core CPU baseline row (config 2).
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-cfg}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); import oracle; oracle.build(omp=True)" > $O/build.log 2>&1 || exit 1
for c in 0 1 2; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --e2e-steps 1 > $O/bench_config$c.jsonl 2> $O/bench_config$c.err; echo "config $c rc=$?"
done
timeout 1500 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 1 > $O/bench_config4.jsonl 2> $O/bench_config4.err; echo "config 4 rc=$?"
timeout 1800 python tools/cpu_baseline_config2.py 2 > $O/cpu_baseline_config2.jsonl 2> $O/cpu_baseline_config2.err; echo "cpu baseline rc=$?"
cat $O/cpu_baseline_config2.jsonl
