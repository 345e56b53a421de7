#!/bin/bash
# Timing probes of the Q-update panel kernel (config 3): SN_TMA_DBG variants applied to kind 2
# only (Q results are then wrong; nothing downstream reads Q).  Each line: the variant and the
# bench line's isolated per-kind kernel times.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-qprobe}
mkdir -p $O
[ -f paper_1905_04975_b200/libsn_b200.so ] || python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for v in ${VARIANTS:-0 2 32 8 64 34 40 0}; do
  SN_TMA_DBG=$v SN_TMA_DBG_KINDS=4 timeout 600 python bench.py --config ${CFG:-3} --steps 1 --warmup 3 --e2e-steps 0 \
    --no-cpu-baseline > $O/v$v.log 2>&1
  python - "$v" "$O/v$v.log" >> $O/summary.jsonl <<'PY'
import json, sys
v, p = sys.argv[1], sys.argv[2]
line = [l for l in open(p) if l.startswith('{')]
d = json.loads(line[-1]) if line else {}
print(json.dumps({"dbg": int(v), "ms_per_step": d.get("ms_per_step"), "kernel_ms_isolated": d.get("kernel_ms_isolated")}))
PY
done
cat $O/summary.jsonl
