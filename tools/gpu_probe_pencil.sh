#!/bin/bash
# Phase timing of the pencil window kernel (SN_PPROF) at the config-1 and config-2 pencils.
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-pprobe}
mkdir -p $O
[ -f paper_1905_04975_b200/libsn_b200.so ] || python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for c in ${CONFIGS:-1 2}; do
  SN_PPROF=1 timeout 600 python tools/bench_pencil.py --config $c --steps 1 --warmup 0 > $O/c$c.log 2>&1
  grep -h '^{' $O/c$c.log >> $O/summary.jsonl
done
cat $O/summary.jsonl
