#!/bin/bash
# Measure the f-rows (tools/bench_rows.py) and capture their ncu launch lists.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-rows}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
for r in ${ROWS:-f4 f3 f2}; do
  timeout 900 python tools/bench_rows.py --row $r --steps ${STEPS:-3} --warmup 1 > $O/bench_$r.jsonl 2> $O/bench_$r.err; echo "$r rc=$?"
  tail -1 $O/bench_$r.jsonl
done
if [ -n "${F3VARIANTS:-}" ]; then
  for v in $F3VARIANTS; do   # window:chain
    timeout 900 python tools/bench_rows.py --row f3 --steps 2 --warmup 1 --window ${v%:*} --chain ${v#*:} >> $O/bench_f3_variants.jsonl 2>> $O/bench_f3_variants.err
    tail -1 $O/bench_f3_variants.jsonl
  done
fi
if [ "${LAUNCHES:-1}" = 1 ]; then
  for r in ${LROWS:-f4 f3}; do
    timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$r.csv \
      python tools/bench_rows.py --row $r --steps 1 --warmup 0 > $O/ncu_$r.log 2>&1; echo "ncu $r rc=$?"
  done
fi
