#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over tools/racecheck_cases.py
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-san}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
for tool in racecheck synccheck memcheck; do
  for c in reorder pencil sweep eigvec; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/racecheck_cases.py $c > $O/${tool}_$c.log 2>&1
    echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $O/${tool}_$c.log | tail -2 | tr '\n' ' ')"
  done
done
