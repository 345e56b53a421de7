#!/bin/bash
# Iteration pass: build, all GPU tests, the default bench line, then (optional) ncu captures.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-iter}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
if [ "${PROF:-0}" = 1 ]; then
  CMD="python bench.py --config 2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
  $CMD > $O/plain.log 2>&1 || { echo plain failed; exit 1; }
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k regex:"${KREGEX:-panel_tma_kernel<.int.256, .int.2}" -s ${KSKIP:-200} -c 1 -o $O/prof_q $CMD > $O/ncu_q.log 2>&1
  echo "q rc=$?" >> $O/ncu_q.log
fi
