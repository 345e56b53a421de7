#!/bin/bash
# ncu --set full captures (source-level) of the Q-update panel kernel and the window kernel
# (config 2), after a plain run of the same command; then the sharded-path GPU tests.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-prof}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; exit 1; }
CMD="python bench.py --config 2 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline"
$CMD > $O/plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"panel_kernel<256, 64, 2" -s 200 -c 1 -o $O/prof_q $CMD > $O/ncu_q.log 2>&1
echo "q rc=$?" >> $O/ncu_q.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:window_kernel -s 60 -c 1 -o $O/prof_w $CMD > $O/ncu_w.log 2>&1
echo "w rc=$?" >> $O/ncu_w.log
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q -s > $O/pytest_dist.log 2>&1; echo "pytest rc=$?" >> $O/pytest_dist.log
