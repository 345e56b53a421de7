#!/bin/bash
# Round-2 iteration: sweep/eigvec tests, their bench lines, an ncu capture of the eigenvector
# solve kernel and the config-3 Q-update kernel (summaries only).
set -u
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-r02j}
mkdir -p $O
tools/gpu_tests.sh $(basename $O) "tests/test_gpu_sweep.py tests/test_gpu_eigvec.py -m gpu"
SN_EIG_PROFILE=1 ROWS="f3 f4" LAUNCHES=0 tools/gpu_rows.sh $(basename $O)
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:eig_solve_kernel -s 150 -c 1 -o $O/solve python tools/bench_rows.py --row f4 --steps 1 --warmup 0 > $O/ncu_solve.log 2>&1; echo "ncu solve rc=$?"
python tools/ncu_summary.py $O/solve.ncu-rep > $O/solve_summary.txt 2>&1
ncu -i $O/solve.ncu-rep --page source --csv --print-source sass > $O/solve_source_sass.csv 2>&1
rm -f $O/solve.ncu-rep
tools/gpu_prof_q.sh $(basename $O)
