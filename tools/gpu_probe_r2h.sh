#!/bin/bash
# Round-2 probe call h: lane-group Sylvester solve -- bitwise A/B against the previous build,
# pencil GPU tests, phase timing.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-r2h}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
SN_LIB_PATH=paper_1905_04975_b200/libsn_b200_prev.so timeout 600 python tools/pencil_ab_bitwise.py $O/prev.npz 0 > $O/ab.log 2>&1
timeout 600 python tools/pencil_ab_bitwise.py $O/new.npz 0 >> $O/ab.log 2>&1
python tools/pencil_ab_bitwise.py --compare $O/prev.npz $O/new.npz >> $O/ab.log 2>&1
rm -f $O/*.npz
for c in 1 2; do
  SN_PPROF=1 timeout 600 python tools/bench_pencil.py --config $c --steps 2 --warmup 1 > $O/pencil_c$c.log 2>&1
done
timeout 1200 python -m pytest tests/test_gpu_pencil.py -x -q > $O/pytest_pencil.log 2>&1; echo "pytest rc=$?" >> $O/pytest_pencil.log
tail -1 $O/ab.log; tail -3 $O/pytest_pencil.log; grep -h '^{' $O/pencil_*.log
