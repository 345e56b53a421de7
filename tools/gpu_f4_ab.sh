#!/bin/bash
# Row f4 A/B (base build vs current, bitwise digests), the SN_EIG_PROFILE phase split, eigvec GPU tests
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-f4ab}
mkdir -p $O
timeout 900 python tools/eigvec_ab.py --reps 3 paper_1905_04975_b200/libsn_b200_base.so default paper_1905_04975_b200/libsn_b200_base.so default > $O/ab.jsonl 2> $O/ab.err
echo "ab rc=$?"; cat $O/ab.jsonl; tail -n 3 $O/ab.err
SN_EIG_PROFILE=1 timeout 600 python tools/bench_rows.py --row f4 --steps 3 --warmup 1 > $O/rows_f4.jsonl 2> $O/rows_f4.err
cat $O/rows_f4.jsonl; tail -n 5 $O/rows_f4.err
timeout 1200 python -m pytest tests/test_gpu_eigvec.py -q -rA > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -n 8 $O/pytest.log
