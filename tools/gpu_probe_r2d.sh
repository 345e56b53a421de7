#!/bin/bash
# Round-2 probe call d: per-type transform latency of the pencil window kernel (SN_PPROF) and an
# ncu --set full capture of one config-2 pencil window launch.  Outputs under gpurun_out/$TAG.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-r2d}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
SN_PPROF=1 timeout 600 python tools/bench_pencil.py --config 2 --steps 1 --warmup 0 > $O/pencil_c2.log 2>&1
CMD="python tools/bench_pencil.py --config 2 --steps 1 --warmup 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pencil_window_kernel -s 30 -c 1 \
  -o $O/pw $CMD > $O/ncu_pw.log 2>&1; echo "ncu rc=$?" >> $O/ncu_pw.log
ncu -i $O/pw.ncu-rep --page raw --csv > $O/pw_raw.csv 2>&1
ncu -i $O/pw.ncu-rep --page source --csv --print-source sass > $O/pw_source_sass.csv 2>&1
python tools/ncu_summary.py $O/pw.ncu-rep > $O/pw_summary.txt 2>&1
grep -h '^{' $O/pencil_c2.log; cat $O/pw_summary.txt | head -30
