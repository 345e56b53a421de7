#!/bin/bash
# Round-2 probe call g: ncu --set full (with source) of one config-2 pencil window launch,
# plus the SN_PPROF phase line of the same build.
set -u
cd "$(dirname "$0")/.."
TAG=${1:-r2g}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
SN_PPROF=1 timeout 600 python tools/bench_pencil.py --config 2 --steps 1 --warmup 0 > $O/pencil_c2.log 2>&1
CMD="python tools/bench_pencil.py --config 2 --steps 1 --warmup 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:pencil_window_kernel -s 30 -c 1 \
  -o $O/pw $CMD > $O/ncu_pw.log 2>&1; echo "ncu rc=$?" >> $O/ncu_pw.log
ncu -i $O/pw.ncu-rep --page source --csv --print-source sass > $O/pw_source_sass.csv 2>&1
ncu -i $O/pw.ncu-rep --page source --csv --print-source cuda > $O/pw_source_cuda.csv 2>&1
python tools/ncu_summary.py $O/pw.ncu-rep > $O/pw_summary.txt 2>&1
rm -f $O/pw.ncu-rep
grep -h '^{' $O/pencil_c2.log; cat $O/pw_summary.txt | head -30
