#!/bin/bash
# One GPU-box pass for a pytest selection: build, host info, the selected GPU tests.
# usage: tools/gpu_tests.sh TAG "pytest args..."
set -u
cd "$(dirname "$0")/.."
TAG=${1:-t}
SEL=${2:-"tests -m gpu"}
O=gpurun_out/$TAG
mkdir -p $O
{ nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; free -g; nproc; } > $O/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo build failed; tail -30 $O/build.log; exit 1; }
eval timeout ${PT_TIMEOUT:-1500} python -m pytest $SEL -x -q -s -rA > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -5 $O/pytest.log
