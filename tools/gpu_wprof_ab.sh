#!/bin/bash
# Window-kernel phase cycles (SN_WPROF) of the default library and the variants in $LIBS (config 2)
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-wprof_ab}
mkdir -p $O
for L in default ${LIBS:-}; do
  if [ "$L" = default ]; then unset SN_LIB_PATH; else export SN_LIB_PATH=$PWD/$L; fi
  echo "== $L" >> $O/wprof.txt
  SN_WPROF=1 timeout 600 python tools/wprof.py 2 >> $O/wprof.txt 2>&1
done
unset SN_LIB_PATH
cat $O/wprof.txt
