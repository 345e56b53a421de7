#!/bin/bash
# Window-kernel variants: quad 2x2|2x2 transform bitwise check + latency, then A/B timings
O=gpurun_out/ab2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt 2>&1
timeout 120 tools/swap_quad_check > $O/quad_check.jsonl 2>&1; echo "quad_check rc=$?" >> $O/quad_check.jsonl
cat $O/quad_check.jsonl
L=paper_1905_04975_b200
timeout 1500 python tools/window_ab.py --configs ${CFGS:-2 3} --reps 3 ${LIBS:-default $L/libsn_b200_q256.so $L/libsn_b200_t384.so $L/libsn_b200_q384.so} > $O/ab.jsonl 2> $O/ab.err
echo rc=$?
cat $O/ab.jsonl; tail -n 5 $O/ab.err
