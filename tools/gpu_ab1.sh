mkdir -p gpurun_out/ab1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ab1/gpu.txt 2>&1
timeout 1500 python tools/window_ab.py --configs 2 3 --reps 3 default paper_1905_04975_b200/libsn_b200_t384.so paper_1905_04975_b200/libsn_b200_t512.so > gpurun_out/ab1/ab.jsonl 2> gpurun_out/ab1/ab.err
echo rc=$?
cat gpurun_out/ab1/ab.jsonl; tail -5 gpurun_out/ab1/ab.err
