mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attn_fa_kernel -s 3 -c 3 -o gpurun_out/attn_fa_full python scripts/bench_attn.py --reps 2 > gpurun_out/prof_fa_full.log 2>&1; echo "ncu rc=$?"
timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x > gpurun_out/t_k.log 2>&1; echo "kernel tests rc=$?"; tail -1 gpurun_out/t_k.log
