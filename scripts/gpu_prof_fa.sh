mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attn_fa_kernel -c 1 -o gpurun_out/fa_v2 python scripts/bench_attn.py --reps 1 > gpurun_out/prof_fa_v2.log 2>&1; echo "ncu rc=$?"
