mkdir -p gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -c 1 -o gpurun_out/attn_v6 python scripts/bench_attn.py --reps 1 > gpurun_out/prof_attn_v6.log 2>&1; echo "rc=$?"
