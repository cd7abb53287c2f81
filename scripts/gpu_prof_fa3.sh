# ncu full capture (source-level stall sampling) of the spatial attention kernel
mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attn_fa -s 2 -c 1 -o gpurun_out/fa16 -f python scripts/bench_attn.py --config C3 --reps 1 > gpurun_out/ncu_fa16.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_fa16.log
