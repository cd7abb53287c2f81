# refresh: ncu full capture of attn_fa (spatial x2, cross x1), step launch lists, bench line
mkdir -p gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:attn_fa_kernel -s 3 -c 3 -o gpurun_out/attn_fa_full -f python scripts/bench_attn.py --reps 2 > gpurun_out/prof_fa_full.log 2>&1; echo "ncu rc=$?"
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_step0.csv python scripts/profile_step.py --config C3 --step 0 > /dev/null 2>&1; echo "step0 rc=$?"
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_step4.csv python scripts/profile_step.py --config C3 --step 4 > /dev/null 2>&1; echo "step4 rc=$?"
timeout -s KILL 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
