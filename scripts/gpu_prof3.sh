mkdir -p gpurun_out
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_step0.csv python scripts/profile_step.py --config C3 --step 0 > /dev/null 2>&1; echo "step0 rc=$?"
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_step4.csv python scripts/profile_step.py --config C3 --step 4 > /dev/null 2>&1; echo "step4 rc=$?"
timeout -s KILL 900 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -c 3 -o gpurun_out/r01_attn_final python scripts/bench_attn.py --reps 1 > /dev/null 2>&1; echo "attn rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none -k regex:residual_modnorm -c 2 -o gpurun_out/r01_modnorm_final python scripts/bench_modnorm.py > /dev/null 2>&1; echo "mn rc=$?"
python bench.py --steps 3 --warmup 3 > gpurun_out/r01_bench_final.log 2>&1; echo "bench rc=$?"
