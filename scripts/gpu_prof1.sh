mkdir -p gpurun_out
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_step0.csv python scripts/profile_step.py --config C3 --step 0 > gpurun_out/prof_step0.log 2>&1; echo "launch list rc=$?"
timeout -s KILL 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_tc_kernel -c 3 -o gpurun_out/attn_c3 python scripts/profile_step.py --config C3 --step 0 > gpurun_out/prof_full.log 2>&1; echo "full rc=$?"
timeout -s KILL 600 ncu --profile-from-start off --set full --clock-control none -k regex:residual_modnorm -c 2 -o gpurun_out/modnorm_c3 python scripts/profile_step.py --config C3 --step 0 > gpurun_out/prof_mn.log 2>&1; echo "full mn rc=$?"
ls -la gpurun_out
