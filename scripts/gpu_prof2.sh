mkdir -p gpurun_out
python scripts/gelu_check.py
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3_step4.csv python scripts/profile_step.py --config C3 --step 4 > /dev/null 2>&1; echo "launches rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc_kernel -c 3 -o gpurun_out/attn_r01 python scripts/bench_attn.py --reps 1 > /dev/null 2>&1; echo "attn full rc=$?"
