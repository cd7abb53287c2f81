# ncu captures behind profiles/ (free-running clocks, the bench's regime), launch lists, bench line
#   bash scripts/gpu_profile.sh            (on the GPU box, from the repo root)
N="ncu --set full --import-source on --clock-control none"
$N -k regex:attn_fa --launch-skip 3 -c 1 -o gpurun_out/ncu_spatial python scripts/bench_attn.py --reps 1 > gpurun_out/ncu.log 2>&1
$N -k regex:attn_fa --launch-skip 7 -c 1 -o gpurun_out/ncu_cross python scripts/bench_attn.py --reps 1 >> gpurun_out/ncu.log 2>&1
$N -k regex:attn_tm --launch-skip 3 -c 1 -o gpurun_out/ncu_temporal python scripts/bench_attn.py --reps 1 >> gpurun_out/ncu.log 2>&1
$N -k regex:attn_tm --launch-skip 3 -c 1 -o gpurun_out/ncu_temporal_c5 python scripts/bench_attn.py --reps 1 --config C5 >> gpurun_out/ncu.log 2>&1
for s in 0 4; do
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_s$s.csv python scripts/profile_step.py --config C3 --step $s > /dev/null 2>&1
done
