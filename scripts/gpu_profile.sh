# ncu captures behind profiles/ (free-running clocks, the bench's regime), launch lists,
# sanitizer passes and the C3 bench line; run on the GPU box from the repo root:
#   bash scripts/gpu_profile.sh
mkdir -p gpurun_out
N="ncu --set full --import-source on --clock-control none"
$N -k regex:attn_fa --launch-skip 3 -c 1 -o gpurun_out/ncu_spatial python scripts/bench_attn.py --reps 1 > gpurun_out/ncu.log 2>&1
$N -k regex:attn_fa --launch-skip 7 -c 1 -o gpurun_out/ncu_cross python scripts/bench_attn.py --reps 1 >> gpurun_out/ncu.log 2>&1
$N -k regex:attn_tm --launch-skip 3 -c 1 -o gpurun_out/ncu_temporal python scripts/bench_attn.py --reps 1 >> gpurun_out/ncu.log 2>&1
for s in 0 4; do
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_s$s.csv python scripts/profile_step.py --config C3 --step $s > /dev/null 2>&1
done
# memcheck / racecheck of the kernels changed this round (attention epilogue warps, peer barrier,
# residual GEMM h output, diff sums) on small shapes
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_kernels_gpu.py \
      tests/test_gemm_gpu.py -q -x -k "cross or spatial or residual_h or tails" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_$tool.log
done
python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
