mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x 2>&1 | tail -1
for v in "" "-DPAB_NO_MUFU_TOKEN"; do
  PAB_NVCC_FLAGS="$v" python -m paper_2408_12588_b200.build --force > /dev/null 2>&1 || echo "build fail $v"
  echo "variant [$v]: $(timeout 120 python scripts/bench_attn.py --config C3 | cut -c1-100)"
  echo "variant [$v]: $(timeout 120 python scripts/bench_attn.py --config C5 | cut -c1-100)"
done
