for v in "" "-DPAB_POLY_EVERY=0" "-DPAB_POLY_EVERY=4"; do
  PAB_NVCC_FLAGS="$v" python -m paper_2408_12588_b200.build --force > /dev/null 2>&1 || echo "build fail $v"
  echo "variant [$v]: $(timeout 120 python scripts/bench_attn.py --config C3 | cut -c1-100)"
done
python -m pytest tests/test_kernels_gpu.py -q -m gpu -x 2>&1 | tail -1
