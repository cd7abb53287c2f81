for v in "" "-DPAB_DIAG_FAKE_EXP -DPAB_POLY_EVERY=0" "-DPAB_NO_MUFU_TOKEN -DPAB_DIAG_FAKE_EXP -DPAB_POLY_EVERY=0"; do
  PAB_NVCC_FLAGS="$v" python -m paper_2408_12588_b200.build --force > /dev/null 2>&1 || echo "build fail $v"
  echo "variant [$v]: $(timeout 120 python scripts/bench_attn.py --config C3 | cut -c1-100)"
done
