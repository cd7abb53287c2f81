timeout -s KILL 60 python scripts/fa_debug.py 1 3 1560 16 72; echo rc=$?
timeout -s KILL 200 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "attention and not tc_split" > gpurun_out/t_attn.log 2>&1; echo "attn tests rc=$?"; tail -2 gpurun_out/t_attn.log; grep -E "^E |Error" gpurun_out/t_attn.log | head -5
for v in default barr noexp tokpoly3; do
  if [ $v = default ]; then L=""; else L=$PWD/_variants/$v.so; fi
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | cut -c1-200
done
echo "== trace"; PAB_LIB_PATH=$PWD/_variants/trace.so TL_ITERS=8 timeout -s KILL 60 python scripts/fa_timeline.py | tail -40
