# bulk-copy epilogue + packed K/V slots: parity, A/B, cross timeline
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py tests/test_model_gpu.py -q -m gpu -x > gpurun_out/t_attn.log 2>&1; echo "attn+model tests rc=$?"; tail -1 gpurun_out/t_attn.log; grep -E "^E |FAILED" gpurun_out/t_attn.log | head -5
for v in prod orig layout prod orig; do
  if [ $v = prod ]; then L=""; else L=$PWD/_variants/$v.so; fi
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | cut -c1-330
done
PAB_LIB_PATH=$PWD/_variants/trace.so TL_ITERS=12 timeout -s KILL 60 python scripts/fa_timeline.py cross > gpurun_out/tl_bulk.txt 2>&1
grep -E "it= 3 t=.  sm:(exp_done|p_full)|it= 6 t=.  sm:(exp_done|p_full)" gpurun_out/tl_bulk.txt
