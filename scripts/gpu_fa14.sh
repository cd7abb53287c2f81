# batched-epilogue attention: parity, A/B vs the committed kernel, cross timeline
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "attention" > gpurun_out/t_attn.log 2>&1; echo "attn tests rc=$?"; tail -1 gpurun_out/t_attn.log; grep -E "^E |FAILED" gpurun_out/t_attn.log | head -5
for v in prod orig prod orig; do
  if [ $v = prod ]; then L=""; else L=$PWD/_variants/$v.so; fi
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | cut -c1-330
done
PAB_LIB_PATH=$PWD/_variants/trace.so TL_ITERS=24 timeout -s KILL 60 python scripts/fa_timeline.py cross > gpurun_out/timeline_cross.txt 2>&1; echo "timeline rc=$?"
