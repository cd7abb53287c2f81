# ping-pong attention: parity tests, poly-fraction variants, timeline
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "attention" > gpurun_out/t_attn.log 2>&1; echo "attn tests rc=$?"; tail -2 gpurun_out/t_attn.log; grep -E "^E |FAILED" gpurun_out/t_attn.log | head -5
for v in prod p0 p12 p25 p37; do
  if [ $v = prod ]; then L=""; else L=$PWD/_variants/$v.so; fi
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | cut -c1-400
done
PAB_LIB_PATH=$PWD/_variants/trace.so TL_ITERS=20 timeout -s KILL 60 python scripts/fa_timeline.py > gpurun_out/timeline.txt 2>&1; echo "timeline rc=$?"
