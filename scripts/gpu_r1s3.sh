# round-1 session-3 state check: gpu tests, attention variants, timeline, bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout -s KILL 900 python -m pytest tests -q -m gpu -x > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu.log; grep -E "^E |FAILED" gpurun_out/t_gpu.log | head -5
for v in prod noexp barr s2; do
  if [ $v = prod ]; then L=""; else L=$PWD/_variants/$v.so; fi
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | cut -c1-400
done
PAB_LIB_PATH=$PWD/_variants/trace.so TL_ITERS=20 timeout -s KILL 60 python scripts/fa_timeline.py > gpurun_out/timeline.txt 2>&1; echo "timeline rc=$?"
timeout -s KILL 600 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"; cut -c1-3000 gpurun_out/bench_c3.json
