# S prefetch + setmaxnreg variants of the in-phase attention kernel
mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "attention" > gpurun_out/t_attn.log 2>&1; echo "attn tests rc=$?"; tail -1 gpurun_out/t_attn.log; grep -E "^E |FAILED" gpurun_out/t_attn.log | head -5
for v in prod orig nopf noregs p12 p4 p0 prod orig; do
  if [ $v = prod ]; then L=""; else L=$PWD/_variants/$v.so; fi
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | cut -c1-330
done
