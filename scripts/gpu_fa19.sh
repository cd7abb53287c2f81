timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x > gpurun_out/t_attn.log 2>&1; echo "attn tests rc=$?"; tail -1 gpurun_out/t_attn.log; grep -E "^E |FAILED" gpurun_out/t_attn.log | head -5
for v in prod nopm orig prod nopm orig; do
  if [ $v = prod ]; then L=""; else L=$PWD/_variants/$v.so; fi
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: round(v.get('us'),1) for k,v in d.items()})"
done
