timeout -s KILL 600 python -m pytest tests -q -m gpu -x > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/t_gpu.log; grep -E "FAILED" gpurun_out/t_gpu.log | head -3
for v in prod nowin orig prod nowin orig; do
  if [ $v = prod ]; then L=""; else L=$PWD/_variants/$v.so; fi
  for cfg in C3 C5; do
  echo "== $v $cfg"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config $cfg --impl 1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: round(v.get('us'),1) for k,v in d.items()})"
  done
done
