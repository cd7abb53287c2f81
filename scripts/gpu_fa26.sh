timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py tests/test_model_gpu.py tests/test_fullshape_gpu.py -q -m gpu -x 2>&1 | tail -1
for v in prod nosl prod nosl prod nosl; do
  if [ $v = prod ]; then L=""; else L=$PWD/_variants/$v.so; fi
  for cfg in C3 C5; do
  echo "== $v $cfg"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config $cfg --impl 1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: round(v.get('us'),1) for k,v in d.items()})"
  done
done
