for v in prod notok pe0 pe4 prod notok pe0 pe4; do
  if [ $v = prod ]; then L=""; else L=$PWD/_variants/$v.so; fi
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | python -c "import json,sys; d=json.load(sys.stdin); print({k: round(v.get('us'),1) for k,v in d.items()})"
done
