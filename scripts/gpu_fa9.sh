for v in notoken barr noexp; do
  L=$PWD/_variants/$v.so
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1
done
