for v in default fpoly2 fpoly3 fpoly0 fnoexp; do
  if [ $v = default ]; then L=""; else L=$PWD/_variants/$v.so; fi
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1
done
