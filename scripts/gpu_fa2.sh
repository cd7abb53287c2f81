mkdir -p gpurun_out
for v in default poly0 poly2 noexp nosm; do
  if [ $v = default ]; then L=""; else L=$PWD/_variants/$v.so; fi
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 120 python scripts/bench_attn.py --config C3 --impl 1
done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_fa_kernel -c 1 -o gpurun_out/fa_v1 python scripts/bench_attn.py --reps 1 > gpurun_out/prof_fa_v1.log 2>&1; echo "ncu rc=$?"
