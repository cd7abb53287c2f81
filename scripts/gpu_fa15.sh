# epilogue bisection: no global stores / no TMEM loads (timing diagnostics only)
mkdir -p gpurun_out
for v in nost_p nold_p; do
  echo "== $v"; PAB_LIB_PATH=$PWD/_variants/$v.so timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | cut -c1-330
done
echo "== prod"; timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | cut -c1-330
for v in trace nost nold; do
  PAB_LIB_PATH=$PWD/_variants/$v.so TL_ITERS=12 timeout -s KILL 60 python scripts/fa_timeline.py cross > gpurun_out/tl_$v.txt 2>&1
  echo "== $v"; grep -E "it= 3 t=.  sm:(exp_done|p_full)|it= 6 t=.  sm:(exp_done|p_full)" gpurun_out/tl_$v.txt
done
