PAB_LIB_PATH=$PWD/_variants/s1.so timeout -s KILL 60 python scripts/fa_debug.py 1 3 1560 16 72; echo rc=$?
PAB_LIB_PATH=$PWD/_variants/s1.so timeout -s KILL 200 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "attention and not tc_split" > gpurun_out/t_attn.log 2>&1; echo "attn tests rc=$?"; tail -1 gpurun_out/t_attn.log
PAB_LIB_PATH=$PWD/_variants/s2p3.so timeout -s KILL 200 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "attention and not tc_split" > gpurun_out/t_attn2.log 2>&1; echo "attn tests s2 rc=$?"; tail -1 gpurun_out/t_attn2.log
for v in s1 s1barr s1noexp s1p3 s2p3 s2barr; do
  L=$PWD/_variants/$v.so
  echo "== $v"; PAB_LIB_PATH=$L timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1 | cut -c1-100
done
