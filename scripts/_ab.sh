timeout -s KILL 600 python -m pytest tests/test_gemm_gpu.py tests/test_model_gpu.py -q -x 2>&1 | tail -2
python scripts/bench_gemm.py 2>&1 | grep -A1 -E '"w2_ours"|"w2_resid_ours"' | tr -d '\n '; echo
for v in 1 0 1 0; do PAB_W2_RESID=$v python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-none > gpurun_out/ab$v.json 2> gpurun_out/ab$v.err; python -c "
import json;d=json.loads(open('gpurun_out/ab$v.json').read().strip().splitlines()[-1]); print('w2resid=$v', round(d['value'],4), d['gpu_launches'], d['clocks']['sm_mhz'], round(d['kernels_in_step']['gemm']['w2']['ms'],4))"; done
