timeout -s KILL 600 python -m pytest tests -q -m gpu -x > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu.log; grep -E "^E |Error|FAILED" gpurun_out/t_gpu.log | head -5
timeout -s KILL 60 python scripts/bench_attn.py --config C3 --impl 1
timeout -s KILL 60 python scripts/bench_attn.py --config C5 --impl 1
timeout -s KILL 300 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"; cat gpurun_out/bench_c3.json | cut -c1-1500
