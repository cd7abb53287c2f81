mkdir -p gpurun_out
timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x > gpurun_out/t_k.log 2>&1; echo "kernel tests rc=$?"; tail -3 gpurun_out/t_k.log
timeout -s KILL 120 python scripts/bench_attn.py --config C3
timeout -s KILL 120 python scripts/bench_attn.py --config C5
