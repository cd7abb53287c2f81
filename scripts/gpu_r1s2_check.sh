mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout -s KILL 900 python -m pytest tests -q -m gpu -x > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_gpu.log
timeout -s KILL 120 python scripts/bench_attn.py --config C3
timeout -s KILL 120 python scripts/bench_attn.py --config C5
timeout -s KILL 300 python scripts/sdpa_compare.py
