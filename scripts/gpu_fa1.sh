mkdir -p gpurun_out
timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k "attention" > gpurun_out/t_attn.log 2>&1; echo "attn tests rc=$?"; grep -E "passed|failed|Error|assert" gpurun_out/t_attn.log | head -20
timeout -s KILL 120 python scripts/bench_attn.py --config C3 --impl 1
timeout -s KILL 120 python scripts/bench_attn.py --config C3 --impl 3
timeout -s KILL 120 python scripts/bench_attn.py --config C5 --impl 1
