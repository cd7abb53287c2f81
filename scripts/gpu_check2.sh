mkdir -p gpurun_out
export PAB_TEST_REPORT=1
timeout -s KILL 600 python -m pytest tests/test_model_gpu.py -q -m gpu -rA > gpurun_out/t_model.log 2>&1; echo "model rc=$?"
timeout -s KILL 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout -s KILL 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
tail -5 gpurun_out/smoke.log gpurun_out/bench1.log
