# round-1 session-3: full GPU tests, multi-rank bench paths (gloo on one GPU), step launch lists, bench line
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests -q -m gpu -x > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/t_gpu.log; grep -E "^E |FAILED" gpurun_out/t_gpu.log | head -5
for spec in "2 C1 " "2 C1cfg --split-batch" "4 C1cfg --split-batch" "4 C1cfg "; do
  set -- $spec
  echo "== torchrun N=$1 $2 $3"
  PAB_DIST_BACKEND=gloo timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus $1 --steps 1 --warmup 1 --config $2 $3 --no-cpu-baseline 2>&1 | grep -E "metric|Error|error" | cut -c1-300
done
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_step0.csv python scripts/profile_step.py --config C3 --step 0 > /dev/null 2>&1; echo "step0 rc=$?"
timeout -s KILL 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_step4.csv python scripts/profile_step.py --config C3 --step 4 > /dev/null 2>&1; echo "step4 rc=$?"
timeout -s KILL 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"; cut -c1-600 gpurun_out/bench_c3.json
