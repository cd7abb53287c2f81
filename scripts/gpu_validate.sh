mkdir -p gpurun_out
echo "== sanitizer"
for tool in memcheck racecheck synccheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k "spatial_attention and 1-1-300-2-16 or temporal_attention and 2-4-16-4-8 and tcgen05 or cross_attention and 1-64-16-2-72 and tcgen05 or modnorm and 144-1-2 or ddim" > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_$tool.log | tail -2
done
echo "== full-shape parity"
timeout -s KILL 900 python -m pytest tests/test_fullshape_gpu.py -q -m gpu 2>&1 | tail -2
echo "== torchrun N=2 on one GPU (gloo staging)"
PAB_DIST_BACKEND=gloo timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 1 --warmup 1 --config C1 --no-cpu-baseline 2>&1 | grep -E "metric|Error|error" | cut -c1-400
