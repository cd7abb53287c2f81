mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import torch;print(torch.cuda.get_device_name(0))"
timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k "simt or modnorm or ddim or gelu or fill" > gpurun_out/t_simt.log 2>&1; echo "simt rc=$?"
PAB_ATTN_IMPL=simt timeout -s KILL 300 python -m pytest tests/test_model_gpu.py -q -m gpu -x > gpurun_out/t_model_simt.log 2>&1; echo "model rc=$?"
timeout -s KILL 300 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k "tcgen05 or select or null" > gpurun_out/t_tc.log 2>&1; echo "tc rc=$?"
tail -3 gpurun_out/*.log
