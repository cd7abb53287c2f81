timeout -s KILL 60 python scripts/fa_debug.py 1 3 1560 16 72; echo rc=$?
timeout -s KILL 60 python scripts/fa_debug.py 1 1 1560 2 72; echo rc=$?
for k in "spatial_attention and tcgen05" "temporal_attention and tcgen05" "cross_attention and tcgen05" "rising and tcgen05"; do
timeout -s KILL 60 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k "$k" 2>&1 | grep -E "passed|failed|Error" | tail -3; echo "rc=$? [$k]"
done
