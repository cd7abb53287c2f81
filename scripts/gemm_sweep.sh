#!/bin/bash
# A/B sweep of the GEMM tile width and raster group at the C3 projection shapes
for bn in 192 256 128; do for grp in 4 8 16; do
  echo "BN=$bn GROUP=$grp"; PAB_GEMM_BN=$bn PAB_GEMM_GROUP=$grp timeout -s KILL 120 python scripts/bench_gemm.py | python -c "
import json,sys; d=json.load(sys.stdin); print('  ', {k: v['tflops'] for k, v in d.items() if 'ours' in k})"
done; done
