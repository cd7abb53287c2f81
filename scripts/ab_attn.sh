#!/bin/bash
# Same-box A/B of attention kernels across library builds: scripts/ab_attn.sh <config> <rounds> <name=lib.so>...
# ("prod" = the in-tree libpab_b200.so); prints scripts/bench_attn.py's line per build and round.
cfg=$1; rounds=$2; shift 2
for r in $(seq "$rounds"); do
  for spec in "$@"; do
    name=${spec%%=*}; lib=${spec#*=}
    [ "$lib" = prod ] && lib=$PWD/paper_2408_12588_b200/libpab_b200.so
    echo "== $cfg $name"
    PAB_LIB_PATH=$lib timeout 300 python scripts/bench_attn.py --config "$cfg" 2>&1 | tail -1
  done
done
