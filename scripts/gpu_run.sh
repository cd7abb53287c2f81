#!/bin/bash
# One parametrised GPU-box entry point (replaces the per-experiment gpu_*.sh logs).
#   scripts/gpu_run.sh tests            -> pytest -m gpu
#   scripts/gpu_run.sh smoke            -> __graft_entry__.smoke()
#   scripts/gpu_run.sh bench [args...]  -> bench.py line
#   scripts/gpu_run.sh probe <binary>   -> run a probe binary
#   scripts/gpu_run.sh py <script> ...  -> any python script
# Several can be chained: scripts/gpu_run.sh tests + smoke + bench --steps 2
mkdir -p gpurun_out
run_one() {
  local what=$1; shift
  case "$what" in
    tests) timeout -s KILL 1200 python -m pytest tests -q -m gpu -x "$@" > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/t_gpu.log ;;
    smoke) timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 ;;
    bench) timeout -s KILL 1200 python bench.py "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.json ;;
    probe) timeout -s KILL 300 "$@" 2>&1 | tee -a gpurun_out/probe.log ;;
    py) timeout -s KILL 1200 python "$@" 2>&1 | tee -a gpurun_out/py.log | tail -40 ;;
    *) echo "unknown step $what" ;;
  esac
}
args=()
for a in "$@"; do
  if [ "$a" = "+" ]; then run_one "${args[@]}"; args=(); else args+=("$a"); fi
done
[ ${#args[@]} -gt 0 ] && run_one "${args[@]}"
exit 0
