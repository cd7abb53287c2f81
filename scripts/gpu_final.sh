# final round-1 validation: clean build, GPU suite, smoke, default bench line
mkdir -p gpurun_out
python -c "from paper_2408_12588_b200.build import build; build(force=True)" > gpurun_out/build.log 2>&1; echo "build rc=$?"
timeout -s KILL 900 python -m pytest tests -q -m gpu > gpurun_out/t_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/t_gpu.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
