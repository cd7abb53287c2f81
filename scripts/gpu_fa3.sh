echo "== trace"; PAB_LIB_PATH=$PWD/_variants/trace.so TL_ITERS=12 timeout -s KILL 120 python scripts/fa_timeline.py
echo "== trace nosm"; PAB_LIB_PATH=$PWD/_variants/trace_nosm.so TL_ITERS=8 timeout -s KILL 120 python scripts/fa_timeline.py
