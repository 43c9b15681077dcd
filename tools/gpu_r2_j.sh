python tools/c3_timing.py > gpurun_out/c3t.log 2>&1; echo c3t rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t8.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/t8.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/b8.json 2> gpurun_out/b8.err; echo bench rc=$?
