set -x
python tools/c3_timing.py > gpurun_out/c3t.log 2>&1; echo c3t rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or config3 or many or fuzz" > gpurun_out/t3.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/t3.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-secondary --no-e2e > gpurun_out/b3.json 2> gpurun_out/b3.err; echo bench rc=$?
