set -x
python tools/c3_timing.py > gpurun_out/c3t.log 2>&1; echo c3t rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 --no-secondary --no-e2e > gpurun_out/b2.json 2> gpurun_out/b2.err; echo bench rc=$?
timeout 2000 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/t2.log 2>&1; echo tests rc=$?
tail -8 gpurun_out/t2.log
