set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --steps 10 --warmup 3 --check > gpurun_out/b1.json 2> gpurun_out/b1.err; echo bench rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/t1.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/t1.log
