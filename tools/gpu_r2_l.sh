# round-2 re-entry check: GPU tests, smoke, bench at HEAD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t10.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t10.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/b10.json 2> gpurun_out/b10.err; echo bench rc=$?
head -c 600 gpurun_out/b10.json
