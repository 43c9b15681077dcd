python tools/c3_timing.py > gpurun_out/c3t.log 2>&1; echo c3t rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or config3 or many or fuzz" > gpurun_out/t5.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/t5.log
