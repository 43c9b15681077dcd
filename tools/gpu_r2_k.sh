python tools/c3_timing.py > gpurun_out/c3t.log 2>&1; echo c3t rc=$?
ONLY=c0,c1,u256,c4,c2 timeout 600 python tools/workloads.py > gpurun_out/wl_y.log 2>&1; echo wl rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t9.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/t9.log
