python tools/c3_timing.py > gpurun_out/c3t.log 2>&1; echo c3t rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t6.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t6.log
ONLY=c0,c1,u256,c4,c2 timeout 600 python tools/workloads.py > gpurun_out/wl_sp2.log 2>&1; echo wl rc=$?
