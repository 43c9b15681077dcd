timeout 900 python -m pytest tests/test_gpu_kphase.py -x -q > gpurun_out/t_kp.log 2>&1; echo kphase tests rc=$?
tail -5 gpurun_out/t_kp.log
ONLY=c2,c4 timeout 900 python tools/workloads.py 2>&1 | cut -c1-250
for k in 2 4 8; do echo "== K=$k"; CDC_KPHASE=$k ONLY=c2 timeout 900 python tools/workloads.py 2>&1 | grep "base" | cut -c1-200; done
