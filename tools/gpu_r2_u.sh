timeout 900 python -m pytest tests/test_gpu_kphase.py -x -q > gpurun_out/t_kp.log 2>&1; echo kphase tests rc=$?
tail -5 gpurun_out/t_kp.log
for k in 2 4 8; do echo "== K=$k"; CDC_KPHASE=$k ONLY=c2 timeout 900 python tools/workloads.py 2>&1 | grep "base" | cut -c1-220; done
CDC_KPHASE=4 K=4 timeout 300 python tools/kphase_timing.py
