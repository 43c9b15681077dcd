# K-phase: parity tests, then the configs[2]/[4] workloads against the previous build
timeout 900 python -m pytest tests/test_gpu_kphase.py -x -q > gpurun_out/t_kp.log 2>&1; echo kphase tests rc=$?
tail -15 gpurun_out/t_kp.log
for v in old new; do
  if [ $v = old ]; then export CDC_LIB=$PWD/build/libcdc_old.so; else unset CDC_LIB; fi
  echo "== $v"; ONLY=c2,c4 timeout 900 python tools/workloads.py 2>&1 | cut -c1-250
done
