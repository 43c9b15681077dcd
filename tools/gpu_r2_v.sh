CDC_KPHASE=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_kspec -s 2 -c 1 -o gpurun_out/prof_kp -f python tools/kphase_timing.py > gpurun_out/ncu_kp.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_kp.log
