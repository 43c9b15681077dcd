# end of round 2: whole -m gpu suite, smoke, then the final profile (tools/gpu_prof_r2b.sh: default bench line,
# ncu launch list, k_speculate and k_maxp_scan full captures), the configs[0] dense-mode launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/rc.txt
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
bash tools/gpu_prof_r2b.sh > gpurun_out/prof.log 2>&1
grep "rc=" gpurun_out/prof.log >> gpurun_out/rc.txt
STAMPS=1 timeout 300 python tools/dense_timing.py > gpurun_out/dense_timing.txt 2>&1
STAMPS=0 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 30 -c 30 --csv --log-file gpurun_out/dn_launches.csv python tools/dense_timing.py > /dev/null 2>&1; echo "dn launches rc=$?" >> gpurun_out/rc.txt
cat gpurun_out/rc.txt
tail -1 gpurun_out/bench.log | cut -c1-400
