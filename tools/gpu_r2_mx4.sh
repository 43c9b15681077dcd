cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_maxp.py -x -q > gpurun_out/mx.log 2>&1; echo maxp rc=$?
tail -3 gpurun_out/mx.log
timeout 600 python tools/maxp_timing.py 2>&1 | tail -6
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_maxp -c 12 --csv python tools/maxp_timing.py > gpurun_out/mx_ncu.csv 2>/dev/null; echo ncu rc=$?
grep -E "k_maxp" gpurun_out/mx_ncu.csv | awk -F'","' '{print $5" | "$(NF-2)" | "$NF}' | cut -c1-90 | head -12
