cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/maxp_timing.py 2>&1 | tail -6
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_maxp -c 20 --csv python tools/maxp_timing.py > gpurun_out/mx_ncu.csv 2>/dev/null; echo ncu rc=$?
grep -E "k_maxp" gpurun_out/mx_ncu.csv | awk -F'","' '{print $5" | "$(NF-2)" | "$NF}' | head -24
