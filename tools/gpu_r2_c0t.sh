cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=$((16<<20)) ALGO=ram AVG=8192 DATA=uniform timeout 120 python tools/timing_dump.py > gpurun_out/c0_timing.txt 2>&1
N=$((16<<20)) ALGO=ae_max AVG=8192 DATA=uniform timeout 120 python tools/timing_dump.py >> gpurun_out/c0_timing.txt 2>&1
cat gpurun_out/c0_timing.txt
