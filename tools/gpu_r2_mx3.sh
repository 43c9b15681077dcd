cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_maxp_scan -s 2 -c 1 -o gpurun_out/prof_mx -f python tools/maxp_timing.py > gpurun_out/ncu_mx.log 2>&1; echo full rc=$?
