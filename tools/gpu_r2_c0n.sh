cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_speculate -s 3 -c 1 -o gpurun_out/prof_c0 -f python tools/c0_sweep.py > gpurun_out/ncu_c0.log 2>&1; echo rc=$?
tail -3 gpurun_out/ncu_c0.log
