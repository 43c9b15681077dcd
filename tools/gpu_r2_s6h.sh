cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
STAMPS=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_dense_index -s 12 -c 1 -o gpurun_out/prof_dn -f python tools/dense_timing.py > gpurun_out/ncu_dn.log 2>&1; echo rc=$?
