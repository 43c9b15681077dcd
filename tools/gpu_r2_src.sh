# source-level ncu capture of k_speculate on the configs[3] headline
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-secondary --no-e2e --no-cpu-baseline"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_speculate -s 3 -c 1 -o gpurun_out/prof_src -f $B > gpurun_out/ncu_src.log 2>&1; echo full rc=$?
