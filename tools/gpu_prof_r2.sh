# round-2 profile of the bench (configs[3] headline): the bench line, the ncu
# launch list of the same command, and one ncu --set full capture of k_speculate
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench rc=$?
B="python bench.py --steps 2 --warmup 3 --no-secondary --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_speculate -s 3 -c 1 -o gpurun_out/prof_c3 -f $B > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
