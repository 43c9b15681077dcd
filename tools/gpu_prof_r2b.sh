# round-2 final profile: the default bench line, the ncu launch list of the
# headline command, one ncu --set full capture of k_speculate (batch instance)
# and of k_maxp_scan, and the MAXP launch list
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench rc=$?
B="python bench.py --steps 2 --warmup 3 --no-secondary --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k_speculate -s 3 -c 1 -o gpurun_out/prof_c3 -f $B > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
timeout 600 python tools/maxp_timing.py > gpurun_out/mx_plain.log 2>&1; echo mx plain rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_maxp -c 60 --csv --log-file gpurun_out/mx_launches.csv python tools/maxp_timing.py > gpurun_out/ncu_mx_launch.log 2>&1; echo mx launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_maxp_scan -s 2 -c 1 -o gpurun_out/prof_mx -f python tools/maxp_timing.py > gpurun_out/ncu_mx_full.log 2>&1; echo mx full rc=$?
