cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export N=$((1<<30)) DATA=ver ALGO=ram AVG=16384
timeout 300 python tools/c0_sweep.py > gpurun_out/c2_plain.txt 2>&1; cat gpurun_out/c2_plain.txt | tail -2
AVG=8192 timeout 300 python tools/c0_sweep.py >> gpurun_out/c2_plain.txt 2>&1; tail -1 gpurun_out/c2_plain.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_kspec -s 3 -c 1 -o gpurun_out/prof_c2k -f python tools/c0_sweep.py > gpurun_out/ncu_c2.log 2>&1; echo rc=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 30 --csv --log-file gpurun_out/c2_launches.csv python tools/c0_sweep.py > /dev/null 2>&1; echo rc=$?
