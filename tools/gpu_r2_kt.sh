cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for avg in 16384 8192; do AVG=$avg K=$([ $avg = 16384 ] && echo 4 || echo 2) timeout 300 python tools/kphase_timing.py; done > gpurun_out/kt.txt 2>&1
cat gpurun_out/kt.txt
