cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ONLY="c0 c1 c2 c4 small v128" timeout 1200 python tools/workloads.py > gpurun_out/wl.log 2>&1; echo wl rc=$?
cut -c1-220 gpurun_out/wl.log
K=4 AVG=16384 timeout 300 python tools/kphase_timing.py 2>&1 | tail -12
K=2 AVG=8192 timeout 300 python tools/kphase_timing.py 2>&1 | tail -12
