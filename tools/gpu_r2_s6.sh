# session 6: final profile of HEAD (gpu_prof_r2b.sh) + configs[2] / configs[0] diagnostics
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/gpu_prof_r2b.sh > gpurun_out/prof.log 2>&1
ONLY="c0 c2" timeout 900 python tools/workloads.py > gpurun_out/wl.log 2>&1; echo wl rc=$?
for a in 8192 16384; do
  AVG=$a ALGO=ram timeout 600 python tools/kphase_timing.py > gpurun_out/kt_ram_$a.log 2>&1; echo kt $a rc=$?
done
DATA=ver N=$((1<<30)) ALGO=ram AVG=8192 timeout 600 python tools/timing_dump.py > gpurun_out/td_ram_8192.log 2>&1; echo td rc=$?
cat gpurun_out/wl.log | cut -c1-260
tail -12 gpurun_out/kt_ram_8192.log gpurun_out/kt_ram_16384.log
