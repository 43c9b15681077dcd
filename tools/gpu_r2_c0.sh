# configs[0] path-selection sweep (T-mode vs K-phase geometries), each in its own process
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { env "$@" timeout 120 python tools/c0_sweep.py 2>&1 | tail -1; }
{
run CDC_X=0
run CDC_TMODE=0
for K in 4 8; do for G in 64 128 256 512; do run CDC_TMODE=0 CDC_KPHASE=$K CDC_KSEGS=$G; done; done
run ALGO=ae_max
run ALGO=ae_max CDC_TMODE=0 CDC_KPHASE=8 CDC_KSEGS=128
run AVG=16384
run AVG=16384 CDC_TMODE=0 CDC_KPHASE=8 CDC_KSEGS=128
} > gpurun_out/c0_sweep.txt
cat gpurun_out/c0_sweep.txt
