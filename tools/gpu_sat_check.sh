# saturation-index path: parity, uniform workloads (index on and off), configs[1] A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --tb=short > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" > gpurun_out/rc.txt
tail -3 gpurun_out/pytest_gpu.log
ONLY="c0 u256 c4" timeout 600 python tools/workloads.py 2>&1 | cut -c1-200
echo "== CDC_TMODE=0"
CDC_TMODE=0 ONLY="c0" timeout 600 python tools/workloads.py 2>&1 | cut -c1-200
STEPS=200 VARIANTS="${VARIANTS:-P A}" bash tools/gpu_variants.sh 2>&1 | grep step
