cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_kphase.py -x -q > gpurun_out/t1.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t1.log
VARIANTS="A E F" bash tools/gpu_r2_ab.sh
