cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_abi.py -x -q > gpurun_out/t3.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t3.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "config3" > gpurun_out/t3b.log 2>&1; echo fullsize rc=$?
tail -2 gpurun_out/t3b.log
VARIANTS="A K" BENCH_ARGS=" " bash tools/gpu_r2_ab.sh
