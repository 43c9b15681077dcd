cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_dense.py tests/test_gpu_kphase.py tests/test_gpu_tables.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_sparse.py -x -q --tb=short > gpurun_out/t6j.log 2>&1; echo tests rc=$?; tail -4 gpurun_out/t6j.log
STAMPS=0 timeout 300 python tools/dense_timing.py
timeout 600 python tools/small_versioned.py
