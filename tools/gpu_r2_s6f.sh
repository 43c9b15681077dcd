cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py -x -q --tb=short > gpurun_out/t_dense.log 2>&1; echo dense rc=$?; tail -5 gpurun_out/t_dense.log
timeout 300 python tools/dense_timing.py
N=$((64<<20)) timeout 300 python tools/dense_timing.py
