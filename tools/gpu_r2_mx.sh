cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_maxp.py -x -q --durations=5 > gpurun_out/mx.log 2>&1; echo maxp rc=$?
tail -25 gpurun_out/mx.log
