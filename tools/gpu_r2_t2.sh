cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in G H; do CDC_LIB=$PWD/build/libcdc_$v.so timeout 600 python -m pytest tests/test_gpu_sparse.py -x -q 2>&1 | tail -1; done
VARIANTS="A G H I" bash tools/gpu_r2_ab.sh
