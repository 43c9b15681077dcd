cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/maxp_debug.py 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_maxp.py -x -q 2>&1 | tail -2
for v in A X256 X1024; do
  if [ "$v" = A ]; then unset CDC_LIB; else export CDC_LIB=$PWD/build/libcdc_$v.so; fi
  echo "== $v"; timeout 600 python tools/maxp_timing.py 2>&1 | tail -4
done
