cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kphase.py tests/test_gpu_parity.py tests/test_gpu_tables.py tests/test_gpu_fuzz.py tests/test_gpu_sparse.py -x -q > gpurun_out/t4.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/t4.log
for v in A P; do
  if [ "$v" = A ]; then unset CDC_LIB; else export CDC_LIB=$PWD/build/libcdc_$v.so; fi
  echo "== $v"
  timeout 300 python tools/graph_timeline.py 2>&1 | tail -3
  ONLY="c0 c1 c2" timeout 900 python tools/workloads.py 2>&1 | grep -E "c0|c1|ram" | cut -c1-75
done
