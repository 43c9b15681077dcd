cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_kphase.py tests/test_gpu_tables.py -x -q > gpurun_out/t5.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/t5.log
for v in A B; do
  if [ "$v" = A ]; then unset CDC_LIB; else export CDC_LIB=$PWD/build/libcdc_$v.so; fi
  echo "== $v"; ONLY="c0 c1 c2 c4" timeout 900 python tools/workloads.py 2>&1 | grep -E "c0|c1|c4|ram|ae_max" | cut -c1-72
done
