# ping-pong continuation copies: parity of the sparse / K-phase / parity suites, then A/B timings
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sparse.py tests/test_gpu_kphase.py tests/test_gpu_parity.py -x -q --tb=short -p no:cacheprovider > gpurun_out/cont_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/cont_pytest.log
for v in A old; do
  if [ "$v" = A ]; then unset CDC_LIB; else export CDC_LIB=$PWD/build/libcdc_$v.so; fi
  for a in "ram 16384" "ram 8192" "ae_max 16384" "ram 4096"; do set -- $a
    N=$((1<<30)) DATA=ver ALGO=$1 AVG=$2 timeout 300 python tools/c0_sweep.py 2>&1 | tail -1 | sed "s/^/$v /"
  done
  N=$((16<<20)) timeout 300 python tools/c0_sweep.py 2>&1 | tail -1 | sed "s/^/$v /"
done
unset CDC_LIB
VARIANTS="A old" STEPS=10 bash tools/gpu_r2_ab.sh
