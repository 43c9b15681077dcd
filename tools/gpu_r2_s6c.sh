cd $GRAFT_REPO_ROOT
for v in T1 T2; do
  echo "== $v"; CDC_LIB=$PWD/build/libcdc_$v.so SPTIME=1 timeout 600 python tools/sparse_probe.py 2>&1 | tail -8
done
