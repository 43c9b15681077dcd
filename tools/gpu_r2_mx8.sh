# k_maxp_scan variants: schedule (ticket / static), next-tile L2 prefetch, tile size
cd $GRAFT_REPO_ROOT
for v in A mxs mxsp mxtp t16 t16s t8 old; do
  if [ "$v" = A ]; then unset CDC_LIB; else export CDC_LIB=$PWD/build/libcdc_$v.so; fi
  echo "== $v"; timeout 300 python tools/maxp_timing.py 2>&1 | grep -v "^$"
done
unset CDC_LIB
for v in t16 t8; do CDC_LIB=$PWD/build/libcdc_$v.so timeout 600 python -m pytest tests/test_gpu_maxp.py -x -q -p no:cacheprovider 2>&1 | tail -1; done
