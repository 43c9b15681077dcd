# lone-walker cycle accounting of the sparse walk, HEAD vs lean (CDC_SPTIME builds)
for v in old new; do
  echo "== $v"; SPTIME=1 CDC_LIB=$PWD/build/libcdc_${v}_spt.so timeout 300 python tools/sparse_probe.py 2>&1 | tail -6
  echo "== $v plain"; CDC_LIB=$PWD/build/libcdc_old.so; [ $v = new ] && unset CDC_LIB; timeout 300 python tools/sparse_probe.py 2>&1 | tail -6
done
