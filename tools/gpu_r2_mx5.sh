cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in A T64 T16; do
  if [ "$v" = A ]; then unset CDC_LIB; else export CDC_LIB=$PWD/build/libcdc_$v.so; fi
  echo "== $v"; timeout 600 python tools/maxp_timing.py 2>&1 | tail -4
done
unset CDC_LIB
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_maxp_scan -s 2 -c 1 -o gpurun_out/prof_mx2 -f python tools/maxp_timing.py > gpurun_out/ncu_mx2.log 2>&1; echo full rc=$?
