# A/B of tuning builds under build/ on the workloads of tools/workloads.py (ONLY= selects)
cd $GRAFT_REPO_ROOT
for v in ${VARIANTS:-A B}; do
  echo "== $v"
  CDC_LIB=$PWD/build/libcdc_$v.so timeout 600 python tools/workloads.py 2>&1 | cut -c1-110
done
