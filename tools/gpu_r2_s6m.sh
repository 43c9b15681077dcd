cd $GRAFT_REPO_ROOT
for K in 2 4; do
echo "== K=$K"
CDC_KPHASE=$K KIND=uniform MIB="256 512" timeout 600 python tools/small_versioned.py | grep "ae_max 16384"
CDC_KPHASE=$K KIND=versioned MIB="256 512" timeout 600 python tools/small_versioned.py | grep "ae_max 16384"
CDC_KPHASE=$K ONLY=c2 timeout 600 python tools/workloads.py 2>&1 | grep "ae_max 16384" | cut -c1-72
done
