cd $GRAFT_REPO_ROOT
for k in versioned uniform; do
echo "== $k default (K-phase first)"; KIND=$k MIB="128 256 512" timeout 600 python tools/small_versioned.py
echo "== $k CDC_KPHASE=0 (transfer tables first)"; CDC_KPHASE=0 KIND=$k MIB="128 256 512" timeout 600 python tools/small_versioned.py
done
