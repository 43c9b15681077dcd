cd $GRAFT_REPO_ROOT
echo "== default"; timeout 600 python tools/small_versioned.py
echo "== CDC_DENSE=0"; CDC_DENSE=0 timeout 600 python tools/small_versioned.py
echo "== CDC_DENSE=0 CDC_TMODE=0 (K-phase where its rules allow)"; CDC_DENSE=0 CDC_TMODE=0 timeout 600 python tools/small_versioned.py
echo "== CDC_DENSE=0 CDC_TMODE=0 CDC_KPHASE=4"; CDC_DENSE=0 CDC_TMODE=0 CDC_KPHASE=4 timeout 600 python tools/small_versioned.py
echo "== CDC_DENSE=0 CDC_TMODE=0 CDC_KPHASE=0"; CDC_DENSE=0 CDC_TMODE=0 CDC_KPHASE=0 timeout 600 python tools/small_versioned.py
