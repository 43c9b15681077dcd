CDC_SYNC_DEBUG=1 timeout 300 python tools/kphase_debug.py 2>&1 | tail -8
timeout 300 python tools/kphase_debug.py 2>&1 | tail -8
