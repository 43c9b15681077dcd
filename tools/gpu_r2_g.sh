echo "== sparse default"; python tools/sparse_probe.py
echo "== dense (CDC_SPARSE=0)"; CDC_SPARSE=0 python tools/sparse_probe.py
echo "== counters"; COUNTERS=1 CDC_LIB=build/libcnt.so python tools/sparse_probe.py
echo "== spec 1k"; CDC_LIB=build/libspec1k.so python tools/sparse_probe.py
echo "== spec 4k"; CDC_LIB=build/libspec4k.so python tools/sparse_probe.py
