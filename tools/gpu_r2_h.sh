echo "== v2 sm_first"; python tools/sparse_probe.py
echo "== v1 LDG"; CDC_LIB=build/libv1.so python tools/sparse_probe.py
echo "== v3 stage_find"; CDC_LIB=build/libv3.so python tools/sparse_probe.py
