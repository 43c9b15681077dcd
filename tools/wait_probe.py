"""Fraction of walker time spent waiting for TMA stages (CDC_WAIT_PROBE build; diagnostic)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2508_05797_b200 as cdc
from paper_2508_05797_b200._lib import lib
n = 256 << 20
d = synth.zipf_bytes(n, 1.1, 1)
t = torch.from_numpy(d).cuda()
p = cdc.params("ae_max", avg_size=4096)
ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
ns = ctypes.c_ulonglong()
for _ in range(3):
    cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
lib.cdc_debug_wait_ns(ctypes.byref(ns))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cdc.chunk_async(t, p, b, c, ws)
e1.record()
torch.cuda.synchronize()
lib.cdc_debug_wait_ns(ctypes.byref(ns))
st = cdc.stats(p, ws, 1, n, n)
ms = e0.elapsed_time(e1)
G = st["segments"]
print("step ms %.3f  warps %d  summed wait %.1f us  avg wait per warp %.1f us (%.0f%% of step)" % (ms, G, ns.value / 1e3, ns.value / 1e3 / G, 100 * ns.value / 1e6 / G / ms))
