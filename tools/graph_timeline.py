"""Launch timeline of one configs[1] call replayed from a CUDA graph (diagnostic;
not a measurement): globaltimer stamps of k_reset / k_speculate / k_fixup and the
walkers' ends, relative to the first walker's start."""
import os, sys
import numpy as np
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
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
G = cdc.stats(p, ws, 1, n, n)["segments"]
tm = torch.zeros(8 + 7 * G, dtype=torch.int64, device="cuda")
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    cdc.chunk_async(t, p, b, c, ws)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(5):
    g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(20):
    g.replay()
e1.record()
torch.cuda.synchronize()
print("graph step ms (no stamps)", e0.elapsed_time(e1) / 20)
for rep in range(3):
    tm.zero_()
    tm[[0, 2, 3, 5, 6]] = -1
    lib.cdc_debug_timing(tm.data_ptr())
    g.replay()
    g.replay()  # the stamps of the second replay overwrite the walker slots; launch slots min/max over both
    torch.cuda.synchronize()
    lib.cdc_debug_timing(None)
tm.zero_()
tm[[0, 2, 3, 5, 6]] = -1
lib.cdc_debug_timing(tm.data_ptr())
g.replay()
torch.cuda.synchronize()
lib.cdc_debug_timing(None)
a = tm.cpu().numpy()
w = a[8:].reshape(G, 7)
t0 = w[:, 0].min()
rel = lambda x: (x - t0) / 1e3
names = ["reset begin", "reset end", "spec begin", "spec waited", "spec end", "fix begin", "fix waited", "fix end"]
print(", ".join("%s %.2f" % (names[i], rel(a[i])) for i in range(8) if a[i] not in (0, -1)))
walk_end, done = rel(w[:, 2]), rel(w[:, 3])
print("walk end us: p50 %.1f p90 %.1f max %.1f; written: p50 %.1f max %.1f" % (
    np.median(walk_end), np.percentile(walk_end, 90), walk_end.max(), np.median(done), done.max()))
