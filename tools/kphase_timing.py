"""Per-node walk timing of one K-phase call (diagnostic; not a measurement)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2508_05797_b200 as cdc
from paper_2508_05797_b200._lib import lib

n = int(os.environ.get("N", 1 << 30))
algo = os.environ.get("ALGO", "ram")
avg = int(os.environ.get("AVG", "16384"))
kind = os.environ.get("DATA", "ver")
d = (synth.versioned(n, 0, seed=2)[0] if kind == "ver" else
     synth.alternating(n, region=256 << 20, seed=5) if kind == "alt" else synth.uniform(n, 0))
t = torch.from_numpy(d).cuda()
p = cdc.params(algo, avg_size=avg)
ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(3):
    cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
st = cdc.stats(p, ws, 1, n, n)
K = int(os.environ.get("K", "0")) or (8 if p.window >= 12288 else 4)
N = st["segments"] * K
tm = torch.zeros(8 + 7 * N, dtype=torch.int64, device="cuda")
tm[[0, 2, 3, 5, 6]] = -1
lib.cdc_debug_timing(tm.data_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cdc.chunk_async(t, p, b, c, ws)
e1.record()
torch.cuda.synchronize()
lib.cdc_debug_timing(None)
print(st, "call ms (with stamps)", e0.elapsed_time(e1))
a = tm[8:].cpu().numpy().reshape(N, 7)
t0 = a[:, 0].min()
start, end = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3
cnt = a[:, 2] >> 32
dur = end - start
print("nodes %d  walk us: mean %.1f p50 %.1f p99 %.1f max %.1f  last end %.1f" % (
    N, dur.mean(), np.median(dur), np.percentile(dur, 99), dur.max(), end.max()))
print("entries per node: mean %.1f p99 %.0f max %d  total %d" % (cnt.mean(), np.percentile(cnt, 99), cnt.max(), cnt.sum()))
print("us per entry (walkers in flight): %.3f" % (dur.sum() / max(cnt.sum(), 1)))
for q in (0.25, 0.5, 0.75, 0.9, 1.0):
    print("  nodes started by %.0f%% of the span: %d" % (q * 100, (start <= q * end.max()).sum()))
slow = np.argsort(-dur)[:8]
print("slowest nodes", [(int(v), round(float(dur[v]), 1), int(cnt[v]), round(float(start[v]), 1)) for v in slow])
