"""Per-segment walk timing of one full configs[3] batch call (diagnostic; not a measurement).

Prints the walkers' busy curve and the segments that finish last (their file
sizes and start times): where the batch's k_speculate time goes."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2508_05797_b200 as cdc  # noqa: E402
from paper_2508_05797_b200._lib import lib  # noqa: E402

NF = int(os.environ.get("NF", "100000"))
data_np, offs = synth.many_files(NF, seed=3)
sizes = np.diff(offs)
nf = offs.size - 1
total, max_len = int(offs[-1]), int(sizes.max())
p = cdc.params("ram", avg_size=8192, seg_bytes=int(os.environ.get("SEG", "0")))
t = torch.from_numpy(data_np).cuda()
od = torch.from_numpy(offs).cuda()
cap = total // (p.window + 1) + nf
b = torch.empty(cap, dtype=torch.int64, device="cuda")
bo = torch.zeros(nf + 1, dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = torch.empty(cdc.workspace_size(p, nf, total, max_len), dtype=torch.uint8, device="cuda")
for _ in range(3):
    cdc.chunk_batch_async(t, od, total, max_len, p, b, bo, c, ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    cdc.chunk_batch_async(t, od, total, max_len, p, b, bo, c, ws)
e1.record()
torch.cuda.synchronize()
print("step ms %.3f  (%.1f GB/s)" % (e0.elapsed_time(e1) / 5, total / (e0.elapsed_time(e1) / 5) / 1e6))
cdc.profile_enable(True)
for _ in range(5):
    cdc.chunk_batch_async(t, od, total, max_len, p, b, bo, c, ws)
torch.cuda.synchronize()
cdc.profile_enable(False)
pr = cdc.profile_collect()
print("kernel ms:", {k: round(v[0] / max(1, v[1]), 4) for k, v in pr.items() if k != "calls"})
st = cdc.stats(p, ws, nf, total, max_len)
print(st)
G = st["segments"]
tm = torch.zeros(8 + 7 * G, dtype=torch.int64, device="cuda")
tm[[0, 2, 3, 5, 6]] = -1
lib.cdc_debug_timing(tm.data_ptr())
cdc.chunk_batch_async(t, od, total, max_len, p, b, bo, c, ws)
torch.cuda.synchronize()
lib.cdc_debug_timing(None)
hdr = tm[:8].cpu().numpy().view(np.uint64).astype(np.float64)
a = tm[8:].cpu().numpy().reshape(G, 7).astype(np.float64)
t0 = a[:, 0].min()
names = ["reset begin", "reset end", "spec begin", "spec waited", "spec end", "fix begin", "fix waited", "fix end"]
print("launch stamps us rel. to first walker start:",
      ", ".join(f"{k} {(v - t0) / 1e3:.1f}" if 0 < v < 2**63 else f"{k} -" for k, v in zip(names, hdr)))
start = (a[:, 0] - t0) / 1e3
end = (a[:, 2] - t0) / 1e3
walk = end - start
# segment lengths (batch: one segment per file unless the file exceeds S)
seg_first = np.zeros(nf + 1, dtype=np.int64)
nseg = np.where(sizes == 0, 0, np.where(sizes < st["seg_bytes"], 1, sizes // st["seg_bytes"]))
seg_first[1:] = np.cumsum(nseg)
seg_file = np.repeat(np.arange(nf), nseg)
seg_len = sizes[seg_file] / np.maximum(nseg[seg_file], 1)
print("walkers end: p50 %.1f p90 %.1f p99 %.1f max %.1f us" % (*np.percentile(end, [50, 90, 99]), end.max()))
rate = seg_len / np.maximum(walk, 1e-3) / 1e3
big = seg_len > (1 << 20)
print("per-walk GB/s: all p50 %.2f; segments > 1 MiB: p50 %.2f min %.2f (n=%d)" % (
    np.median(rate), np.median(rate[big]) if big.any() else 0, rate[big].min() if big.any() else 0, big.sum()))
T = end.max()
for q in np.linspace(0, T, 21):
    print("  t=%7.1f us busy walkers %d" % (q, int(((start <= q) & (end > q)).sum())))
last = np.argsort(end)[-15:]
for g in last:
    print("  seg %6d file %6d len %9d start %8.1f end %8.1f (%.2f GB/s)" % (
        g, seg_file[g], seg_len[g], start[g], end[g], rate[g]))
