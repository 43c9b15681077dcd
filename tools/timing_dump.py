"""Per-segment walk timing of one configs[1] call (diagnostic; not a measurement)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2508_05797_b200 as cdc  # noqa: E402
from paper_2508_05797_b200._lib import lib  # noqa: E402

n = int(os.environ.get("N", 256 << 20))
algo = os.environ.get("ALGO", "ae_max")
avg = int(os.environ.get("AVG", "4096"))
seg = int(os.environ.get("SEG", "0"))
kind = os.environ.get("DATA", "zipf")
d = (synth.zipf_bytes(n, 1.1, 1) if kind == "zipf" else
     synth.alternating(n, region=256 << 20, seed=5) if kind == "alt" else
     synth.versioned(n, 0, seed=2)[0] if kind == "ver" else synth.uniform(n, 0))
t = torch.from_numpy(d).cuda()
p = cdc.params(algo, avg_size=avg, seg_bytes=seg)
ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
cap = cdc.max_boundaries(p, n)
b = torch.empty(cap, dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(3):
    cdc.chunk_async(t, p, b, c, ws)
st = cdc.stats(p, ws, 1, n, n)
G = st["segments"]
tm = torch.zeros(8 + 7 * G, dtype=torch.int64, device="cuda")
tm[[0, 2, 3, 5, 6]] = -1  # "first" stamps: atomicMin slots
lib.cdc_debug_timing(tm.data_ptr())
cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
lib.cdc_debug_timing(None)
hdr = tm[:8].cpu().numpy().view(np.uint64).astype(np.float64)
a = tm[8:].cpu().numpy().reshape(G, 7)
t0 = a[:, 0].min()
names = ["reset begin", "reset end", "spec begin", "spec waited", "spec end", "fix begin", "fix waited", "fix end"]
print("launch stamps us rel. to first walker start:",
      ", ".join(f"{k} {(v - t0) / 1e3:.2f}" if 0 < v < 2**63 else f"{k} -" for k, v in zip(names, hdr)))
start = (a[:, 0] - t0) / 1e3
walk = (a[:, 2] - a[:, 0]) / 1e3
body = np.where(a[:, 1] > 0, (a[:, 1] - a[:, 0]) / 1e3, walk)
done = (a[:, 3] - t0) / 1e3
sm = a[:, 4] & 0xFFFFFFFF
halo = a[:, 4] >> 32
print(st)
print("start us: min %.1f max %.1f" % (start.min(), start.max()))
print("walk us: min %.1f p10 %.1f p50 %.1f p90 %.1f max %.1f mean %.1f" % (walk.min(), *np.percentile(walk, [10, 50, 90]), walk.max(), walk.mean()))
print("body us: p10 %.1f p50 %.1f p90 %.1f max %.1f" % (*np.percentile(body, [10, 50, 90]), body.max()))
hw = walk - body
print("halo walk us: p50 %.1f p90 %.1f p99 %.1f max %.1f; per halo chunk us: mean %.2f" % (
    *np.percentile(hw, [50, 90, 99]), hw.max(), hw.sum() / max(1, halo.sum())))
if (a[:, 5] > 0).any():
    ok = (a[:, 5] > 0) & (a[:, 6] > 0)
    ib = (a[ok, 5] - a[ok, 0]) / 1e3
    tb = (a[ok, 6] - a[ok, 5]) / 1e3
    print("T-mode: from start to index built us p50 %.1f max %.1f; table us p50 %.1f max %.1f" % (
        np.percentile(ib, 50) if ib.size else 0, ib.max() if ib.size else 0, np.percentile(tb, 50) if tb.size else 0, tb.max() if tb.size else 0))
if st["fast_path"] == 2:  # T-mode phases: tm[2] published, tm[4] composed, tm[5] scanned, tm[1] verdict, tm[3] done
    rel = lambda v: (v - t0) / 1e3
    comp = a[a[:, 4] > 0, 4]
    ver = a[a[:, 1] > 0, 1]
    print("T-mode abs us: published p50 %.1f max %.1f; composed max %.1f (%d composers); scan done %.1f; verdict seen p50 %.1f max %.1f; written p50 %.1f max %.1f" % (
        np.percentile(rel(a[:, 2]), 50), rel(a[:, 2]).max(), rel(comp).max() if comp.size else -1, comp.size,
        rel(a[:, 5]).max(), np.percentile(rel(ver), 50) if ver.size else -1, rel(ver).max() if ver.size else -1,
        np.percentile(rel(a[:, 3]), 50), rel(a[:, 3]).max()))
    sys.exit(0)
print("walk end us (abs): p50 %.1f p90 %.1f max %.1f" % tuple(np.percentile(start + walk, [50, 90, 100])))
print("done us (abs): p50 %.1f max %.1f" % (np.percentile(done, 50), done.max()))
print("halo chunks: mean %.2f max %d" % (halo.mean(), halo.max()))
# per-SM: segments and summed walk
for s_ in np.argsort([-walk[sm == k].max() if (sm == k).any() else 0 for k in range(148)])[:5]:
    m = sm == s_
    print("sm", s_, "segs", m.sum(), "walk max %.1f mean %.1f" % (walk[m].max(), walk[m].mean()))
# correlation of walk time with halo length and with g
print("corr(walk, halo) %.2f corr(walk, g) %.2f" % (np.corrcoef(walk, halo)[0, 1], np.corrcoef(walk, np.arange(G))[0, 1]))
slow = np.argsort(-walk)[:10]
print("slowest segs", slow.tolist(), walk[slow].round(1).tolist(), "body", body[slow].round(1).tolist(), "halo", halo[slow].tolist(), "sm", sm[slow].tolist())
gs = int(np.argmax(start + walk))
we = start + walk
print("slowest walker g*=%d walk_end %.1f done %.1f" % (gs, we[gs], done[gs]))
late = np.argsort(-done)[:8]
print("latest done:", [(int(g), round(float(done[g]), 1), round(float(we[g]), 1)) for g in late])
print("done - max(walk_end of predecessors..self): p50 %.2f p99 %.2f max %.2f" % tuple(
    np.percentile(done - np.maximum.accumulate(we), [50, 99, 100])))
