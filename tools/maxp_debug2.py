"""MAXP stage probe: the scan+gather list q (workspace offset 0) against numpy/scipy local maxima (diagnostic)."""
import os, sys
import numpy as np
import torch
from scipy.ndimage import maximum_filter1d
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2508_05797_b200 as cdc

n = 256 << 20
d = synth.uniform(n, 1)
h = 447
di = d.astype(np.int16)
# left window max of t: max d[t-h .. t-1]; right: max d[t+1 .. t+h]
mf = maximum_filter1d(di, size=h, origin=(h - 1) // 2 - (h - 1) + 0, mode="constant", cval=-1)
# compute window max W[i] = max d[i : i+h] directly with a cumulative trick for exactness
W = maximum_filter1d(di, size=h, mode="constant", cval=-1, origin=-(h // 2))  # W[i] = max d[i .. i+h-1]
t = np.arange(h, n - h)
ok = (di[t] > W[t - h]) & (di[t] > W[t + 1])
Q = t[ok]
print("expected maxima", Q.size, flush=True)
p = cdc.params("maxp", avg_size=8192)
tt = torch.from_numpy(d).cuda()
cap = cdc.max_boundaries(p, n)
b = torch.empty(cap, dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
for rep in range(4):
    cdc.chunk_async(tt, p, b, c, ws)
    torch.cuda.synchronize()
    q = ws[:Q.size * 8].view(torch.int64).cpu().numpy()
    bad = np.nonzero(q != Q)[0]
    print(rep, "q mismatches", bad.size, "first", (int(bad[0]), int(Q[bad[0]]), int(q[bad[0]])) if bad.size else None, flush=True)
    if bad.size:
        i = bad[0]
        print("   expected around", Q[i-2:i+3].tolist(), "got", q[i-2:i+3].tolist(), "tile", Q[i] // 32768, Q[i] % 32768)
