"""One K-phase call with its node records dumped (diagnostic)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
import paper_2508_05797_b200 as cdc

n = int(os.environ.get("N", (24 << 20) + 4321))
w = int(os.environ.get("W", 4096))
algo = os.environ.get("ALGO", "ram")
d = synth.uniform(n, 31 + w)
p = cdc.params(algo, window=w, max_size=4 * (w + 256), seg_bytes=512 << 10)
ws = torch.zeros(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
t = torch.from_numpy(d).cuda()
b = torch.zeros(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
print("count", int(c.item()), "launches", cdc.last_launch_count())
print("stats", cdc.stats(p, ws, 1, n, n))
exp = oracle.chunk(algo, d, w, p.max_size)
got = b[: int(c.item())].cpu().numpy().astype(np.uint64)
print("oracle", exp.size, "match", got.size == exp.size and bool((got == exp).all()))
