"""A few cdc_chunk calls on a uniform 256 MiB stream through the transfer
tables (for ncu: `ncu -k regex:k_speculate -s 2 -c 1 python tools/tmode_run.py`)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2508_05797_b200 as cdc

algo = os.environ.get("ALGO", "ram")
avg = int(os.environ.get("AVG", "8192"))
n = int(os.environ.get("N", 256 << 20))
t = torch.from_numpy(synth.uniform(n, 0)).cuda()
p = cdc.params(algo, avg_size=avg)
ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(4):
    cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
print("chunks", int(c.item()), cdc.stats(p, ws, 1, n, n)["fast_path"])
