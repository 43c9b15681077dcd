"""configs[0] (16 MiB uniform, RAM 8 KiB) under the current CDC_* environment: time
and element-wise check against the oracle (diagnostic for path selection)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
import paper_2508_05797_b200 as cdc

n = int(os.environ.get("N", 16 << 20))
algo = os.environ.get("ALGO", "ram")
avg = int(os.environ.get("AVG", "8192"))
kind = os.environ.get("DATA", "uniform")
d = synth.uniform(n, 0) if kind == "uniform" else synth.versioned(n, 0, seed=2)[0]
t = torch.from_numpy(d).cuda()
p = cdc.params(algo, avg_size=avg, seg_bytes=int(os.environ.get("SEG", "0")))
ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
for _ in range(3):
    cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
reps = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    cdc.chunk_async(t, p, b, c, ws)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
# graph of one call
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    cdc.chunk_async(t, p, b, c, ws)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
e0.record()
for _ in range(reps):
    g.replay()
e1.record()
torch.cuda.synchronize()
gms = e0.elapsed_time(e1) / reps
k = int(c.item())
got = b[:k].cpu().numpy().astype(np.uint64)
exp = oracle.chunk(algo, d, p.window, p.max_size)
ok = got.size == exp.size and bool((got == exp).all())
st = cdc.stats(p, ws, 1, n, n)
env = {k: v for k, v in os.environ.items() if k.startswith("CDC_")}
print(f"{kind} {n>>20}MiB {algo} {avg} env={env} direct {ms*1e3:.1f} us graph {gms*1e3:.1f} us chunks {k} parity {ok} "
      f"{ {k: st[k] for k in ('segments', 'fast_path', 'synced', 'unsynced', 'halo_chunks') if k in st} }", flush=True)
