"""configs[0] (16 MiB uniform, RAM 8 KiB) through the dense-index mode: direct launches and a CUDA
graph of 9 calls over 9 device copies (L2 never warm) (diagnostic; not a measurement)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2508_05797_b200 as cdc

n = int(os.environ.get("N", 16 << 20))
algo = os.environ.get("ALGO", "ram")
avg = int(os.environ.get("AVG", "8192"))
NC = max(2, (160 << 20) // n)
d = synth.uniform(n, 0)
bufs = [torch.from_numpy(d).cuda() for _ in range(NC)]
p = cdc.params(algo, avg_size=avg)
ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
for i in range(NC):
    cdc.chunk_async(bufs[i], p, b, c, ws)
torch.cuda.synchronize()
print(cdc.stats(p, ws, 1, n, n), "launches", cdc.last_launch_count())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for r in range(5):
    for i in range(NC):
        cdc.chunk_async(bufs[i], p, b, c, ws)
e1.record()
torch.cuda.synchronize()
print("direct: %.4f ms per call" % (e0.elapsed_time(e1) / (5 * NC)))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    cdc.chunk_async(bufs[0], p, b, c, ws)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(NC):
        cdc.chunk_async(bufs[i], p, b, c, ws)
g.replay()
torch.cuda.synchronize()
e0.record()
for r in range(10):
    g.replay()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / (10 * NC)
print("graph: %.4f ms per call  %.1f GB/s" % (ms, n / ms / 1e6))
if os.environ.get("STAMPS", "1") == "1":
    from paper_2508_05797_b200._lib import lib
    G = cdc.stats(p, ws, 1, n, n)["segments"]
    tm = torch.zeros(8 + 7 * (G + 1), dtype=torch.int64, device="cuda")
    tm[[0, 2, 3, 5, 6]] = -1
    lib.cdc_debug_timing(tm.data_ptr())
    cdc.chunk_async(bufs[1], p, b, c, ws)
    torch.cuda.synchronize()
    lib.cdc_debug_timing(None)
    a = tm[8:].cpu().numpy().reshape(G + 1, 7).astype(np.float64)
    t0 = a[:G, 0].min()
    for k, name in enumerate(("start", "index built", "checked+buckets", "table done", "(unused)", "w0 first data", "w0 blocks done")):
        v = (a[:G, k] - t0) / 1e3
        print("%-16s us: min %6.1f p50 %6.1f max %6.1f" % (name, v.min(), np.median(v), v.max()))
    print("resolve: begin %.1f  tables loaded %.1f  done %.1f us; pass 1 done %.1f  pass 2 done %.1f" % tuple((a[G, :5] - t0) / 1e3))
