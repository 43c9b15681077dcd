"""MAXP call timing on device-resident inputs (diagnostic; bench.py's maxp key is the measurement)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2508_05797_b200 as cdc

avg = int(os.environ.get("AVG", "8192"))
for name, n, gen in (("uniform 256MiB", 256 << 20, lambda n: synth.uniform(n, 1)),
                     ("zipf 256MiB", 256 << 20, lambda n: synth.zipf_bytes(n, 1.1, 1)),
                     ("uniform 1GiB", 1 << 30, lambda n: synth.uniform(n, 2)),
                     ("versioned 1GiB", 1 << 30, lambda n: synth.versioned(n, 0, seed=2)[0])):
    d = gen(n)
    t = torch.from_numpy(d).cuda()
    p = cdc.params("maxp", avg_size=avg)
    cap = cdc.max_boundaries(p, n)
    b = torch.empty(cap, dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        cdc.chunk_async(t, p, b, c, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        cdc.chunk_async(t, p, b, c, ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print("%-16s h=%d  %.3f ms  %.1f GB/s  chunks %d" % (name, p.window, ms, n / ms / 1e6, int(c.item())), flush=True)
    del t, b, ws
