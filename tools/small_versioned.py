"""Small versioned streams (configs[2]'s recipe at 16-128 MiB): time per call (diagnostic)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2508_05797_b200 as cdc

KIND = os.environ.get("KIND", "versioned")
for mib in [int(x) for x in os.environ.get("MIB", "16 64 128").split()]:
    n = mib << 20
    d = synth.versioned(n, 0, seed=2)[0] if KIND == "versioned" else synth.uniform(n, 4)
    t = torch.from_numpy(d).cuda()
    for algo in ("ram", "ae_max"):
        for avg in (8192, 16384):
            p = cdc.params(algo, avg_size=avg)
            ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
            b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
            c = torch.zeros(1, dtype=torch.int64, device="cuda")
            for _ in range(2):
                cdc.chunk_async(t, p, b, c, ws)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                cdc.chunk_async(t, p, b, c, ws)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            st = cdc.stats(p, ws, 1, n, n)
            print(KIND[:9] + " %4d MiB %-6s %5d  %7.3f ms  %7.1f GB/s  path %d segs %d" % (
                mib, algo, avg, ms, n / ms / 1e6, st["fast_path"], st["segments"]), flush=True)
