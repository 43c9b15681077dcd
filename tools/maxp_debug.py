"""MAXP determinism / parity probe on the 256 MiB uniform stream (diagnostic)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
import paper_2508_05797_b200 as cdc

d = synth.uniform(256 << 20, 1)
p = cdc.params("maxp", avg_size=8192)
exp = oracle.chunk("maxp", d, p.window, p.max_size)
t = torch.from_numpy(d).cuda()
for rep in range(8):
    got = cdc.chunk(t, p).cpu().numpy().astype(np.uint64)
    n = min(got.size, exp.size)
    bad = np.nonzero(got[:n] != exp[:n])[0]
    print(rep, got.size, exp.size, "first mismatch", (int(bad[0]), int(exp[bad[0]]), int(got[bad[0]])) if bad.size else None,
          "mismatches", bad.size, flush=True)
