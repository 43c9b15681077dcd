"""Random parity sweep aimed at the dense-index mode and what follows its gate (K-phase, transfer
tables, speculation): default-segment single streams of 1-70 MiB with windows of 4-26 KiB, uniform
bytes with random holes (stretches without the saturating byte), versioned and alternating streams
(diagnostic; prints failures and a count; every comparison is against the oracle)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import oracle
import synth
import paper_2508_05797_b200 as cdc

N = int(os.environ.get("FUZZ_DENSE", "200"))
BASE = int(os.environ.get("FUZZ_BASE", "90000"))
ok = bad = 0
paths = {}
for i in range(N):
    rng = np.random.default_rng(BASE + i)
    algo = ("ram", "ae_max", "ae_min")[i % 3]
    sat = 0 if algo == "ae_min" else 255
    n = int(rng.integers(1 << 20, 70 << 20)) if rng.random() < 0.7 else int(rng.integers(1 << 20, 4 << 20))
    w = int(rng.choice([4096, 5000, 7936, 12000, 16128, 20000, 24576, 26000]))
    mx = int(rng.choice([2 * w + 1, 2 * w + 2, 3 * w, 4 * w + 1024, 8 * w]))
    kind = rng.choice(["uniform", "holes", "holes", "versioned", "alternating", "edge"])
    if kind == "versioned":
        d = synth.versioned(n, 0, seed=int(rng.integers(1, 1000)))[0].copy()
    elif kind == "alternating":
        d = synth.alternating(n, region=int(rng.choice([1 << 20, 4 << 20])), seed=int(rng.integers(1, 1000))).copy()
    else:
        d = synth.uniform(n, int(rng.integers(1, 100000))).copy()
    if kind == "holes":
        for _ in range(int(rng.integers(1, 4))):
            ln = int(rng.choice([w - 1, w, w + 1, 2 * w, 100 << 10]))
            at = int(rng.integers(0, max(1, n - ln)))
            seg = d[at:at + ln]
            seg[seg == sat] = 9
    if kind == "edge":  # exact gaps of w / w + 1 at the start, a segment edge and the end
        g = w + int(rng.integers(0, 2))
        for at in (0, 3 * 65536 - g // 2, n - g - 1):
            at = max(0, min(at, n - g - 1))
            seg = d[at + 1:at + g]
            seg[seg == sat] = 9
            d[at] = sat
            d[at + g] = sat
    off = int(rng.choice([0, 0, 1, 7, 16]))
    t = torch.from_numpy(d).cuda()[off:]
    dd = d[off:]
    p = cdc.params(algo, window=w, max_size=mx)
    m = dd.size
    ws = torch.empty(cdc.workspace_size(p, 1, m, m), dtype=torch.uint8, device="cuda")
    b = torch.full((cdc.max_boundaries(p, m),), -1, dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    cdc.chunk_async(t, p, b, c, ws)
    got = b[:int(c.item())].cpu().numpy().astype(np.uint64)
    exp = oracle.chunk(algo, dd, w, mx)
    fp = cdc.stats(p, ws, 1, m, m)["fast_path"]
    paths[fp] = paths.get(fp, 0) + 1
    if got.size == exp.size and (got == exp).all():
        ok += 1
    else:
        bad += 1
        print("FAIL", i, algo, kind, n, w, mx, off, "path", fp, flush=True)
print("ok", ok, "bad", bad, "paths (0/1 ordinary, 2 tables, 3 K-phase, 4 dense):", dict(sorted(paths.items())))
