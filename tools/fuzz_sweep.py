"""Larger random parity sweeps than tests/test_gpu_fuzz.py runs by default:
FUZZ_SEEDS seeds of the batch cases and FUZZ_LARGE large streams (diagnostic;
prints only failures and a count)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_2508_05797_b200 as cdc
import test_gpu_fuzz as F

ok = bad = 0
for s in range(int(os.environ.get("FUZZ_SEEDS", "5"))):
    for c in F._batch_cases(16, 1000 + s):
        try:
            F.test_fuzz_batch(cdc, c); ok += 1
        except AssertionError as e:
            bad += 1; print("batch FAIL seed", 1000 + s, c[:6], len(c[6]), flush=True)
for i in range(int(os.environ.get("FUZZ_LARGE", "0"))):
    rng = np.random.default_rng(50000 + i)
    algo = F.ALGOS[i % 3]
    kind = ["zipf", "uniform", "runs", "satedge", "small"][rng.integers(0, 5)]
    n = int(rng.integers(1 << 20, 96 << 20))
    w = int(rng.choice([64, 255, 1000, 3840, 5000, 8000]))
    mx = w + 1 + int(rng.choice([0, 3, w, 3 * w, 7 * w]))
    d = F._data(kind, n, 60000 + i)
    p = cdc.params(algo, window=w, max_size=mx)
    import oracle, torch
    exp = oracle.chunk(algo, d, w, mx)
    got = cdc.chunk(torch.from_numpy(d).cuda(), p).cpu().numpy().astype(np.uint64)
    if got.size == exp.size and (got == exp).all():
        ok += 1
    else:
        bad += 1; print("large FAIL", i, algo, kind, n, w, mx, flush=True)
print("ok", ok, "bad", bad)
