"""Re-run fuzz cases of tests/test_gpu_fuzz.py by index and print the first
difference from the oracle (diagnostic)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import oracle
import paper_2508_05797_b200 as cdc
import test_gpu_fuzz as F

cases = F._cases(int(os.environ.get("FUZZ_N", "48")), int(os.environ.get("FUZZ_SEED", "20261020")))
idx = [int(a) for a in sys.argv[1:]] or range(len(cases))
for i in idx:
    c = cases[i]
    _, algo, kind, w, mx, n, seg, halo = c
    d = F._data(kind, n, 100 + i)
    p = cdc.params(algo, window=w, max_size=mx, seg_bytes=seg, halo_bytes=halo)
    exp = oracle.chunk(algo, d, w, mx)
    cap = cdc.max_boundaries(p, n)
    bounds = torch.zeros(cap + 64, dtype=torch.int64, device="cuda")
    count = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    dd = torch.from_numpy(d).cuda()
    cdc.chunk_async(dd, p, bounds, count, ws)
    m = int(count.item())
    got = bounds[:min(m, cap + 64)].cpu().numpy().astype(np.uint64)
    st = cdc.stats(p, ws, 1, n, n)
    ok = got.size == exp.size and (got == exp).all()
    msg = f"case {i} {c} cap={cap} gpu={m} oracle={exp.size} ok={ok} stats={st}"
    if not ok:
        k = int(np.argmax(got[:min(got.size, exp.size)] != exp[:min(got.size, exp.size)])) if min(got.size, exp.size) else 0
        msg += f" first diff at {k}: gpu {got[max(0,k-2):k+3].tolist()} oracle {exp[max(0,k-2):k+3].tolist()}"
    print(msg, flush=True)
