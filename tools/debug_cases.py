"""Run one chunking case in a fresh process (a device trap kills the context).

usage: python tools/debug_cases.py            -> runs every case in a subprocess
       python tools/debug_cases.py CASE       -> runs one case
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {
    "chain_ram": ("chain", "ram", 0),
    "chain_ae": ("chain", "ae_max", 0),
    "one_seg_ram": ("chunk", "ram", 4 << 20),
    "one_seg_ae": ("chunk", "ae_max", 4 << 20),
    "small_seg_ram": ("chunk", "ram", 16384),
    "small_seg_ae": ("chunk", "ae_max", 16384),
    "seg4k_halo8k_ram": ("chunk", "ram", 4096, 8192),
    "seg4k_halo8k_ae": ("chunk", "ae_max", 4096, 8192),
    "seg64k_halo4k_ram": ("chunk", "ram", 65536, 4096),
    "seg64k_halo4k_ae": ("chunk", "ae_max", 65536, 4096),
    "chains_ram": ("chains", "ram", 0),
    "chains_ae": ("chains", "ae_max", 0),
}


def run(name):
    import numpy as np
    import torch
    import oracle
    import synth
    import paper_2508_05797_b200 as cdc
    kind, algo, seg, *rest = CASES[name]
    halo = rest[0] if rest else 0
    n = 3 * (1 << 20) + 777
    d = synth.uniform(n, 7)
    w, mx = 600, 4000
    t = torch.from_numpy(d).cuda()
    p = cdc.params(algo, window=w, max_size=mx, seg_bytes=seg, halo_bytes=halo)
    if kind == "chains":
        rng = np.random.default_rng(1)
        for st in rng.integers(0, n, 40).tolist() + [n - 1, n - 600, n - 601, n - 602, 17, 4095, 4096]:
            got = cdc.chain(t, p, st, n).cpu().numpy().astype(np.uint64)
            exp = oracle.chain_from(algo, d, st, n, w, mx)
            if not (got.size == exp.size and (got == exp).all()):
                print("chain mismatch from", st, got[:5], exp[:5], got.size, exp.size, flush=True)
                return
        print(name, "OK", flush=True)
        return
    if kind == "chain":
        got = cdc.chain(t, p, 0, n).cpu().numpy().astype(np.uint64)
        exp = oracle.chain_from(algo, d, 0, n, w, mx)
    else:
        got = cdc.chunk(t, p).cpu().numpy().astype(np.uint64)
        exp = oracle.chunk(algo, d, w, mx)
    ok = got.size == exp.size and (got == exp).all()
    print(name, "OK" if ok else f"MISMATCH got {got.size} exp {exp.size}", flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(sys.argv[1])
    else:
        import time
        sel = os.environ.get("CASES")
        for c in (sel.split(",") if sel else CASES):
            t0 = time.time()
            r = subprocess.run([sys.executable, __file__, c], capture_output=True, text=True, timeout=120,
                               env=dict(os.environ, CDC_SYNC_DEBUG='1'))
            print(c, "rc", r.returncode, "%.1fs" % (time.time() - t0), r.stdout.strip()[-200:], r.stderr.strip()[-300:], flush=True)
