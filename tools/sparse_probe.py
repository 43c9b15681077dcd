"""Single-warp chain walk (cdc_chain, k_chain: one warp) timing per chunk, and
the sparse walker's event counts (CDC_COUNTERS build via CDC_LIB): where a
lone walker's time goes (diagnostic)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
import paper_2508_05797_b200 as cdc  # noqa: E402
from paper_2508_05797_b200._lib import lib  # noqa: E402

N = 16 << 20      # chain length walked per timing
TOT = 768 << 20   # buffer: every timed walk reads a slice no earlier walk touched (not in L2)
cases = [("uniform", synth.uniform(TOT, 0)), ("zipf2003", synth.zipf_bytes(TOT, 1.1, 2003))]
counters = os.environ.get("COUNTERS", "0") == "1"
sptime = os.environ.get("SPTIME", "0") == "1"
for name, d in cases:
    tt = torch.from_numpy(d).cuda()
    sl = 0
    for algo, avg in (("ram", 8192), ("ae_max", 8192), ("ae_max", 4096)):
        p = cdc.params(algo, avg_size=avg)
        cdc.chain(tt[sl * N:(sl + 1) * N], p, 0, N)
        torch.cuda.synchronize()
        t = tt[(sl + 1) * N:(sl + 2) * N]
        sl += 2
        if counters:
            cnt = (ctypes.c_ulonglong * 16)()
            lib.cdc_debug_counters(cnt)
        if sptime:
            ev = (ctypes.c_ulonglong * 16)()
            lib.cdc_debug_evtime(ev)
        t0 = time.perf_counter()
        r = cdc.chain(t, p, 0, N)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        n = r.numel()
        line = "%-9s %-6s %5d chunks %6d  %7.3f ms  %6.3f us/chunk  %6.2f GB/s" % (
            name, algo, avg, n, dt * 1e3, dt * 1e6 / max(n, 1), N / dt / 1e9)
        if counters:
            lib.cdc_debug_counters(cnt)
            line += "  spec-miss %.3f cont %.3f probe %.3f stages %.2f /chunk" % (
                cnt[13] / n, cnt[14] / n, cnt[15] / n, cnt[0] / n)
        if sptime:
            lib.cdc_debug_evtime(ev)
            line += "  cycles/chunk: window %.0f wait %.0f scan %.0f emit %.0f total %.0f" % tuple(
                ev[11 + i] / n for i in range(5))
        print(line, flush=True)
