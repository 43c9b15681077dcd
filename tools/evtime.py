"""Per-event-type cycle accounting of the walkers for one configs[1] call (CDC_EVTIME build; diagnostic)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2508_05797_b200 as cdc
from paper_2508_05797_b200._lib import lib
n = 256 << 20
d = synth.zipf_bytes(n, 1.1, 1)
t = torch.from_numpy(d).cuda()
p = cdc.params("ae_max", avg_size=4096)
ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
ev = (ctypes.c_ulonglong * 16)()
cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
lib.cdc_debug_evtime(ev)
cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
lib.cdc_debug_evtime(ev)
names = ["stage transition (wait+setup)", "find_block", "record", "boundary event", "pending",
         "iter: saturated (whole iteration)", "iter: no-hit find (whole iteration, incl. find)",
         "  of which halo stage transitions", "walk total"]
tot = ev[8]
chunks = int(c.item())
for i, k in enumerate(names):
    if k:
        print("%-32s %14d cycles  %5.1f%%  per chunk %8.0f" % (k, ev[i], 100.0 * ev[i] / tot, ev[i] / chunks))
print("other (loop control, sat jumps, etc.) %5.1f%%" % (100.0 * (tot - sum(ev[i] for i in range(7))) / tot))
hs, hc = ev[9], ev[10]
if hs:
    print("halo phase: %d stages, %d cycles (%.1f%% of walk); per halo stage %.0f cycles, of which transition %.0f"
          % (hs, hc, 100.0 * hc / tot, hc / hs, ev[7] / hs))
