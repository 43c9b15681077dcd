"""Walker event counts for one call (CDC_COUNTERS build; diagnostic)."""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2508_05797_b200 as cdc
from paper_2508_05797_b200._lib import lib
n = 256 << 20
algo = os.environ.get("ALGO", "ae_max")
avg = int(os.environ.get("AVG", "4096"))
d = synth.zipf_bytes(n, 1.1, 1) if os.environ.get("DATA", "zipf") == "zipf" else synth.uniform(n, 0)
t = torch.from_numpy(d).cuda()
p = cdc.params(algo, avg_size=avg)
ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
c = torch.zeros(1, dtype=torch.int64, device="cuda")
cnt = (ctypes.c_ulonglong * 16)()
cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
lib.cdc_debug_counters(cnt)
cdc.chunk_async(t, p, b, c, ws)
torch.cuda.synchronize()
lib.cdc_debug_counters(cnt)
names = ["stages", "ae_pending", "ae_find_calls", "ae_records", "-", "ae_saturated_iters", "boundaries",
         "find_block_calls", "pair_iters", "head_partial", "tail_partial", "ram_window_calls", "ram_find_calls"]
nb = int(c.item())
print(algo, "chunks", nb)
for i, k in enumerate(names):
    if k != "-":
        print("%-20s %10d  per chunk %.2f" % (k, cnt[i], cnt[i] / nb))
