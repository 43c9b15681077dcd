"""Throughput of the single-GPU path on the shapes of every BASELINE config (diagnostic)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2508_05797_b200 as cdc


def run(name, data_np, algo, avg, reps=10, seg=0):
    t = torch.from_numpy(data_np).cuda()
    n = t.numel()
    p = cdc.params(algo, avg_size=avg, seg_bytes=seg)
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        cdc.chunk_async(t, p, b, c, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        cdc.chunk_async(t, p, b, c, ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    cdc.profile_enable(True)
    cdc.chunk_async(t, p, b, c, ws)
    torch.cuda.synchronize()
    cdc.profile_enable(False)
    pr = cdc.profile_collect()
    st = cdc.stats(p, ws, 1, n, n)
    st["k_ms"] = {k: round(v[0], 3) for k, v in pr.items() if k != "calls" and v[1]}
    print("%-28s %-6s %5d  %8.3f ms  %8.1f GB/s  chunks %d  %s" % (name, algo, avg, ms, n / ms / 1e6, int(c.item()),
          {k: st[k] for k in ("segments", "fast_path", "synced", "unsynced", "skipped_or_end", "halo_chunks", "k_ms")}),
          flush=True)


sel = os.environ.get("ONLY", "")
if not sel or "c0" in sel:
    run("c0 uniform 16MiB", synth.uniform(16 << 20, 0), "ram", 8192)
if not sel or "c1" in sel:
    run("c1 zipf 256MiB", synth.zipf_bytes(256 << 20, 1.1, 1), "ae_max", 4096)
if not sel or "u256" in sel:
    u = synth.uniform(256 << 20, 0)
    for algo in ("ram", "ae_max"):
        for avg in (4096, 8192, 16384):
            run("uniform 256MiB", u, algo, avg, reps=3)
if not sel or "c4" in sel:
    run("c4-shape alternating 1GiB", synth.alternating(1 << 30, region=256 << 20, seed=5), "ram", 8192, reps=3)


def run_batch(name, data_np, offs, algo, avg, reps=5):
    """cdc_chunk_batch on preallocated device buffers (the host-side setup of
    api.chunk_batch is outside the timed region)."""
    t = torch.from_numpy(data_np).cuda()
    p = cdc.params(algo, avg_size=avg, seg_bytes=int(os.environ.get("SEG", "0")))
    sizes = np.diff(offs)
    total, max_len = int(sizes.sum()), int(sizes.max())
    od = torch.from_numpy(np.asarray(offs, dtype=np.int64)).cuda()
    cap = total // (p.window + 1) + len(offs)
    b = torch.empty(cap, dtype=torch.int64, device="cuda")
    bo = torch.zeros(len(offs), dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(cdc.workspace_size(p, len(offs) - 1, total, max_len), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        cdc.chunk_batch_async(t, od, total, max_len, p, b, bo, c, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        cdc.chunk_batch_async(t, od, total, max_len, p, b, bo, c, ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    cdc.profile_enable(True)
    cdc.chunk_batch_async(t, od, total, max_len, p, b, bo, c, ws)
    torch.cuda.synchronize()
    cdc.profile_enable(False)
    pr = cdc.profile_collect()
    st = cdc.stats(p, ws, len(offs) - 1, total, max_len)
    st["k_ms"] = {k: round(v[0], 3) for k, v in pr.items() if k != "calls" and v[1]}
    print("%-28s %-6s %5d  %8.3f ms  %8.1f GB/s  files %d chunks %d  %s" % (
        name, algo, avg, ms, total / ms / 1e6, len(offs) - 1, int(c.item()),
        {k: st[k] for k in ("segments", "fast_path", "synced", "skipped_or_end", "halo_chunks", "k_ms")}), flush=True)


if "c2" in sel:  # configs[2]: the 1 GiB base and its last snapshot, AE and RAM at 4/8/16 KiB
    snaps = synth.versioned(1 << 30, 9, seed=2)
    for name, d in (("c2 versioned base 1GiB", snaps[0]), ("c2 versioned snap9 1GiB", snaps[-1])):
        for algo in ("ae_max", "ram"):
            for avg in (4096, 8192, 16384):
                run(name, d, algo, avg, reps=3)
    del snaps
if "u1g" in sel:  # a whole 1 GiB uniform stream (453 KB segments: transfer tables near their capacity)
    u = synth.uniform(1 << 30, 4)
    for algo in ("ram", "ae_max"):
        run("uniform 1GiB", u, algo, 8192, reps=3)
    del u
if "c4full" in sel:  # configs[4], one GPU's 8 GiB share of the 64 GiB stream
    d = synth.alternating(8 << 30, region=256 << 20, seed=5)
    run("c4 alternating 8GiB (1/8)", d, "ram", 8192, reps=3)
    run("c4 alternating 8GiB (1/8)", d, "ae_max", 8192, reps=3)
    del d
if "c4big" in sel:
    d = synth.alternating(4 << 30, region=256 << 20, seed=5)
    run("c4-shape alternating 4GiB", d, "ram", 8192, reps=3)
    run("c4-shape alternating 4GiB", d, "ae_max", 8192, reps=3)
if "c3" in sel:  # configs[3], one GPU's share at 8 GPUs
    data, offs = synth.many_files(12500, seed=3)
    run_batch("c3 many files (12.5k)", data, offs, "ram", 8192)
if "v128" in sel:  # versioned bytes at 24-128 MiB: transfer tables attempted and refused (CDC_TMODE=0 to compare)
    for mib in (24, 128):
        v = synth.versioned(mib << 20, 1, seed=2)[-1]
        for algo in ("ram", "ae_max"):
            for avg in (8192, 16384):
                run("versioned %dMiB" % mib, v, algo, avg, reps=5)
if "small" in sel:  # 16 MiB streams one segment per SM: saturated (tables) and not (refused after the sample)
    run("zipf 16MiB", synth.zipf_bytes(16 << 20, 1.1, 1), "ae_max", 8192)
    run("zipf 16MiB", synth.zipf_bytes(16 << 20, 1.1, 1), "ram", 8192)
    run("versioned 16MiB", synth.versioned(16 << 20, 0, seed=2)[0], "ram", 8192)
