#!/usr/bin/env python
"""bench.py -- chunking throughput of the B200 CDC hot path (driver contract).

Headline workload (N=1): BASELINE.json configs[3] at full size, the largest
configuration that fits one GPU -- 100,000 files with lognormal sizes (median
64 KiB, sigma 1.5, capped at 16 MiB: 18.67 GiB; BASELINE.json's "~8 GiB" is not
what its stated distribution gives), 70 % uniform / 30 % Zipf(1.1) content,
RAM at an 8 KiB average.  One step = one cdc_chunk_batch call over all the
resident files: the batch segment table (k_seg_prefix), the list reset
(k_reset), the speculative walkers (k_speculate: Extreme Byte Search, Range
Scan and the RAM rule, DESIGN.md §0 rows a1-a3, a5) and the chain resolver and
boundary write (k_fixup, row a4).

With N ranks (torchrun) the same 100,000 files are split N ways by
shard.file_range (contiguous, byte-balanced file ranges; "files shard
directly", north_star (4)): each rank chunks its share with one
cdc_chunk_batch call and no data-path collective ("scaling": "strong").

Secondary keys in the same JSON line:
  configs0        configs[0] (RAM 8 KiB, one 16 MiB uniform stream) on every rank:
                  the dense-index mode;
  configs1        configs[1] (AE-Max 4 KiB, one 256 MiB Zipf stream) on every
                  rank, with its own roofline (the round-1 headline);
  configs4_sharded  configs[4]: the 64 GiB alternating stream split by byte
                  range with a halo over the N ranks (shard.chunk_sharded: NCCL
                  all_gather of segment-edge chain states), RAM and AE-Max at
                  8 KiB, timed through the public API;
  paper_cpu_vector  the paper's own CPU-vector numbers, as context only.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--impl reference times the CPU oracle (oracle/, plain C) on the host cores on
the same configs[3] workload, one ~1 GiB range of files per step; under
torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "chunking GB/s of input (1/2/4/8 B200) and % of HBM roofline; boundaries == oracle"
NFILES, FSEED, C3_ALGO, C3_AVG = 100_000, 3, "ram", 8192
WORKLOAD = ("configs[3]: 100,000 files, lognormal sizes (median 64 KiB, sigma 1.5, capped at 16 MiB; 18.67 GiB), "
            "70% uniform / 30% Zipf(1.1) bytes, RAM avg 8 KiB, one cdc_chunk_batch call per rank")
C1_ALGO, C1_AVG, C1_STREAM = "ae_max", 4096, 256 << 20
C4_LEN = 64 << 30
REF_SAMPLE = 1 << 30          # --impl reference: bytes of files per step
CPU_SECONDS = 12.0           # cpu_baseline: whole passes over the batch until this much wall time

# PAPER.md's own numbers (single CPU core, its datasets), quoted as context only
PAPER_CPU = {
    "note": "PAPER.md single-core numbers on its real datasets and CPUs; context, not a target",
    "VAE-Max/VAE-Min/VMAXP/VRAM, AVX-512, 8 KB chunks (PAPER.md l.661-665, sec. 6 throughput)": "6.5-29.9 GB/s",
    "VRAM-EBS (Extreme Byte Search only) on DEB (l.737)": "18.5 GB/s",
    "RAM, NEON-128, ARM v8 Atlas (l.797)": "2.91 GB/s",
    "RAM, VSX-128, IBM Power 8 (l.803)": "8.54 GB/s",
    "unaccelerated AE-Max/AE-Min/MAXP/RAM (l.663)": "1.5-1.7 GB/s",
    "machines (l.430-437)": "Intel Emerald Rapids Xeon Gold 5512U, Skylake Xeon Silver 4114, AMD EPYC 7302P, "
                            "ARM v8 Atlas, IBM Power 8 (CloudLab)",
}


def load_traffic(name):
    """DRAM traffic per k_speculate launch from a committed ncu --set full capture, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            t = json.load(f)
        return float(t["traffic_bytes"]) / 1e9, f"dram__bytes_read.sum + dram__bytes_write.sum per launch (GB), " \
            f"profiles/{name}"
    except Exception:
        return None, None


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.02):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def c3_window():
    return C3_AVG - 256, 4 * C3_AVG  # cdc_params_default's window / cap (reading R4, R5)


def oracle_files(data, offs, files, threads):
    """The oracle as it stands (oracle.chunk per file), files spread over host threads."""
    import oracle
    w, mx = c3_window()

    def one(f):
        return oracle.chunk(C3_ALGO, data[offs[f]:offs[f + 1]], w, mx).size

    with ThreadPoolExecutor(threads) as ex:
        return sum(ex.map(one, files, chunksize=64))


def run_reference(args, world, rank):
    """CPU oracle arm (rank 0 only): the configs[3] workload on the box's host cores,
    each step one contiguous ~1 GiB range of files (rotating through the batch)."""
    if rank != 0:
        return 0
    import synth
    offs = synth.many_files_offsets(NFILES, FSEED)
    nsteps = args.warmup + args.steps
    # contiguous file ranges of ~REF_SAMPLE bytes, as many as the run needs
    starts = [0]
    while len(starts) <= nsteps and starts[-1] < NFILES:
        starts.append(int(np.searchsorted(offs, offs[starts[-1]] + REF_SAMPLE)))
    ranges = [(a, min(b, NFILES)) for a, b in zip(starts, starts[1:]) if b > a]
    f_lo, f_hi = ranges[0][0], ranges[-1][1]
    data, loc = synth.many_files(NFILES, FSEED, files=(f_lo, f_hi))
    threads = os.cpu_count() or 1
    w, mx = c3_window()

    def step(i):
        a, b = ranges[i % len(ranges)]
        oracle_files(data, loc, range(a - f_lo, b - f_lo), threads)
        return int(offs[b] - offs[a])

    for i in range(args.warmup):
        step(i)
    nbytes = 0
    t0 = time.perf_counter()
    for i in range(args.steps):
        nbytes += step(args.warmup + i)
    dt = time.perf_counter() - t0
    gbs = nbytes / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": WORKLOAD, "algo": C3_ALGO, "avg_size": C3_AVG, "window": w, "max_size": mx,
                   "parallelism": "cpu oracle, rank 0 only"},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
                         "sample": f"per step one contiguous range of ~{REF_SAMPLE >> 30} GiB of the 100,000 files, "
                                   f"oracle.chunk per file on {threads} threads"},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(data, offs):
    """The oracle (oracle.chunk per file, as it stands) on all host cores: whole passes over
    this rank's files, repeated until about CPU_SECONDS of wall time have gone by."""
    threads = os.cpu_count() or 1
    nf = offs.size - 1
    nb = int(offs[nf] - offs[0])
    passes, t0 = 0, time.perf_counter()
    while True:
        oracle_files(data, offs, range(nf), threads)
        passes += 1
        dt = time.perf_counter() - t0
        if dt >= CPU_SECONDS or passes >= 64:
            break
    return {"value": round(nb * passes / dt / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": f"{passes} pass(es) over all {nf} files ({nb / 2**30:.2f} GiB) of the configs[3] batch, "
                      f"oracle.chunk per file (C, gcc -O2) on {threads} threads ({dt:.1f} s)"}


def timed(run, steps, stream, dist, dev, torch):
    """Device time of `steps` steps (CUDA events on the launch stream, barrier +
    synchronize on both sides), max over ranks, in ms."""
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    return float(ms.item())


def make_graph(torch, dev, stream, fn, reps):
    side = torch.cuda.Stream(dev)
    side.wait_stream(stream)
    with torch.cuda.stream(side):
        for _ in range(reps):
            fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    torch.cuda.synchronize()
    return g


def kernel_profile(cdc, step, steps, torch):
    """Per-kernel CUDA events on the launch stream over `steps` direct-launch steps."""
    cdc.profile_enable(True)
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    cdc.profile_enable(False)
    return cdc.profile_collect()


def measure_c3(args, cdc, torch, dist, dev, world, rank, local):
    import synth
    from paper_2508_05797_b200 import shard
    offs_all = synth.many_files_offsets(NFILES, FSEED)
    f0, f1 = shard.file_range(offs_all, world, rank)
    data_np, offs = synth.many_files(NFILES, FSEED, files=(f0, f1))
    nf = f1 - f0
    total = int(offs[-1])
    max_len = int(np.diff(offs).max()) if nf else 0
    p = cdc.params(C3_ALGO, avg_size=C3_AVG)
    data = torch.from_numpy(data_np).to(dev)
    od = torch.from_numpy(offs).to(dev)
    cap = total // (p.window + 1) + nf
    bounds = torch.empty(max(cap, 1), dtype=torch.int64, device=dev)
    bo = torch.zeros(nf + 1, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(cdc.workspace_size(p, nf, total, max_len), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():  # on the current stream (the graph capture's stream while capturing)
        cdc.chunk_batch_async(data, od, total, max_len, p, bounds, bo, count, ws)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    n_bounds = int(count.item())
    launches = cdc.last_launch_count()
    checked = None
    if args.check:
        import oracle
        bad = oracle.check_batch(C3_ALGO, data_np, offs, bounds[:n_bounds].cpu().numpy().astype(np.uint64),
                                 bo.cpu().numpy().astype(np.uint64), p.window, p.max_size)
        assert bad is None, f"boundary mismatch vs oracle at {bad}"
        checked = "every chunk of this rank's files == oracle (oracle.check_batch)"
    stats = cdc.stats(p, ws, nf, total, max_len)
    fetched = cdc.fetched(p, ws, nf, total, max_len)  # bytes the walkers copied from HBM in one call
    graph = None if args.no_graph else make_graph(torch, dev, stream, step, 1)

    def run(k):
        for _ in range(k):
            graph.replay() if graph is not None else step()

    with ClockSampler(local) as clk:
        t_end = time.perf_counter() + 0.3  # load the GPU so clock samples reflect the timed region
        while time.perf_counter() < t_end:
            run(1)
            torch.cuda.synchronize()
        ms = timed(run, args.steps, stream, dist, dev, torch)
        prof = kernel_profile(cdc, step, args.steps, torch)
    assert int(count.item()) == n_bounds, "boundary count changed between steps"
    # global boundary count: one all_gather of the per-rank counts (shard.chunk_files_sharded's exchange)
    n_all = n_bounds
    bytes_all = total
    if dist is not None:
        t = torch.tensor([n_bounds, total], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        n_all, bytes_all = int(t[0]), int(t[1])
    res = {"ms": ms, "bytes_rank": total, "bytes_all": bytes_all, "boundaries": n_all, "files": (f0, f1),
           "prof": prof, "launches": launches, "stats": stats, "fetched": fetched, "clocks": clk.summary(), "checked": checked,
           "graph": graph is not None, "p": p}
    if not args.no_e2e:
        res["e2e"] = measure_e2e_c3(cdc, torch, p, data_np, offs, dist, dev, world, args.steps)
    if not args.no_cpu_baseline and world == 1 and rank == 0:
        res["cpu_baseline"] = cpu_baseline(data_np, offs)
    del data, ws, bounds
    torch.cuda.empty_cache()
    return res


def measure_e2e_c3(cdc, torch, p, data_np, offs, dist, dev, world, steps):
    """The same metric through cdc_chunk_batch_host: pinned host bytes in (grouped,
    pipelined H2D copies inside the call), host boundaries out."""
    pinned = torch.empty(data_np.size, dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = data_np
    host_in = pinned.numpy()
    out = np.empty(int(offs[-1]) // (p.window + 1) + offs.size, dtype=np.uint64)
    b, bo = cdc.chunk_batch_host(host_in, offs, p, out)
    n = b.size
    k = max(3, min(steps, 5))
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(k):
        b, bo = cdc.chunk_batch_host(host_in, offs, p, out)
    dt = time.perf_counter() - t0
    tt = torch.tensor([dt], dtype=torch.float64, device=dev)
    tb = torch.tensor([float(data_np.size)], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.all_reduce(tb)
    del pinned
    return {"value": round(float(tb.item()) * k / float(tt.item()) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": int(data_np.size + offs.nbytes), "d2h_bytes_per_step": int(8 * n + bo.nbytes),
            "timing": f"wall clock around {k} synchronous cdc_chunk_batch_host calls (pinned input), max over ranks"}


def measure_c1(args, cdc, torch, dist, dev, world):
    """configs[1] on every rank (secondary; round 1's headline): 256 MiB Zipf stream,
    AE-Max 4 KiB; CUDA graph of two steps over two device copies (L2 never warm)."""
    import synth
    data_np = synth.zipf_bytes(C1_STREAM, 1.1, 1)
    bufs = [torch.from_numpy(data_np).to(dev) for _ in range(2)]
    p = cdc.params(C1_ALGO, avg_size=C1_AVG)
    cap = cdc.max_boundaries(p, C1_STREAM)
    bounds = torch.empty(cap, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(cdc.workspace_size(p, 1, C1_STREAM, C1_STREAM), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    it = [0]

    def step():  # on the current stream (the graph capture's stream while capturing)
        cdc.chunk_async(bufs[it[0] & 1], p, bounds, count, ws)
        it[0] += 1

    for _ in range(4):
        step()
    torch.cuda.synchronize()
    n_bounds = int(count.item())
    if args.check:
        import oracle
        bad = oracle.check_chunking(C1_ALGO, data_np, bounds[:n_bounds].cpu().numpy().astype(np.uint64),
                                    p.window, p.max_size)
        assert bad is None, f"configs[1] mismatch vs oracle at {bad}"
    graph = make_graph(torch, dev, stream, step, 2)

    def run(k):
        for _ in range(k // 2):
            graph.replay()
        if k % 2:
            step()

    steps = max(args.steps, 20)
    ms = timed(run, steps, stream, dist, dev, torch)
    prof = kernel_profile(cdc, step, steps, torch)
    peak, peak_src = load_peaks()
    spec_ms = prof["k_speculate"][0] / max(1, prof["k_speculate"][1])
    traffic, traffic_src = load_traffic("ncu_k_speculate_c1.json")
    out = {
        "workload": "configs[1]: AE-Max avg 4 KiB, single 256 MiB stream of Zipf(s=1.1) bytes, seed 1, on every rank",
        "value": round(C1_STREAM * world * steps / (ms / 1e3) / 1e9, 2), "unit": "GB/s",
        "ms_per_step": round(ms / steps, 4), "steps": steps, "boundaries": n_bounds, "scaling": "weak",
        "roofline": {"bound": "hbm", "kernel": "k_speculate",
                     "achieved": round(C1_STREAM / (spec_ms / 1e3) / 1e9, 1), "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s",
                     "frac": round(C1_STREAM / (spec_ms / 1e3) / 1e9 / peak, 4), "traffic": traffic,
                     "traffic_source": traffic_src, "kernel_ms": round(spec_ms, 4),
                     "step_frac": round(C1_STREAM * steps / (ms / 1e3) / 1e9 / peak, 4)},
        "timing": "CUDA graph (2 steps per replay), events on the launch stream, max over ranks; kernel_ms from "
                  "per-kernel events in a second pass of direct launches",
    }
    del bufs, ws, bounds
    torch.cuda.empty_cache()
    return out


C0_STREAM, C0_COPIES = 16 << 20, 10


def measure_c0(args, cdc, torch, dist, dev, world):
    """configs[0] on every rank (secondary): RAM 8 KiB on one 16 MiB stream of uniform
    bytes, seed 0 -- the small saturated stream the dense-index mode resolves.
    CUDA graph of 10 calls over 10 device copies (160 MiB > L2: no call finds its input cached)."""
    import synth
    data_np = synth.uniform(C0_STREAM, 0)
    bufs = [torch.from_numpy(data_np).to(dev) for _ in range(C0_COPIES)]
    p = cdc.params("ram", avg_size=8192)
    cap = cdc.max_boundaries(p, C0_STREAM)
    bounds = torch.empty(cap, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(cdc.workspace_size(p, 1, C0_STREAM, C0_STREAM), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    it = [0]

    def step():
        cdc.chunk_async(bufs[it[0] % C0_COPIES], p, bounds, count, ws)
        it[0] += 1

    for _ in range(C0_COPIES):
        step()
    torch.cuda.synchronize()
    n_bounds = int(count.item())
    launches = cdc.last_launch_count()
    path = cdc.stats(p, ws, 1, C0_STREAM, C0_STREAM)
    if args.check:
        import oracle
        bad = oracle.check_chunking("ram", data_np, bounds[:n_bounds].cpu().numpy().astype(np.uint64),
                                    p.window, p.max_size)
        assert bad is None, f"configs[0] mismatch vs oracle at {bad}"
    graph = make_graph(torch, dev, stream, step, C0_COPIES)

    def run(k):
        for _ in range(k // C0_COPIES):
            graph.replay()

    steps = C0_COPIES * max(5, args.steps // 2)
    t_end = time.perf_counter() + 0.2  # (the first key measured: bring the clocks up before a 3 ms timed region)
    while time.perf_counter() < t_end:
        run(C0_COPIES)
        torch.cuda.synchronize()
    ms = timed(run, steps, stream, dist, dev, torch)
    peak, peak_src = load_peaks()
    gbs = C0_STREAM * steps / (ms / 1e3) / 1e9
    out = {
        "workload": "configs[0]: RAM avg 8 KiB, single 16 MiB stream of uniform bytes, seed 0, on every rank",
        "value": round(gbs * world, 2), "unit": "GB/s", "ms_per_step": round(ms / steps, 5), "steps": steps,
        "boundaries": n_bounds, "scaling": "weak", "gpu_launches": launches * steps, "path": path,
        "roofline": {"bound": "hbm", "kernel": "k_dense_index (whole call)", "achieved": round(gbs, 1), "peak": peak,
                     "peak_source": peak_src, "unit": "GB/s", "frac": round(gbs / peak, 4),
                     "per_unit": "1 B per input byte (every byte is read once to index the saturating bytes; "
                                 "the 2w bytes after each segment are read again: +14 %, not counted)"},
        "timing": f"CUDA graph of {C0_COPIES} calls over {C0_COPIES} device copies (L2 cold), events on the launch "
                  "stream, max over ranks",
    }
    del bufs, ws, bounds
    torch.cuda.empty_cache()
    return out


MX_STREAM = 1 << 30


def measure_maxp(args, cdc, torch, dist, dev, world):
    """MAXP (§2.1.2 l.173/l.196; not in BASELINE's configs -- the algorithm
    the paper accelerates besides AE and RAM): one 1 GiB uniform stream per rank at
    the 8 KiB default (h = 447); CUDA graph of one call; the 1 GiB input exceeds L2."""
    import synth
    data_np = synth.uniform(MX_STREAM, 2)
    data = torch.from_numpy(data_np).to(dev)
    p = cdc.params("maxp", avg_size=8192)
    cap = cdc.max_boundaries(p, MX_STREAM)
    bounds = torch.empty(cap, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(cdc.workspace_size(p, 1, MX_STREAM, MX_STREAM), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        cdc.chunk_async(data, p, bounds, count, ws)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    n_bounds = int(count.item())
    launches = cdc.last_launch_count()
    if args.check:
        import oracle
        bad = oracle.check_chunking("maxp", data_np, bounds[:n_bounds].cpu().numpy().astype(np.uint64),
                                    p.window, p.max_size)
        assert bad is None, f"MAXP mismatch vs oracle at {bad}"
    graph = make_graph(torch, dev, stream, step, 1)

    def run(k):
        for _ in range(k):
            graph.replay()

    steps = max(args.steps, 10)
    ms = timed(run, steps, stream, dist, dev, torch)
    peak, peak_src = load_peaks()
    call_gbs = MX_STREAM * steps / (ms / 1e3) / 1e9
    tile = 32768  # k_maxp_scan reads each 32 KiB tile with both h-byte margins
    read = MX_STREAM + (MX_STREAM // tile) * 2 * p.window
    out = {
        "workload": "MAXP avg 8 KiB (window h = 447 per side, max_size 32 KiB), one 1 GiB stream of uniform bytes, "
                    "seed 2, on every rank",
        "value": round(call_gbs * world, 2), "unit": "GB/s", "ms_per_step": round(ms / steps, 4), "steps": steps,
        "boundaries": n_bounds, "scaling": "weak", "gpu_launches": launches * steps,
        "roofline": {"bound": "hbm", "kernel": "k_maxp_scan..k_maxp_write (whole call)",
                     "achieved": round(read * steps / (ms / 1e3) / 1e9, 1), "peak": peak, "peak_source": peak_src,
                     "unit": "GB/s", "frac": round(read * steps / (ms / 1e3) / 1e9 / peak, 4),
                     "algorithmic_gb_per_launch": round(read / 1e9, 4),
                     "per_unit": "every input byte read once, plus the two h-byte margins of each 32 KiB tile "
                                 "(DESIGN.md §5, MAXP)"},
        "timing": "CUDA graph of one call, events on the launch stream, max over ranks",
    }
    del data, ws, bounds
    torch.cuda.empty_cache()
    return out


def measure_c4(args, cdc, torch, dist, dev, world, rank):
    """configs[4]: one 64 GiB stream split by byte range with a halo over the ranks
    (shard.chunk_sharded through the public API; NCCL all_gather of edge chain
    states), RAM and AE-Max at 8 KiB."""
    import synth
    from paper_2508_05797_b200 import shard
    out = {"workload": "configs[4]: one 64 GiB stream of alternating 256 MiB regions (uniform / runs of one value, "
                       "geometric mean 512), split by byte range with a halo over the ranks (shard.chunk_sharded)",
           "stream_bytes": C4_LEN, "scaling": "strong", "unit": "GB/s"}
    buf = None
    for algo in ("ram", "ae_max"):
        p = cdc.params(algo, avg_size=8192)
        halo = shard.default_halo(p.max_size, p.window)
        pl = shard.plan(C4_LEN, world, rank, halo)
        if buf is None:
            buf = torch.from_numpy(synth.alternating(C4_LEN, region=256 << 20, seed=5,
                                                     part=(pl.a, pl.buf_end))).to(dev)
        comm = shard.DistComm() if dist is not None else None
        backend = shard.CudaBackend()
        res = [None]

        def run(k):
            for _ in range(k):
                res[0] = shard.chunk_sharded(buf, pl, p, backend, comm)

        run(1)
        steps = max(3, min(args.steps, 10))
        ms = timed(run, steps, torch.cuda.current_stream(dev), dist, dev, torch)
        out[algo] = {"value": round(C4_LEN * steps / (ms / 1e3) / 1e9, 2), "ms_per_step": round(ms / steps, 3),
                     "steps": steps, "boundaries": int(res[0][2]), "halo_bytes": halo}
    out["timing"] = ("CUDA events on the current stream around shard.chunk_sharded (allocations, the local "
                     "cdc_chunk, the all_gather and the resync included), barrier + synchronize, max over ranks")
    del buf
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--check", action="store_true", help="verify every boundary against the oracle once")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end host-buffer measurement")
    ap.add_argument("--no-graph", action="store_true", help="time direct launches instead of a CUDA graph")
    ap.add_argument("--no-secondary", action="store_true", help="skip the configs[1] and configs[4] keys")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import paper_2508_05797_b200 as cdc

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    c0 = None if args.no_secondary else measure_c0(args, cdc, torch, dist, dev, world)
    c1 = None if args.no_secondary else measure_c1(args, cdc, torch, dist, dev, world)
    c3 = measure_c3(args, cdc, torch, dist, dev, world, rank, local)
    c4 = None if args.no_secondary else measure_c4(args, cdc, torch, dist, dev, world, rank)
    mx = None if args.no_secondary else measure_maxp(args, cdc, torch, dist, dev, world)

    if rank == 0:
        ms = c3["ms"]
        gbs = c3["bytes_all"] * args.steps / (ms / 1e3) / 1e9
        prof = c3["prof"]
        spec_ms = prof["k_speculate"][0] / max(1, prof["k_speculate"][1])
        step_ms = ms / args.steps
        peak, peak_src = load_peaks()
        traffic, traffic_src = load_traffic("ncu_k_speculate_c3.json")
        fetched = c3["fetched"]  # algorithmic bytes of one launch, counted by the kernel
        achieved = fetched / (spec_ms / 1e3) / 1e9
        input_gbs = c3["bytes_rank"] / (spec_ms / 1e3) / 1e9
        ksum = sum(prof[k][0] for k in cdc.KERNELS)
        p = c3["p"]
        line = {
            "metric": METRIC, "value": round(gbs, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(step_ms, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD, "algo": C3_ALGO, "avg_size": C3_AVG, "window": p.window,
                       "max_size": p.max_size, "files": NFILES, "total_bytes": c3["bytes_all"],
                       "rank0_files": list(c3["files"]), "rank0_bytes": c3["bytes_rank"],
                       "boundaries": c3["boundaries"],
                       "l2": "no flush: the resident input (18.67 GiB / N per rank) is far larger than L2 (126 MB)",
                       "parallelism": f"files{world}: contiguous byte-balanced file ranges per rank "
                                      f"(shard.file_range), no data-path collective"},
            "roofline": {"bound": "hbm", "kernel": "k_speculate", "achieved": round(achieved, 1), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_gb_per_launch": round(fetched / 1e9, 4),
                         "per_unit": "bytes the walkers must copy from HBM: 1 B per byte the TMA ring walker streams, "
                                     "SP_SPEC = 2 KiB per chunk the sparse walk decides (plus its rare continuation "
                                     "and window-probe copies); counted by k_speculate during the run (cdc_fetched), "
                                     "DESIGN.md §5",
                         "fetched_bytes_per_input_byte": round(fetched / c3["bytes_rank"], 4),
                         "input_gb_per_launch": round(c3["bytes_rank"] / 1e9, 4),
                         "input_gbs": round(input_gbs, 1),
                         "kernel_ms": round(spec_ms, 4),
                         "share_of_step": {k: round(prof[k][0] / max(1e-9, ksum), 4) for k in cdc.KERNELS}},
            "gpu_launches": c3["launches"] * args.steps,
            "path": c3["stats"],
            "timing": {"value": ("CUDA graph of one step" if c3["graph"] else "direct launches")
                       + ", CUDA events on the launch stream, barrier + synchronize, max over ranks",
                       "kernel_ms": "per-kernel CUDA events on the launch stream in a second pass of K direct-launch "
                                    "steps"},
            "clocks": c3["clocks"],
            "e2e": c3.get("e2e"),
        }
        if traffic is not None and world == 1:  # (the capture is of the whole batch on one GPU)
            line["roofline"]["traffic_over_algorithmic"] = round(traffic * 1e9 / max(1, fetched), 4)
        if c3.get("checked"):
            line["checked"] = c3["checked"]
        if "cpu_baseline" in c3:
            line["cpu_baseline"] = c3["cpu_baseline"]
        if c0 is not None:
            line["configs0"] = c0
        if c1 is not None:
            line["configs1"] = c1
        if c4 is not None:
            line["configs4_sharded"] = c4
        if mx is not None:
            line["maxp"] = mx
        line["paper_cpu_vector"] = PAPER_CPU
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
