#!/usr/bin/env python
"""bench.py -- chunking throughput of the B200 CDC hot path (driver contract).

One step = one cdc_chunk call over the whole resident stream: speculative
segment chunking with the fused look-back resolution and boundary write
(k_speculate), and the fix-up kernel (k_fixup, which exits at once when the
fused fast path succeeded) -- every row of DESIGN.md §0(a).  Workload at N=1 = BASELINE.json
configs[1]: AE (AE-Max) at a 4 KiB target average, one 256 MiB stream of
Zipf(s=1.1) bytes, seed 1.  With N ranks (torchrun) every rank chunks its own
256 MiB stream (the configs[1] stream, seed 1, on every rank): the work shards with no collective on the data
path ("scaling": "weak").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--impl reference times the CPU oracle (oracle/, plain C, one host core) on the
same workload, one 32 MiB slice per step; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "chunking GB/s of input (1/2/4/8 B200) and % of HBM roofline; boundaries == oracle"
ALGO, AVG, STREAM = "ae_max", 4096, 256 << 20
WORKLOAD = "configs[1]: AE (AE-Max) avg 4 KiB, single 256 MiB stream of Zipf(s=1.1) bytes, seed 1"
REF_SLICE = 32 << 20


def load_traffic():
    """DRAM traffic per k_speculate launch from the committed ncu --set full capture
    (profiles/ncu_k_speculate_latest.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_k_speculate_latest.json")) as f:
            t = json.load(f)
        return float(t["traffic_bytes"]) / 1e9, "dram__bytes_read.sum + dram__bytes_write.sum per launch (GB), " \
            "profiles/ncu_k_speculate_latest.json"
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


def run_reference(args, world, rank):
    """CPU oracle arm: rank 0 only, on the box's host cores."""
    if rank != 0:
        return 0
    import oracle
    import synth
    data = synth.zipf_bytes(STREAM, 1.1, 1)
    w, mx = AVG - 256, 4 * AVG  # same window / cap as the GPU arm's cdc_params_default
    nsl = STREAM // REF_SLICE

    def step(i):
        sl = data[(i % nsl) * REF_SLICE:((i % nsl) + 1) * REF_SLICE]
        return oracle.chunk(ALGO, sl, w, mx).size

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    dt = time.perf_counter() - t0
    gbs = args.steps * REF_SLICE / dt / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(gbs, 4), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": WORKLOAD, "algo": ALGO, "avg_size": AVG, "window": w, "max_size": mx,
                   "parallelism": "cpu oracle, rank 0 only"},
        "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"one {REF_SLICE >> 20} MiB slice of the 256 MiB stream per step"},
        "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(data_np, w, mx):
    """The oracle as it stands on one host core over the full 256 MiB stream (one pass)."""
    import oracle
    t0 = time.perf_counter()
    oracle.chunk(ALGO, data_np, w, mx)
    dt = time.perf_counter() - t0
    return {"value": round(data_np.size / dt / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": "the full 256 MiB configs[1] stream, one pass, C oracle (gcc -O2), 1 thread"}


def measure_e2e(cdc, p, data_np, cap, world, dist, dev, steps):
    """Same metric through cdc_chunk_host: pinned host bytes in, host boundaries out."""
    import torch
    pinned = torch.empty(STREAM, dtype=torch.uint8, pin_memory=True)
    pinned.copy_(torch.from_numpy(data_np))
    host_in = pinned.numpy()
    host_out = np.empty(cap, dtype=np.uint64)
    cdc.chunk_host(host_in, p, host_out)
    e2e_steps = max(3, min(steps, 20))
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        nb = cdc.chunk_host(host_in, p, host_out).size
    e2e_s = time.perf_counter() - t0
    e2e_t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
    return {"value": round(STREAM * world * e2e_steps / float(e2e_t.item()) / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": STREAM, "d2h_bytes_per_step": 8 + 8 * nb,
            "timing": "wall clock around the synchronous cdc_chunk_host call (pinned input)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--check", action="store_true", help="verify the boundaries against the oracle once")
    ap.add_argument("--seg-bytes", type=int, default=0, help="speculation segment size (0 = library default)")
    ap.add_argument("--no-e2e", action="store_true", help="skip the end-to-end host-buffer measurement")
    ap.add_argument("--no-graph", action="store_true", help="time direct launches instead of a CUDA graph")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)

    import torch
    import synth
    import paper_2508_05797_b200 as cdc

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    # every rank chunks its own copy of the configs[1] stream (seed 1): equal work
    # per rank for weak scaling (another seed permutes which byte value is the
    # rare 255 and changes AE-Max's chunk statistics)
    data_np = synth.zipf_bytes(STREAM, 1.1, 1)
    # two device copies of the stream at different addresses, used alternately, so
    # that no step finds the previous step's lines in L2 (126 MB < 2 x 256 MiB)
    bufs = [torch.from_numpy(data_np).to(dev) for _ in range(2)]
    data = bufs[0]
    p = cdc.params(ALGO, avg_size=AVG, seg_bytes=args.seg_bytes)
    cap = cdc.max_boundaries(p, STREAM)
    bounds = torch.empty(cap, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = torch.empty(cdc.workspace_size(p, 1, STREAM, STREAM), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    it = [0]

    def step():
        cdc.chunk_async(bufs[it[0] & 1], p, bounds, count, ws, stream)
        it[0] += 1

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    n_bounds = int(count.item())
    if args.check and rank == 0:
        import oracle
        exp = oracle.chunk(ALGO, data_np, p.window, p.max_size)
        got = bounds[:n_bounds].cpu().numpy().astype(np.uint64)
        assert got.size == exp.size and (got == exp).all(), "boundary mismatch vs oracle"
    launches_per_step = cdc.last_launch_count()
    path_stats = cdc.stats(p, ws, 1, STREAM, STREAM)

    # The timed region replays a CUDA graph of two steps (one per input copy):
    # the three launches of a step (k_reset, k_speculate, k_fixup; the last
    # exits at once when the fused fast path succeeded) without
    # host launch overhead.  --no-graph times direct launches instead.
    graph = None
    if not args.no_graph:
        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            for b in bufs:
                cdc.chunk_async(b, p, bounds, count, ws)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for b in bufs:
                cdc.chunk_async(b, p, bounds, count, ws)
        torch.cuda.synchronize()

    def run(k):
        if graph is None:
            for _ in range(k):
                step()
            return
        for _ in range(k // 2):
            graph.replay()
        if k % 2:
            step()

    # keep the GPU loaded ~0.3 s so clock samples reflect the timed region
    with ClockSampler(local) as clk:
        t_end = time.perf_counter() + 0.3
        while time.perf_counter() < t_end:
            run(2)
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        run(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
        # second pass, same K steps as direct launches with CUDA events around
        # every kernel on the launch stream: the per-kernel durations below
        cdc.profile_enable(True)
        ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev2.record(stream)
        for _ in range(args.steps):
            step()
        ev3.record(stream)
        torch.cuda.synchronize()
        cdc.profile_enable(False)
        profiled_ms = ev2.elapsed_time(ev3)
    torch.cuda.synchronize()
    got_n = int(count.item())
    assert got_n == n_bounds, "boundary count changed between steps"
    prof = cdc.profile_collect()
    if dist is not None:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    total_bytes = STREAM * world * args.steps
    gbs = total_bytes / (ms_max / 1e3) / 1e9

    # roofline of the dominant kernel (k_speculate): algorithmic bytes per launch = the
    # stream (each input byte read once); duration = its CUDA-event time on the launch stream
    spec_ms, spec_n = prof["k_speculate"]
    spec_avg_ms = spec_ms / max(1, spec_n)
    peak, peak_src = load_peaks()
    traffic_gb, traffic_src = load_traffic()
    achieved = STREAM / (spec_avg_ms / 1e3) / 1e9
    share = {k: round(prof[k][0] / max(1e-9, sum(prof[x][0] for x in cdc.KERNELS)), 4) for k in cdc.KERNELS}

    # end to end through the public host API (pinned host input, copies inside the call)
    e2e = None if args.no_e2e else measure_e2e(cdc, p, data_np, cap, world, dist, dev, args.steps)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(gbs, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": WORKLOAD, "algo": ALGO, "avg_size": AVG, "window": p.window,
                       "max_size": p.max_size, "stream_bytes": STREAM, "boundaries": n_bounds,
                       "l2": "no flush: input (256 MiB per rank) larger than L2 (126 MB), and consecutive steps "
                             "alternate between two device copies of it",
                       "parallelism": f"dp{world}: one independent stream per rank, no data-path collective"},
            "roofline": {"bound": "hbm", "kernel": "k_speculate", "achieved": round(achieved, 1),
                         "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": traffic_gb,
                         "traffic_source": traffic_src, "algorithmic_gb_per_launch": round(STREAM / 1e9, 4),
                         "kernel_ms": round(spec_avg_ms, 4), "share_of_step": share},
            "gpu_launches": launches_per_step * args.steps,
            "path": path_stats,
            "timing": {"value": "CUDA graph of the step (2 steps per replay), CUDA events on the launch stream, "
                                "max over ranks" if graph is not None else "direct launches, CUDA events, max over ranks",
                       "kernel_ms": "per-kernel CUDA events on the launch stream in a second pass of K direct-launch steps",
                       "ms_per_step_direct_launch_with_kernel_events": round(profiled_ms / args.steps, 4)},
            "clocks": clk.summary(),
            "e2e": e2e,
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(data_np, p.window, p.max_size)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
