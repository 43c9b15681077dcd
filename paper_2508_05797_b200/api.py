"""Thin Python binding over the C ABI (argument marshalling only).

Every computation runs in libcdc_b200.so's CUDA kernels; PyTorch provides the
device memory (CUDA tensors) and the stream.  Names follow include/cdc_b200.h.
"""
from __future__ import annotations

import contextlib
import ctypes

import numpy as np
import torch

from ._lib import CdcError, cdc_params, check, lib

ALGOS = {"ram": 0, "ae_max": 1, "ae_min": 2, "maxp": 3}
MODES = {"max": 0, "min": 1}
CMPS = {"gt": 0, "geq": 1, "lt": 2, "leq": 3, "eq": 4}

__all__ = [
    "CdcError", "ALGOS", "params", "window_for_avg", "max_boundaries", "workspace_size",
    "chunk_async", "chunk", "chunk_batch", "chunk_batch_async", "chunk_host", "chain",
    "extreme_byte_search", "range_scan", "first_common", "last_launch_count", "abi_version",
    "profile_enable", "profile_collect", "KERNELS", "stats", "fetched", "plan_info", "segment_starts",
    "chunk_batch_host", "set_kphase", "set_dense",
]


KERNELS = ["k_seg_prefix", "k_speculate", "k_fixup"]


def profile_enable(on: bool = True) -> None:
    check(lib.cdc_profile_enable(1 if on else 0))


def profile_collect() -> dict:
    """{kernel: (summed ms, launches)} since the last collect (synchronises)."""
    ms = (ctypes.c_double * len(KERNELS))()
    n = (ctypes.c_uint64 * len(KERNELS))()
    calls = ctypes.c_uint64()
    check(lib.cdc_profile_collect(ms, n, ctypes.byref(calls)))
    out = {k: (float(ms[i]), int(n[i])) for i, k in enumerate(KERNELS)}
    out["calls"] = int(calls.value)
    return out


def stats(p: cdc_params, workspace: torch.Tensor, nfiles: int, total_len: int, max_len: int, stream=None) -> dict:
    """Diagnostics of the last call that used `workspace` (synchronises)."""
    out = (ctypes.c_uint64 * 8)()
    check(lib.cdc_stats(ctypes.byref(p), nfiles, total_len, max_len, workspace.data_ptr(), out, _stream_ptr(stream)))
    keys = ["segments", "seg_bytes", "halo_cap", "fast_path", "synced", "unsynced", "skipped_or_end", "halo_chunks"]
    return {k: int(out[i]) for i, k in enumerate(keys)}


def fetched(p: cdc_params, workspace: torch.Tensor, nfiles: int, total_len: int, max_len: int, stream=None) -> int:
    """Bytes k_speculate's walkers copied from global memory in the last call on `workspace` (synchronises)."""
    out = ctypes.c_uint64()
    check(lib.cdc_fetched(ctypes.byref(p), nfiles, total_len, max_len, workspace.data_ptr(), ctypes.byref(out),
                          _stream_ptr(stream)))
    return int(out.value)


def plan_info(p: cdc_params, nfiles: int, total_len: int, max_len: int) -> dict:
    """Speculation geometry (host-only): segment bytes, halo cap, segments of one stream."""
    out = (ctypes.c_uint64 * 3)()
    check(lib.cdc_plan_info(ctypes.byref(p), nfiles, total_len, max_len, out))
    return {"seg_bytes": int(out[0]), "halo_cap": int(out[1]), "segments": int(out[2])}


def segment_starts(p: cdc_params, length: int) -> list:
    """First byte of every speculation segment of a single stream (cdc_plan_segments)."""
    n = ctypes.c_uint64()
    check(lib.cdc_plan_segments(ctypes.byref(p), length, None, 0, ctypes.byref(n)))
    out = np.zeros(max(n.value, 1), dtype=np.uint64)
    check(lib.cdc_plan_segments(ctypes.byref(p), length, out.ctypes.data, out.size, ctypes.byref(n)))
    return out[:n.value].astype(np.int64).tolist()


def abi_version() -> int:
    return lib.cdc_abi_version()


def last_launch_count() -> int:
    return lib.cdc_last_launch_count()


def set_kphase(k: int) -> None:
    """K-phase speculation (cdc_set_kphase): -1 default, 0 off, 1..8 chains per segment (process-wide)."""
    check(lib.cdc_set_kphase(k))


def set_dense(on: int) -> None:
    """Dense-index mode (cdc_set_dense): -1 default, 0 off, 1 on (process-wide)."""
    check(lib.cdc_set_dense(int(on)))


def window_for_avg(algo: str, avg_size: int) -> int:
    w = ctypes.c_uint32()
    check(lib.cdc_window_for_avg(ALGOS[algo], avg_size, ctypes.byref(w)))
    return int(w.value)


def params(algo: str, avg_size: int | None = None, window: int | None = None, max_size: int | None = None,
           seg_bytes: int = 0, halo_bytes: int = 0) -> cdc_params:
    p = cdc_params()
    if avg_size is not None:
        check(lib.cdc_params_default(ctypes.byref(p), ALGOS[algo], avg_size))
    else:
        p.algo = ALGOS[algo]
    if window is not None:
        p.window = window
    if max_size is not None:
        p.max_size = max_size
    p.seg_bytes = seg_bytes
    p.halo_bytes = halo_bytes
    return p


def max_boundaries(p: cdc_params, length: int) -> int:
    return int(lib.cdc_max_boundaries(ctypes.byref(p), length))


def workspace_size(p: cdc_params, nfiles: int, total_len: int, max_len: int) -> int:
    n = ctypes.c_size_t()
    check(lib.cdc_workspace_size(ctypes.byref(p), nfiles, total_len, max_len, ctypes.byref(n)))
    return int(n.value)


def _stream_ptr(stream) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


class _Ctx:
    def __init__(self, caller):
        self.caller = caller
        self.out = []

    def hand_over(self, *tensors):
        """Tensors returned to the caller: the caller's stream may use (and free) them."""
        self.out.extend(tensors)
        return tensors[0] if len(tensors) == 1 else tensors


@contextlib.contextmanager
def _on(stream):
    """Run a wrapper's whole body (allocations, fills, launches, the final count
    read) on `stream`, after the work already queued on the caller's current
    stream; afterwards the caller's stream waits for `stream`, and the tensors
    handed over are recorded as used by the caller's stream."""
    if stream is None:
        yield _Ctx(None)
        return
    caller = torch.cuda.current_stream()
    stream.wait_stream(caller)
    ctx = _Ctx(caller)
    with torch.cuda.stream(stream):
        yield ctx
    caller.wait_stream(stream)
    for t in ctx.out:
        t.record_stream(caller)


def _dev_u8(data: torch.Tensor) -> torch.Tensor:
    if not (isinstance(data, torch.Tensor) and data.is_cuda and data.dtype == torch.uint8):
        raise TypeError("data must be a CUDA uint8 tensor")
    return data.contiguous()


def _workspace(nbytes: int, device) -> torch.Tensor:
    # torch's caching allocator returns 512-byte aligned blocks
    return torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)


def chunk_async(data: torch.Tensor, p: cdc_params, bounds: torch.Tensor, count: torch.Tensor,
                workspace: torch.Tensor, stream=None) -> None:
    """cdc_chunk on preallocated device buffers (no synchronisation)."""
    check(lib.cdc_chunk(ctypes.byref(p), data.data_ptr(), data.numel(), bounds.data_ptr(), bounds.numel(),
                        count.data_ptr(), workspace.data_ptr(), workspace.numel(), _stream_ptr(stream)))


def chunk(data: torch.Tensor, p: cdc_params, stream=None) -> torch.Tensor:
    """Chunk boundaries (exclusive end offsets, int64 tensor on the device) of one stream."""
    data = _dev_u8(data)
    n = data.numel()
    cap = max_boundaries(p, n)
    with _on(stream) as c:
        bounds = torch.empty(max(cap, 1), dtype=torch.int64, device=data.device)
        count = torch.zeros(1, dtype=torch.int64, device=data.device)
        ws = _workspace(workspace_size(p, 1, n, n), data.device)
        chunk_async(data, p, bounds, count, ws)
        m = int(count.item())
        c.hand_over(bounds)
    if m > cap:
        raise CdcError(f"boundary count {m} exceeds capacity {cap}")
    return bounds[:m]


def chunk_batch_async(data: torch.Tensor, file_offsets: torch.Tensor, total_len: int, max_len: int, p: cdc_params,
                      bounds: torch.Tensor, bound_offsets: torch.Tensor, count: torch.Tensor, workspace: torch.Tensor,
                      stream=None) -> None:
    """cdc_chunk_batch on preallocated device buffers (file_offsets: int64[nfiles+1] on the device; no
    synchronisation).  total_len and max_len are the batch's byte count and largest file."""
    check(lib.cdc_chunk_batch(ctypes.byref(p), data.data_ptr(), file_offsets.data_ptr(), file_offsets.numel() - 1,
                              total_len, max_len, bounds.data_ptr(), bounds.numel(), bound_offsets.data_ptr(),
                              count.data_ptr(), workspace.data_ptr(), workspace.numel(), _stream_ptr(stream)))


def chunk_batch(data: torch.Tensor, file_offsets, p: cdc_params, stream=None):
    """Per-file boundaries of a packed batch: (bounds int64[total], bound_offsets int64[nfiles+1])."""
    data = _dev_u8(data)
    offs_h = np.asarray(file_offsets, dtype=np.int64)
    nfiles = offs_h.size - 1
    sizes = np.diff(offs_h)
    total = int(sizes.sum()) if nfiles else 0
    max_len = int(sizes.max()) if nfiles else 0
    cap = total // (p.window + 1) + nfiles  # every chunk but a file's last holds > w bytes
    with _on(stream) as c:
        offs = torch.from_numpy(offs_h.copy()).to(data.device)
        bounds = torch.empty(max(cap, 1), dtype=torch.int64, device=data.device)
        bo = torch.zeros(nfiles + 1, dtype=torch.int64, device=data.device)
        count = torch.zeros(1, dtype=torch.int64, device=data.device)
        ws = _workspace(workspace_size(p, nfiles, total, max_len), data.device)
        check(lib.cdc_chunk_batch(ctypes.byref(p), data.data_ptr(), offs.data_ptr(), nfiles, total, max_len,
                                  bounds.data_ptr(), cap, bo.data_ptr(), count.data_ptr(), ws.data_ptr(), ws.numel(),
                                  _stream_ptr(None)))
        m = int(count.item())
        c.hand_over(bounds, bo)
    if m > cap:
        raise CdcError(f"boundary count {m} exceeds capacity {cap}")
    return bounds[:m], bo


def chunk_host(data: np.ndarray, p: cdc_params, out: np.ndarray | None = None) -> np.ndarray:
    """cdc_chunk_host: host bytes in, host boundaries out (copies inside the call)."""
    data = np.ascontiguousarray(data, dtype=np.uint8)
    cap = max_boundaries(p, data.size)
    if out is None or out.size < cap:
        out = np.empty(max(cap, 1), dtype=np.uint64)
    n = ctypes.c_uint64()
    check(lib.cdc_chunk_host(ctypes.byref(p), data.ctypes.data, data.size, out.ctypes.data, out.size,
                             ctypes.byref(n)))
    return out[:n.value]


def chunk_batch_host(data: np.ndarray, file_offsets, p: cdc_params, out: np.ndarray | None = None):
    """cdc_chunk_batch_host: packed host bytes + host file offsets in, host per-file boundaries out
    (copies inside the call, pipelined by file groups).  Returns (bounds uint64[total], bound_offsets
    uint64[nfiles+1])."""
    data = np.ascontiguousarray(data, dtype=np.uint8)
    offs = np.ascontiguousarray(file_offsets, dtype=np.uint64)
    nfiles = offs.size - 1
    if nfiles < 1:
        raise CdcError("need at least one file")
    cap = int(offs[-1] - offs[0]) // (p.window + 1) + nfiles
    if out is None or out.size < cap:
        out = np.empty(max(cap, 1), dtype=np.uint64)
    bo = np.zeros(nfiles + 1, dtype=np.uint64)
    n = ctypes.c_uint64()
    check(lib.cdc_chunk_batch_host(ctypes.byref(p), data.ctypes.data, offs.ctypes.data, nfiles, out.ctypes.data,
                                   out.size, bo.ctypes.data, ctypes.byref(n)))
    return out[:n.value], bo


def chain(data: torch.Tensor, p: cdc_params, start: int, stop: int, cap: int | None = None,
          stream=None) -> torch.Tensor:
    """Chunk starts of the chain begun at `start`, up to the first start >= stop."""
    data = _dev_u8(data)
    if cap is None:
        cap = max_boundaries(p, max(0, min(stop, data.numel()) - start)) + 2
    with _on(stream) as c:
        out = torch.empty(cap, dtype=torch.int64, device=data.device)
        cnt = torch.zeros(1, dtype=torch.int64, device=data.device)
        check(lib.cdc_chain(ctypes.byref(p), data.data_ptr(), data.numel(), start, stop, out.data_ptr(), cap,
                            cnt.data_ptr(), _stream_ptr(None)))
        m = int(cnt.item())
        c.hand_over(out)
    if m > cap:
        raise CdcError(f"chain length {m} exceeds capacity {cap}")
    return out[:m]


def first_common(a: torch.Tensor, b: torch.Tensor, stream=None) -> torch.Tensor:
    """cdc_first_common: (index in a, index in b) of the first element of sorted a found in sorted b."""
    if not (a.is_cuda and b.is_cuda and a.dtype == torch.int64 and b.dtype == torch.int64):
        raise TypeError("a and b must be CUDA int64 tensors")
    a, b = a.contiguous(), b.contiguous()
    with _on(stream) as c:
        out = torch.empty(2, dtype=torch.int64, device=a.device)
        check(lib.cdc_first_common(a.data_ptr(), a.numel(), b.data_ptr(), b.numel(), out.data_ptr(),
                                   _stream_ptr(None)))
        return c.hand_over(out)


def _regions(offsets, lengths, device):
    off = torch.as_tensor(np.asarray(offsets, dtype=np.int64)).to(device)
    ln = torch.as_tensor(np.asarray(lengths, dtype=np.int64)).to(device)
    return off, ln


def extreme_byte_search(data: torch.Tensor, offsets, lengths, mode: str = "max", stream=None):
    """§4.1 on many regions: (values uint8[n], leftmost positions int64[n])."""
    data = _dev_u8(data)
    if np.size(lengths) and int(np.min(lengths)) < 1:
        raise CdcError("empty region")
    with _on(stream) as c:
        off, ln = _regions(offsets, lengths, data.device)
        n = off.numel()
        val = torch.empty(n, dtype=torch.uint8, device=data.device)
        pos = torch.empty(n, dtype=torch.int64, device=data.device)
        check(lib.cdc_extreme_byte_search(data.data_ptr(), off.data_ptr(), ln.data_ptr(), n, MODES[mode],
                                          val.data_ptr(), pos.data_ptr(), _stream_ptr(None)))
        return c.hand_over(val, pos)


def range_scan(data: torch.Tensor, offsets, lengths, targets, cmp: str, stream=None) -> torch.Tensor:
    """§4.2 on many regions: first matching offset per region (region length if none)."""
    data = _dev_u8(data)
    with _on(stream) as c:
        off, ln = _regions(offsets, lengths, data.device)
        tg = torch.as_tensor(np.asarray(targets, dtype=np.uint8)).to(data.device)
        n = off.numel()
        pos = torch.empty(n, dtype=torch.int64, device=data.device)
        check(lib.cdc_range_scan(data.data_ptr(), off.data_ptr(), ln.data_ptr(), tg.data_ptr(), n, CMPS[cmp],
                                 pos.data_ptr(), _stream_ptr(None)))
        return c.hand_over(pos)
