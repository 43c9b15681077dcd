"""CPU oracle for hashless content-defined chunking (PAPER.md, arxiv 2508.05797).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2508_05797_b200``) never imports it and
the oracle never imports the product; they share only the input generators in
``synth/``.

Contents
--------
* ``cdc_oracle.c`` (loaded through ctypes): Extreme Byte Search (§4.1), Range
  Scan (§4.2), RAM (§2.1.2 Fig. 2c, §4.3), AE-Max / AE-Min (§2.1.2 Fig. 2a,
  §4.3), MAXP (§2.1.2 Fig. 2b l.173/l.196, §4.3 l.361; ``window`` is its
  per-side window h), whole-stream chunking, chains from arbitrary starts.
* ``pyref``: the same operations as pure-Python loops (small inputs only),
  written in the *single-pass* formulation (running extreme + deadline) rather
  than the paper's target/window formulation, so the two cross-check each
  other.
* ``dedup``: space savings, Eq. (1), from exact chunk-content equality.

Parity pins: tests/test_oracle_pins.py (closed forms, brute-force predicate
enumeration, invariants, statistical closed forms, golden fixtures from the
paper's text in tests/golden/).  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import dedup, pyref  # noqa: F401

ALGOS = {"ram": 0, "ae_max": 1, "ae_min": 2, "maxp": 3}
MODES = {"max": 0, "min": 1}
CMPS = {"gt": 0, "geq": 1, "lt": 2, "leq": 3, "eq": 4}

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "cdc_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (plain -O2, no vectorisation flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c99", "-o", _LIB, _SRC])
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64, u8p, u64p = ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(ctypes.c_uint64)
        lib.oracle_extreme_byte_search.argtypes = [u8p, u64, ctypes.c_int, u8p, u64p]
        lib.oracle_extreme_byte_search.restype = ctypes.c_int
        lib.oracle_range_scan.argtypes = [u8p, u64, ctypes.c_uint8, ctypes.c_int]
        lib.oracle_range_scan.restype = u64
        lib.oracle_chunk_end.argtypes = [ctypes.c_int, u8p, u64, u64, u64, u64]
        lib.oracle_chunk_end.restype = u64
        lib.oracle_chunk.argtypes = [ctypes.c_int, u8p, u64, u64, u64, u64p, u64]
        lib.oracle_chunk.restype = u64
        lib.oracle_chain_from.argtypes = [ctypes.c_int, u8p, u64, u64, u64, u64, u64, u64p, u64]
        lib.oracle_chain_from.restype = u64
        lib.oracle_check_ends.argtypes = [ctypes.c_int, u8p, u64, u64, u64, u64p, u64, u64]
        lib.oracle_check_ends.restype = u64
        lib.oracle_check_batch.argtypes = [ctypes.c_int, u8p, u64p, u64p, u64p, u64, u64, u64, u64, u64p]
        lib.oracle_check_batch.restype = u64
        _lib = lib
    return _lib


def _u8(a) -> np.ndarray:
    a = np.ascontiguousarray(np.frombuffer(a, dtype=np.uint8) if isinstance(a, (bytes, bytearray)) else a,
                             dtype=np.uint8)
    return a


def _p8(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))


def _p64(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def _check(w: int, max_size: int):
    if w < 1 or max_size <= w:
        raise ValueError(f"need window >= 1 and max_size > window (w={w}, max_size={max_size})")


def extreme_byte_search(region, mode: str = "max"):
    """§4.1: (value, leftmost position) of the max/min byte of a non-empty region."""
    r = _u8(region)
    if r.size == 0:
        raise ValueError("empty region")
    v = ctypes.c_uint8()
    p = ctypes.c_uint64()
    _load().oracle_extreme_byte_search(_p8(r), r.size, MODES[mode], ctypes.byref(v), ctypes.byref(p))
    return int(v.value), int(p.value)


def range_scan(region, target: int, cmp: str):
    """§4.2: index of the first byte b with (b cmp target), or None."""
    r = _u8(region)
    i = _load().oracle_range_scan(_p8(r), r.size, int(target), CMPS[cmp])
    return None if i == r.size else int(i)


def chunk_end(algo: str, data, s: int, w: int, max_size: int) -> int:
    d = _u8(data)
    _check(w, max_size)
    return int(_load().oracle_chunk_end(ALGOS[algo], _p8(d), d.size, s, w, max_size))


def max_chunks(n: int, w: int) -> int:
    return n // (w + 1) + 2


def chunk(algo: str, data, w: int, max_size: int) -> np.ndarray:
    """Whole-stream chunking: uint64 exclusive chunk end offsets (last = len)."""
    d = _u8(data)
    _check(w, max_size)
    cap = max_chunks(d.size, w)
    out = np.empty(cap, dtype=np.uint64)
    n = _load().oracle_chunk(ALGOS[algo], _p8(d), d.size, w, max_size, _p64(out), cap)
    return out[:n].copy()


def chain_from(algo: str, data, start: int, stop: int, w: int, max_size: int) -> np.ndarray:
    """Chunk starts of the chain begun at `start`, up to the first start >= stop."""
    d = _u8(data)
    _check(w, max_size)
    cap = max_chunks(max(0, min(d.size, stop) - start), w) + 2
    out = np.empty(cap, dtype=np.uint64)
    n = _load().oracle_chain_from(ALGOS[algo], _p8(d), d.size, start, stop, w, max_size, _p64(out), cap)
    return out[:n].copy()


def chunk_batch(algo: str, data, offsets, w: int, max_size: int):
    """Per-file chunking of a packed batch: (ends concatenated, per-file bound offsets)."""
    d = _u8(data)
    offsets = np.asarray(offsets, dtype=np.int64)
    outs = []
    bo = np.zeros(offsets.size, dtype=np.int64)
    for i in range(offsets.size - 1):
        e = chunk(algo, d[offsets[i]:offsets[i + 1]], w, max_size)
        outs.append(e)
        bo[i + 1] = bo[i] + e.size
    ends = np.concatenate(outs) if outs else np.zeros(0, dtype=np.uint64)
    return ends, bo


def _threads(threads):
    return max(1, threads if threads else (os.cpu_count() or 1))


def check_chunking(algo: str, data, ends, w: int, max_size: int, threads: int | None = None):
    """Check a chunking of `data` against the definition, every chunk: returns None
    when ``ends`` equals ``chunk(algo, data, w, max_size)``, else
    (index, expected end, got).  Each entry is checked as
    ends[j] == chunk_end(ends[j-1]) (ends[-1] read as 0), so the work splits
    over host threads (ctypes releases the GIL)."""
    d = _u8(data)
    _check(w, max_size)
    e = np.ascontiguousarray(ends, dtype=np.uint64)
    n, L = e.size, d.size
    if L == 0:
        return None if n == 0 else (0, None, int(e[0]))
    if n == 0:
        return (0, chunk_end(algo, d, 0, w, max_size), None)
    lib = _load()
    T = min(_threads(threads), max(1, n // 64))
    cuts = [n * t // T for t in range(T + 1)]

    def part(t):
        return int(lib.oracle_check_ends(ALGOS[algo], _p8(d), L, w, max_size, _p64(e), cuts[t], cuts[t + 1]))

    with ThreadPoolExecutor(T) as ex:
        bad = [j for t, j in enumerate(ex.map(part, range(T))) if j < cuts[t + 1]]
    if bad:
        j = min(bad)
        s = int(e[j - 1]) if j else 0
        return (j, chunk_end(algo, d, s, w, max_size) if s < L else None, int(e[j]))
    if int(e[-1]) != L:
        return (n, L, int(e[-1]))
    return None


def check_batch(algo: str, data, offsets, ends, bound_offsets, w: int, max_size: int,
                threads: int | None = None):
    """check_chunking for every file of a packed batch (file f: data[offsets[f]:offsets[f+1]],
    its ends relative to the file start in ends[bound_offsets[f]:bound_offsets[f+1]]).
    Returns None when every file's chunking equals the oracle's, else (file, entry index)."""
    d = _u8(data)
    _check(w, max_size)
    offs = np.ascontiguousarray(offsets, dtype=np.uint64)
    bo = np.ascontiguousarray(bound_offsets, dtype=np.uint64)
    e = np.ascontiguousarray(ends, dtype=np.uint64)
    nf = offs.size - 1
    if bo.size != offs.size or bo[0] != 0 or (np.diff(bo.astype(np.int64)) < 0).any() or int(bo[-1]) > e.size:
        return (-1, -1)
    if nf <= 0:
        return None
    lib = _load()
    T = min(_threads(threads), nf)
    # split the files into T ranges of about equal bytes
    cum = offs.astype(np.float64)
    cuts = [0] + [int(np.searchsorted(cum, cum[-1] * t / T)) for t in range(1, T)] + [nf]
    cuts = sorted(set(min(max(c, 0), nf) for c in cuts))

    def part(i):
        bj = ctypes.c_uint64(0)
        f = int(lib.oracle_check_batch(ALGOS[algo], _p8(d), _p64(offs), _p64(e), _p64(bo), cuts[i], cuts[i + 1],
                                       w, max_size, ctypes.byref(bj)))
        return (f, int(bj.value)) if f < cuts[i + 1] else None

    with ThreadPoolExecutor(len(cuts) - 1) as ex:
        bad = [r for r in ex.map(part, range(len(cuts) - 1)) if r is not None]
    return min(bad) if bad else None
