"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and bench.py.

This module holds NO chunking arithmetic: it only draws bytes.  Both sides of a
parity test (the CPU oracle under ``oracle/`` and the CUDA path under
``paper_2508_05797_b200/``) receive the exact same numpy arrays from here.

Recipes (stated again in DESIGN.md §3, "input recipe"):

* ``uniform(n, seed)``        -- i.i.d. uniform bytes (BASELINE configs[0], [2] base).
* ``zipf_bytes(n, s, seed)``  -- i.i.d. bytes whose *rank* r in 1..256 has
  P(r) ∝ r^-s; ranks are mapped to byte values through a seeded permutation of
  0..255 (text-like skew without favouring any particular byte value).
  Drawn with Walker's alias method (one uniform index and one 32-bit
  threshold test per byte).  BASELINE configs[1] (s = 1.1, seed 1).
* ``versioned(base_size, n_snap, seed)`` -- a uniform base with 10% of its
  64 KiB regions zero-filled, plus snapshots each derived from the previous by
  insert/delete/overwrite runs of 1..4 KiB touching ~1% of its bytes
  (BASELINE configs[2]).
* ``file_sizes / many_files`` -- lognormal sizes (median 64 KiB, sigma 1.5,
  capped at 16 MiB), 70% uniform / 30% Zipf content (BASELINE configs[3]).
* ``alternating(n, region, seed)`` -- alternating regions of uniform bytes and
  low-entropy bytes (runs of one repeated value, run length geometric with mean
  512) (BASELINE configs[4]).

Large outputs are generated in 16 MiB pieces, piece k from its own PCG64
stream seeded by (seed, k), on a thread pool: the bytes depend only on the
seed and the size, never on the number of threads.

These stand in for the paper's datasets (Table 2), which are not
available here; no item of any real dataset is reproduced.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

__all__ = [
    "uniform",
    "zipf_bytes",
    "patchwork",
    "versioned",
    "file_sizes",
    "many_files",
    "many_files_offsets",
    "alternating",
    "constant",
    "saturation_edges",
]

PIECE = 1 << 24  # bytes per independently seeded piece


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _piece_rng(seed: int, k: int, tag: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, tag, k])))


def _threads() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def _pieces(n: int, fn) -> None:
    """Run fn(k, lo, hi) over the 16 MiB pieces of [0, n) on a thread pool."""
    ks = range((n + PIECE - 1) // PIECE)
    if len(ks) <= 1:
        for k in ks:
            fn(k, 0, n)
        return
    with ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(lambda k: fn(k, k * PIECE, min(n, (k + 1) * PIECE)), ks))


def uniform(n: int, seed: int) -> np.ndarray:
    """n i.i.d. uniform bytes."""
    out = np.empty(n, dtype=np.uint8)

    def fill(k, lo, hi):
        out[lo:hi] = _piece_rng(seed, k, 1).integers(0, 256, size=hi - lo, dtype=np.uint8)

    _pieces(n, fill)
    return out


def constant(n: int, value: int) -> np.ndarray:
    return np.full(n, value, dtype=np.uint8)


class _Zipf:
    """Alias table of the Zipf(s) rank distribution over 256 values, ranks mapped
    to byte values through a permutation drawn from `seed`."""

    def __init__(self, s: float, seed: int):
        ranks = np.arange(1, 257, dtype=np.float64)
        p = ranks ** (-s)
        p /= p.sum()
        self.perm = _rng(seed).permutation(256).astype(np.uint8)  # rank-1 -> byte value
        # Walker/Vose alias table: column i keeps rank i with probability q[i],
        # else yields alias[i]
        q = p * 256.0
        alias = np.arange(256)
        small = [i for i in range(256) if q[i] < 1.0]
        large = [i for i in range(256) if q[i] >= 1.0]
        while small and large:
            a, b = small.pop(), large.pop()
            alias[a] = b
            q[b] -= 1.0 - q[a]
            (small if q[b] < 1.0 else large).append(b)
        for i in small + large:
            q[i] = 1.0
        self.thr = np.minimum(np.round(q * 2.0 ** 32), 2.0 ** 32).astype(np.uint64)
        self.val_keep = self.perm
        self.val_alias = self.perm[alias]

    def draw(self, rng: np.random.Generator, m: int) -> np.ndarray:
        col = rng.integers(0, 256, size=m, dtype=np.uint8)
        u = rng.integers(0, 1 << 32, size=m, dtype=np.uint32)
        keep = u.astype(np.uint64) < self.thr[col]
        return np.where(keep, self.val_keep[col], self.val_alias[col])


def zipf_bytes(n: int, s: float = 1.1, seed: int = 1) -> np.ndarray:
    """n i.i.d. Zipf(s)-ranked bytes (rank -> value through a seeded permutation)."""
    z = _Zipf(s, seed)
    out = np.empty(n, dtype=np.uint8)

    def fill(k, lo, hi):
        out[lo:hi] = z.draw(_piece_rng(seed, k, 2), hi - lo)

    _pieces(n, fill)
    return out


def saturation_edges(n: int, seed: int = 6, p: float = 1 / 700) -> np.ndarray:
    """Bytes near both ends of the range: 255 and 0 each with probability p, the
    rest from {1, 2, 253, 254}; half the bytes after a 255 are 254 and half
    after a 0 are 1.  Exercises saturating extremes next to near-saturating
    ones (test data for the kernels' saturation scan; no chunking logic)."""
    rng = _rng(seed)
    out = rng.choice(np.array([1, 2, 253, 254], dtype=np.uint8), size=n)
    u = rng.random(n)
    out[u < p] = 255
    out[(u >= p) & (u < 2 * p)] = 0
    if n > 1:
        nxt = rng.random(n - 1) < 0.5
        out[1:][(out[:-1] == 255) & nxt] = 254
        out[1:][(out[:-1] == 0) & nxt] = 1
    return out


def patchwork(n: int, seed: int = 11, piece_lo: int = 2048, piece_hi: int = 65536) -> np.ndarray:
    """Pieces of random lengths in [piece_lo, piece_hi) drawn from different
    kinds of bytes: uniform, Zipf(1.1) with the seed-1 permutation (0xFF is its
    rarest value), constant 0x00, constant 0xFF, uniform over 0..199 (no 0xFF),
    uniform over 56..255 (no 0x00), and saturation edges.  Streams that are
    saturated only in stretches, switching often (test data; no chunking logic)."""
    rng = _rng(seed)
    z = _Zipf(1.1, 1)
    out = np.empty(n, dtype=np.uint8)
    x = 0
    while x < n:
        m = min(n - x, int(rng.integers(piece_lo, piece_hi)))
        k = int(rng.integers(0, 7))
        if k == 0:
            v = rng.integers(0, 256, m, dtype=np.uint8)
        elif k == 1:
            v = z.draw(rng, m)
        elif k == 2:
            v = np.zeros(m, dtype=np.uint8)
        elif k == 3:
            v = np.full(m, 255, dtype=np.uint8)
        elif k == 4:
            v = rng.integers(0, 200, m, dtype=np.uint8)
        elif k == 5:
            v = rng.integers(56, 256, m, dtype=np.uint8)
        else:
            v = saturation_edges(m, int(rng.integers(0, 1 << 30)), p=1 / 300)
        out[x:x + m] = v
        x += m
    return out


def versioned(base_size: int, n_snap: int, seed: int = 2, region: int = 64 << 10,
              zero_frac: float = 0.10, edit_frac: float = 0.01,
              run_lo: int = 1024, run_hi: int = 4096) -> list[np.ndarray]:
    """Backup-like versioned data: [base, snap1, ..., snap_n_snap]."""
    rng = _rng(seed)
    base = uniform(base_size, seed)
    n_regions = (base_size + region - 1) // region
    zero = rng.random(n_regions) < zero_frac
    for r in np.nonzero(zero)[0]:
        base[r * region:(r + 1) * region] = 0
    snaps = [base]
    cur = base
    mean_run = (run_lo + run_hi) / 2.0
    for _ in range(n_snap):
        n_edits = max(1, int(round(edit_frac * cur.size / mean_run)))
        pos = np.sort(rng.integers(0, max(1, cur.size), size=n_edits))
        kinds = rng.integers(0, 3, size=n_edits)      # 0 insert, 1 delete, 2 overwrite
        runs = rng.integers(run_lo, run_hi + 1, size=n_edits)
        pieces = []
        prev = 0
        for p, k, r in zip(pos.tolist(), kinds.tolist(), runs.tolist()):
            if p < prev:
                continue
            pieces.append(cur[prev:p])
            if k == 0:
                pieces.append(rng.integers(0, 256, size=r, dtype=np.uint8))
                prev = p
            elif k == 1:
                prev = min(cur.size, p + r)
            else:
                end = min(cur.size, p + r)
                pieces.append(rng.integers(0, 256, size=end - p, dtype=np.uint8))
                prev = end
        pieces.append(cur[prev:])
        cur = np.concatenate(pieces)
        snaps.append(cur)
    return snaps


def file_sizes(n_files: int, seed: int = 3, median: int = 64 << 10, sigma: float = 1.5,
               cap: int = 16 << 20) -> np.ndarray:
    rng = _rng(seed)
    sz = np.exp(np.log(median) + sigma * rng.standard_normal(n_files))
    sz = np.clip(np.round(sz), 1, cap).astype(np.int64)
    return sz


def many_files_offsets(n_files: int, seed: int = 3, median: int = 64 << 10, sigma: float = 1.5,
                       cap: int = 16 << 20) -> np.ndarray:
    """File offsets int64[n_files+1] of many_files' packed batch (no bytes drawn)."""
    sizes = file_sizes(n_files, seed, median, sigma, cap)
    offsets = np.zeros(n_files + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    return offsets


def many_files(n_files: int, seed: int = 3, median: int = 64 << 10, sigma: float = 1.5,
               cap: int = 16 << 20, uniform_frac: float = 0.7, zipf_s: float = 1.1, files=None):
    """Packed many-file batch: returns (data uint8[total], offsets int64[n_files+1]).

    File kinds are drawn per file (uniform with probability uniform_frac, else
    Zipf-skewed).  The packed bytes are generated piece by piece: inside piece
    k, each file's part is drawn from piece k's generator with its file's kind.
    files=(f0, f1) returns only files [f0, f1) -- the same bytes as the slice of
    the whole batch -- with offsets relative to file f0 (a rank's share)."""
    offsets = many_files_offsets(n_files, seed, median, sigma, cap)
    kinds = _rng(seed + 1000).random(n_files) < uniform_frac  # True: uniform
    f0, f1 = (0, n_files) if files is None else files
    lo0, hi0 = int(offsets[f0]), int(offsets[f1])
    z = _Zipf(zipf_s, seed + 2000)
    out = np.empty(hi0 - lo0, dtype=np.uint8)

    def fill(k, lo, hi):
        # piece k of the whole batch covers [k PIECE, (k+1) PIECE); draw it from
        # its start so that a slice equals the whole batch's bytes
        rng = _piece_rng(seed, k, 3)
        f = int(np.searchsorted(offsets, lo, side="right")) - 1
        x = lo
        while x < hi:
            e = min(hi, int(offsets[f + 1]))
            if e > x:
                if kinds[f]:
                    v = rng.integers(0, 256, size=e - x, dtype=np.uint8)
                else:
                    v = z.draw(rng, e - x)
                a, b = max(x, lo0), min(e, hi0)
                if a < b:
                    out[a - lo0:b - lo0] = v[a - x:b - x]
            x = e
            f += 1

    k0, k1 = lo0 // PIECE, (hi0 + PIECE - 1) // PIECE
    total = int(offsets[-1])
    with ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(lambda k: fill(k, k * PIECE, min(total, (k + 1) * PIECE)), range(k0, k1)))
    return out, offsets[f0:f1 + 1] - lo0


def alternating(n: int, region: int = 256 << 20, seed: int = 5, mean_run: float = 512.0,
                part=None) -> np.ndarray:
    """Alternating regions: uniform random, then runs of repeated values (geometric lengths).
    part=(lo, hi) returns only bytes [lo, hi) of the n-byte stream (a rank's range + halo)."""
    lo0, hi0 = (0, n) if part is None else part
    out = np.empty(hi0 - lo0, dtype=np.uint8)

    def fill_region(k):
        lo, hi = k * region, min(n, (k + 1) * region)
        rng = _piece_rng(seed, k, 4)
        if k % 2 == 0:
            v = rng.integers(0, 256, size=hi - lo, dtype=np.uint8)
        else:
            m = hi - lo
            n_runs = int(m / mean_run * 1.2) + 16
            lens = rng.geometric(1.0 / mean_run, size=n_runs)
            while lens.sum() < m:
                lens = np.concatenate([lens, rng.geometric(1.0 / mean_run, size=n_runs)])
            vals = rng.integers(0, 256, size=lens.size, dtype=np.uint8)
            v = np.repeat(vals, lens)[:m]
        a, b = max(lo, lo0), min(hi, hi0)
        out[a - lo0:b - lo0] = v[a - lo:b - lo]

    ks = range(lo0 // region, (hi0 + region - 1) // region)
    with ThreadPoolExecutor(_threads()) as ex:
        list(ex.map(fill_region, ks))
    return out
