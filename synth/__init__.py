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
  BASELINE configs[1] (s = 1.1, seed 1).
* ``versioned(base_size, n_snap, seed)`` -- a uniform base with 10% of its
  64 KiB regions zero-filled, plus snapshots each derived from the previous by
  insert/delete/overwrite runs of 1..4 KiB touching ~1% of its bytes
  (BASELINE configs[2]).
* ``file_sizes / many_files`` -- lognormal sizes (median 64 KiB, sigma 1.5,
  capped at 16 MiB), 70% uniform / 30% Zipf content (BASELINE configs[3]).
* ``alternating(n, region, seed)`` -- alternating regions of uniform bytes and
  low-entropy bytes (runs of one repeated value, run length geometric with mean
  512) (BASELINE configs[4]).

These stand in for the paper's datasets (Table 2), which are not
available here; no item of any real dataset is reproduced.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "uniform",
    "zipf_bytes",
    "versioned",
    "file_sizes",
    "many_files",
    "alternating",
    "constant",
]

_CHUNK = 1 << 24  # generate in 16 MiB pieces to bound temporary memory


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def uniform(n: int, seed: int) -> np.ndarray:
    """n i.i.d. uniform bytes."""
    return _rng(seed).integers(0, 256, size=n, dtype=np.uint8)


def constant(n: int, value: int) -> np.ndarray:
    return np.full(n, value, dtype=np.uint8)


def _zipf_table(s: float, rng: np.random.Generator):
    ranks = np.arange(1, 257, dtype=np.float64)
    p = ranks ** (-s)
    p /= p.sum()
    perm = rng.permutation(256).astype(np.uint8)  # rank-1 -> byte value
    return np.cumsum(p), perm


def zipf_bytes(n: int, s: float = 1.1, seed: int = 1, rng: np.random.Generator | None = None) -> np.ndarray:
    """n i.i.d. Zipf(s)-ranked bytes (rank -> value through a seeded permutation)."""
    rng = _rng(seed) if rng is None else rng
    cdf, perm = _zipf_table(s, rng)
    cdf[-1] = 1.0
    out = np.empty(n, dtype=np.uint8)
    for lo in range(0, n, _CHUNK):
        hi = min(n, lo + _CHUNK)
        u = rng.random(hi - lo)
        idx = np.searchsorted(cdf, u, side="right")
        np.minimum(idx, 255, out=idx)
        out[lo:hi] = perm[idx]
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


def versioned(base_size: int, n_snap: int, seed: int = 2, region: int = 64 << 10,
              zero_frac: float = 0.10, edit_frac: float = 0.01,
              run_lo: int = 1024, run_hi: int = 4096) -> list[np.ndarray]:
    """Backup-like versioned data: [base, snap1, ..., snap_n_snap]."""
    rng = _rng(seed)
    base = rng.integers(0, 256, size=base_size, dtype=np.uint8)
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


def many_files(n_files: int, seed: int = 3, median: int = 64 << 10, sigma: float = 1.5,
               cap: int = 16 << 20, uniform_frac: float = 0.7, zipf_s: float = 1.1):
    """Packed many-file batch: returns (data uint8[total], offsets int64[n_files+1]).

    File kinds are drawn per file (uniform with probability uniform_frac, else
    Zipf-skewed); the bytes of all uniform files come from one uniform draw and
    those of all Zipf files from one Zipf draw, split in file order."""
    sizes = file_sizes(n_files, seed, median, sigma, cap)
    rng = _rng(seed + 1000)
    offsets = np.zeros(n_files + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    kinds = rng.random(n_files) < uniform_frac
    u = rng.integers(0, 256, size=int(sizes[kinds].sum()), dtype=np.uint8)
    z = zipf_bytes(int(sizes[~kinds].sum()), zipf_s, rng=rng)
    ui = np.split(u, np.cumsum(sizes[kinds])[:-1]) if kinds.any() else []
    zi = np.split(z, np.cumsum(sizes[~kinds])[:-1]) if (~kinds).any() else []
    pieces, a, b = [], 0, 0
    for k in kinds.tolist():
        if k:
            pieces.append(ui[a])
            a += 1
        else:
            pieces.append(zi[b])
            b += 1
    data = np.concatenate(pieces) if pieces else np.zeros(0, dtype=np.uint8)
    return data, offsets


def alternating(n: int, region: int = 256 << 20, seed: int = 5, mean_run: float = 512.0) -> np.ndarray:
    """Alternating regions: uniform random, then runs of repeated values (geometric lengths)."""
    rng = _rng(seed)
    out = np.empty(n, dtype=np.uint8)
    k = 0
    for lo in range(0, n, region):
        hi = min(n, lo + region)
        if k % 2 == 0:
            out[lo:hi] = rng.integers(0, 256, size=hi - lo, dtype=np.uint8)
        else:
            m = hi - lo
            n_runs = int(m / mean_run * 1.2) + 16
            lens = rng.geometric(1.0 / mean_run, size=n_runs)
            while lens.sum() < m:
                lens = np.concatenate([lens, rng.geometric(1.0 / mean_run, size=n_runs)])
            vals = rng.integers(0, 256, size=lens.size, dtype=np.uint8)
            seg = np.repeat(vals, lens)[:m]
            out[lo:hi] = seg
        k += 1
    return out
