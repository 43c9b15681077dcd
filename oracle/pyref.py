"""Pure-Python reference loops (TEST INFRASTRUCTURE ONLY; small inputs).

Written in the single-pass formulation -- one forward scan per chunk keeping
the running extreme and its position -- which is how the AE algorithm cited by
PAPER.md §2.1.2 ([ae]) states it; the C oracle follows the paper's
target/window decomposition (§4.3).  Agreement of the two formulations on
exhaustive small inputs is one of the oracle's pins.
"""
from __future__ import annotations


def ram_chunk_end(d, s, w, max_size):
    """PAPER.md §2.1.2: window max, then first byte >= max after it."""
    L = len(d)
    limit = min(L, s + max_size)
    if s + w >= L:
        return L
    m = -1
    for i in range(s, s + w):
        if d[i] > m:
            m = d[i]
    for i in range(s + w, limit):
        if d[i] >= m:
            return i + 1
    return limit


def ae_chunk_end(d, s, w, max_size, mode="max"):
    """PAPER.md §2.1.2 lines 169-171 in single-pass form.

    Keep the current target (running strict extreme) and its position; a byte
    beating the target becomes the new target; when the scan reaches the last
    byte of the target's window (position + w) with the target unbeaten, the
    chunk ends there.
    """
    L = len(d)
    limit = min(L, s + max_size)
    ext, pos = d[s], s
    for i in range(s + 1, limit):
        beats = d[i] > ext if mode == "max" else d[i] < ext
        if beats:
            ext, pos = d[i], i
        elif i == pos + w:
            return i + 1
    return limit


def maxp_chunk_end(d, s, h, max_size):
    """PAPER.md §2.1.2, as written there: two h-byte windows one byte
    apart slide over the chunk; the target byte between them ends the chunk
    when it is greater than the maximum of both windows (Python max over the
    two slices, not the C oracle's early-exit loop)."""
    L = len(d)
    limit = min(L, s + max_size)
    for t in range(s + h, limit):
        if t + h >= L:
            break
        if d[t] > max(d[t - h:t]) and d[t] > max(d[t + 1:t + h + 1]):
            return t + 1
    return limit


def chunk_end(algo, d, s, w, max_size):
    if algo == "maxp":
        return maxp_chunk_end(d, s, w, max_size)
    if algo == "ram":
        return ram_chunk_end(d, s, w, max_size)
    return ae_chunk_end(d, s, w, max_size, "max" if algo == "ae_max" else "min")


def chunk(algo, d, w, max_size):
    out, s = [], 0
    while s < len(d):
        s = chunk_end(algo, d, s, w, max_size)
        out.append(s)
    return out
