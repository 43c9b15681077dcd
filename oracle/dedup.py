"""Deduplication space savings, §2.2.1 Eq. (1) (TEST INFRASTRUCTURE ONLY).

    Space Savings (%) = (Original Data Size - Deduplicated Data Size)
                        / Original Data Size * 100

The deduplicated size is the total length of the distinct chunks, distinctness
being exact chunk-content equality (no fingerprint, so no collision can occur).
"""
from __future__ import annotations

import numpy as np


def unique_bytes(streams, ends_list) -> tuple[int, int]:
    """(original bytes, deduplicated bytes) over several chunked streams."""
    seen = set()
    total = 0
    uniq = 0
    for data, ends in zip(streams, ends_list):
        buf = np.ascontiguousarray(data, dtype=np.uint8).tobytes()
        s = 0
        for e in np.asarray(ends).tolist():
            piece = buf[s:e]
            total += e - s
            if piece not in seen:
                seen.add(piece)
                uniq += e - s
            s = e
    return total, uniq


def space_savings(total: int, uniq: int) -> float:
    if total <= 0:
        raise ValueError("empty corpus")
    return 100.0 * (total - uniq) / total
