"""Pins of the CPU oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a fixture built from the
paper's text (tests/golden/), a closed form, a brute-force evaluation of the
boundary predicate written from the paper's definition, an independent
single-pass formulation (oracle/pyref.py), a library routine the operation
reduces to, or a statistical closed form.
"""
import glob
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import dedup, pyref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
ALGOS = ["ram", "ae_max", "ae_min"]


# --------------------------------------------------------------------------
# golden fixtures from the paper's text
# --------------------------------------------------------------------------
@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLDEN, "*.json"))))
def test_golden(path):
    g = json.load(open(path))
    data = bytes.fromhex(g["input_hex"])
    if g["op"] == "extreme_byte_search":
        assert oracle.extreme_byte_search(data, g["mode"]) == (g["expected"]["value"], g["expected"]["pos"])
    elif g["op"] == "range_scan":
        assert oracle.range_scan(data, g["target"], g["cmp"]) == g["expected"]
    else:
        ends = oracle.chunk(g["algo"], data, g["w"], g["max_size"]).tolist()
        assert ends == g["expected_ends"]
        assert pyref.chunk(g["algo"], list(data), g["w"], g["max_size"]) == g["expected_ends"]


# --------------------------------------------------------------------------
# primitives reduce to library routines
# --------------------------------------------------------------------------
def test_ebs_is_argmax_argmin():
    rng = np.random.default_rng(0)
    for n in [1, 2, 15, 16, 17, 63, 64, 65, 4096, 8191]:
        r = rng.integers(0, 256, n, dtype=np.uint8)
        assert oracle.extreme_byte_search(r, "max") == (int(r.max()), int(np.argmax(r)))
        assert oracle.extreme_byte_search(r, "min") == (int(r.min()), int(np.argmin(r)))
    z = np.zeros(4096, np.uint8)
    assert oracle.extreme_byte_search(z, "max") == (0, 0)  # leftmost tie-break
    with pytest.raises(ValueError):
        oracle.extreme_byte_search(np.zeros(0, np.uint8))


@pytest.mark.parametrize("cmp,fn", [("gt", np.greater), ("geq", np.greater_equal), ("lt", np.less),
                                    ("leq", np.less_equal), ("eq", np.equal)])
def test_range_scan_is_first_nonzero(cmp, fn):
    rng = np.random.default_rng(1)
    for n in [0, 1, 31, 32, 33, 1000]:
        r = rng.integers(0, 256, n, dtype=np.uint8)
        for t in [0, 1, 127, 128, 200, 254, 255]:
            hits = np.nonzero(fn(r, np.uint8(t)))[0]
            exp = int(hits[0]) if hits.size else None
            assert oracle.range_scan(r, t, cmp) == exp


# --------------------------------------------------------------------------
# closed forms
# --------------------------------------------------------------------------
def _lens(ends):
    e = np.asarray(ends, dtype=np.int64)
    return np.diff(np.concatenate([[0], e]))


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("value", [0, 1, 128, 255])
def test_constant_stream_chunks_are_w_plus_1(algo, value):
    # constant data: RAM max = v and the first post-window byte is >= v;
    # AE: the first byte is the target and no window byte exceeds it.
    w, L = 37, 1000
    ends = oracle.chunk(algo, synth.constant(L, value), w, 4 * w)
    lens = _lens(ends)
    assert (lens[:-1] == w + 1).all() and 1 <= lens[-1] <= w + 1
    assert lens.size == -(-L // (w + 1))


def test_monotone_streams():
    w, mx = 5, 23
    inc = np.arange(200, dtype=np.uint8)
    dec = inc[::-1].copy()
    # increasing: RAM window max d[s+w-1] < d[s+w] -> w+1; AE-Max: every byte
    # beats the target -> only the cap ends chunks; AE-Min: first byte wins -> w+1
    assert (_lens(oracle.chunk("ram", inc, w, mx))[:-1] == w + 1).all()
    assert (_lens(oracle.chunk("ae_max", inc, w, mx))[:-1] == mx).all()
    assert (_lens(oracle.chunk("ae_min", inc, w, mx))[:-1] == w + 1).all()
    # decreasing: mirror images
    assert (_lens(oracle.chunk("ram", dec, w, mx))[:-1] == mx).all()
    assert (_lens(oracle.chunk("ae_max", dec, w, mx))[:-1] == w + 1).all()
    assert (_lens(oracle.chunk("ae_min", dec, w, mx))[:-1] == mx).all()


def test_degenerate_streams():
    for algo in ALGOS:
        assert oracle.chunk(algo, np.zeros(0, np.uint8), 4, 16).tolist() == []
        assert oracle.chunk(algo, np.array([7], np.uint8), 4, 16).tolist() == [1]
        # shorter than the window + 1: one final chunk
        assert oracle.chunk(algo, np.arange(4, dtype=np.uint8), 4, 16).tolist() == [4]
    with pytest.raises(ValueError):
        oracle.chunk("ram", np.zeros(10, np.uint8), 4, 4)


# --------------------------------------------------------------------------
# brute-force predicate enumeration (definition written independently)
# --------------------------------------------------------------------------
def _bf_chunk_end(algo, d, s, w, max_size):
    """Smallest valid end e, by checking the paper's boundary predicate for
    every candidate e with Python slicing; else the cap / end of stream."""
    L = len(d)
    limit = min(L, s + max_size)
    for e in range(s + 1, limit + 1):
        b = e - 1  # boundary byte = last byte of the chunk
        if algo == "ram":
            # b lies outside the window and is >= the window's maximum (Fig. 2c);
            # the first such b is taken (min over e)
            if b >= s + w and s + w <= L and d[b] >= max(d[s:s + w]):
                return e
        else:
            t = b - w  # the target whose window (t, t+w] ends at b
            if t < s:
                continue
            before = d[s:t]
            win = d[t + 1:t + w + 1]
            if algo == "ae_max":
                is_target = all(x < d[t] for x in before)
                wins = d[t] >= max(win)
            else:
                is_target = all(x > d[t] for x in before)
                wins = d[t] <= min(win)
            if is_target and wins:
                return e
    return limit


def _bf_chunk(algo, d, w, max_size):
    out, s = [], 0
    while s < len(d):
        s = _bf_chunk_end(algo, d, s, w, max_size)
        out.append(s)
    return out


@pytest.mark.parametrize("algo", ALGOS)
def test_exhaustive_small_alphabet(algo):
    alphabet = [0, 1, 2]
    count = 0
    for n in range(1, 8):
        for tup in itertools.product(alphabet, repeat=n):
            d = list(tup)
            arr = np.array(d, dtype=np.uint8)
            for w in (1, 2, 3):
                for mx in (w + 1, w + 2, 6):
                    exp = _bf_chunk(algo, d, w, mx)
                    assert oracle.chunk(algo, arr, w, mx).tolist() == exp, (d, w, mx)
                    assert pyref.chunk(algo, d, w, mx) == exp
                    count += 1
    assert count > 10000


@pytest.mark.parametrize("algo", ALGOS)
def test_random_vs_bruteforce_and_pyref(algo):
    rng = np.random.default_rng(7)
    for trial in range(40):
        n = int(rng.integers(1, 400))
        hi = int(rng.choice([2, 4, 16, 256]))
        d = rng.integers(0, hi, n).astype(np.uint8)
        w = int(rng.integers(1, 24))
        mx = int(w + 1 + rng.integers(0, 60))
        exp = _bf_chunk(algo, d.tolist(), w, mx)
        assert oracle.chunk(algo, d, w, mx).tolist() == exp
        assert pyref.chunk(algo, d.tolist(), w, mx) == exp


# --------------------------------------------------------------------------
# invariants on realistic sizes
# --------------------------------------------------------------------------
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("gen", ["uniform", "zipf"])
def test_invariants(algo, gen):
    L = 1 << 20
    d = synth.uniform(L, 11) if gen == "uniform" else synth.zipf_bytes(L, 1.1, 12)
    w, mx = 512, 4096
    ends = oracle.chunk(algo, d, w, mx)
    lens = _lens(ends)
    assert int(ends[-1]) == L and (lens > 0).all()               # chunks tile the input
    assert (lens[:-1] >= w + 1).all() and (lens <= mx).all()     # implicit min, cap
    # boundary property for content (non-cap) boundaries
    s = 0
    for e in ends[:-1].tolist():
        if e - s < mx:
            b = e - 1
            if algo == "ram":
                M = d[s:s + w].max()
                assert d[b] >= M and (d[s + w:b] < M).all()
            else:
                t = b - w
                if algo == "ae_max":
                    assert (d[s:t] < d[t]).all() and d[t] >= d[t + 1:b + 1].max()
                else:
                    assert (d[s:t] > d[t]).all() and d[t] <= d[t + 1:b + 1].min()
        s = e


@pytest.mark.parametrize("algo", ALGOS)
def test_content_defined_resync(algo):
    """A prefix insertion shifts later boundaries by the insertion length."""
    L = 1 << 19
    d = synth.uniform(L, 21)
    w, mx = 256, 2048
    base = oracle.chunk(algo, d, w, mx)
    ins = synth.uniform(777, 22)
    d2 = np.concatenate([ins, d])
    e2 = oracle.chunk(algo, d2, w, mx).astype(np.int64)
    shifted = e2[e2 > 777] - 777
    base = base.astype(np.int64)
    common = np.intersect1d(base, shifted)
    # after re-synchronisation every later boundary coincides
    first = common[0]
    assert (base[base >= first] == shifted[shifted >= first]).all()
    assert first < 64 * mx


def test_chain_from_matches_chunk():
    d = synth.uniform(200000, 3)
    for algo in ALGOS:
        ends = oracle.chunk(algo, d, 300, 3000)
        ch = oracle.chain_from(algo, d, 0, len(d), 300, 3000)
        assert ch.tolist() == [0] + ends.tolist()


# --------------------------------------------------------------------------
# statistical closed form (RAM on uniform bytes)
# --------------------------------------------------------------------------
def test_ram_mean_chunk_length_closed_form():
    """On i.i.d. uniform bytes the window max M of w bytes has
    P(M <= m) = ((m+1)/256)^w, and the scan after the window is geometric with
    success probability (256-M)/256, so E[len] = w + sum_M P(M) * 256/(256-M)
    (no cap).  A GT instead of GEQ comparator, or a window of the wrong length,
    moves the mean by far more than the sampling error."""
    w = 100
    L = 6 << 20
    d = synth.uniform(L, 5)
    lens = _lens(oracle.chunk("ram", d, w, 1 << 40))[:-1]
    pm = np.array([((m + 1) / 256) ** w - (m / 256) ** w for m in range(256)])
    expect = w + float(sum(pm[m] * 256.0 / (256 - m) for m in range(256)))
    se = lens.std() / math.sqrt(lens.size)
    assert abs(lens.mean() - expect) < 4 * se, (lens.mean(), expect, se)


# --------------------------------------------------------------------------
# dedup space savings, Eq. (1)
# --------------------------------------------------------------------------
def test_space_savings_closed_forms():
    assert dedup.space_savings(100, 100) == 0.0
    assert dedup.space_savings(200, 100) == 50.0
    with pytest.raises(ValueError):
        dedup.space_savings(0, 0)
    x = synth.uniform(1 << 20, 9)
    xx = np.concatenate([x, x])
    w, mx = 1000, 16000
    ends = oracle.chunk("ram", xx, w, mx)
    total, uniq = dedup.unique_bytes([xx], [ends])
    assert total == xx.size
    s = dedup.space_savings(total, uniq)
    assert 49.0 <= s <= 50.0
    # disjoint random data: no duplicate chunks
    y = synth.uniform(1 << 20, 10)
    t2, u2 = dedup.unique_bytes([x, y], [oracle.chunk("ram", x, w, mx), oracle.chunk("ram", y, w, mx)])
    assert t2 == u2


# --------------------------------------------------------------------------
# chain_from at interior (start, stop), against the brute-force predicate
# --------------------------------------------------------------------------
def _bf_chain(algo, d, start, stop, w, mx):
    """Every chunk start of the chain begun at `start`, up to the first >= stop (or len)."""
    out, s = [start], start
    while s < stop and s < len(d):
        s = _bf_chunk_end(algo, d, s, w, mx)
        out.append(s)
    return out


@pytest.mark.parametrize("algo", ALGOS)
def test_chain_from_interior_vs_bruteforce(algo):
    rng = np.random.default_rng(17)
    for trial in range(60):
        n = int(rng.integers(1, 300))
        d = rng.integers(0, int(rng.choice([3, 16, 256])), n).astype(np.uint8)
        w = int(rng.integers(1, 12))
        mx = int(w + 1 + rng.integers(0, 30))
        start = int(rng.integers(0, n + 1))
        stop = int(rng.integers(start, n + 8))
        exp = _bf_chain(algo, d.tolist(), start, stop, w, mx)
        assert oracle.chain_from(algo, d, start, stop, w, mx).tolist() == exp, (n, w, mx, start, stop)


# --------------------------------------------------------------------------
# the verifiers used at full size: check_chunking / check_batch
# --------------------------------------------------------------------------
def _mutations(ends, L):
    """Plausible mistakes of a chunker: a boundary moved by one, a dropped or
    duplicated boundary, a spurious split, a truncated or extended stream end."""
    e = [int(x) for x in ends]
    out = []
    if len(e) >= 2:
        i = len(e) // 2
        out.append(e[:i] + [e[i] + 1] + e[i + 1:])
        out.append(e[:i] + [e[i] - 1] + e[i + 1:])
        out.append(e[:i] + e[i + 1:])                           # dropped
        out.append(e[:i] + [e[i], e[i]] + e[i + 1:])            # duplicated
        s = e[i - 1] if i else 0
        out.append(e[:i] + [s + (e[i] - s) // 2] + e[i:])       # spurious split
        out.append(e[:-1])                                      # truncated
    out.append(e + [L + 1])                                     # past the end
    out.append([x + 1 for x in e[:1]] + e[1:])                  # first boundary moved
    return out


@pytest.mark.parametrize("algo", ALGOS)
def test_check_chunking_accepts_oracle_and_rejects_mutations(algo):
    for gen, w, mx in (("uniform", 300, 3000), ("zipf", 1000, 8000), ("runs", 64, 600)):
        L = 300_001
        d = {"uniform": lambda: synth.uniform(L, 31), "zipf": lambda: synth.zipf_bytes(L, 1.1, 32),
             "runs": lambda: np.repeat(synth.uniform(L // 50 + 1, 33), 50)[:L]}[gen]()
        ends = oracle.chunk(algo, d, w, mx)
        assert oracle.check_chunking(algo, d, ends, w, mx, threads=4) is None
        for bad in _mutations(ends, L):
            assert oracle.check_chunking(algo, d, np.array(bad, dtype=np.uint64), w, mx, threads=3) is not None
    # empty stream, empty output
    assert oracle.check_chunking(algo, np.zeros(0, np.uint8), np.zeros(0, np.uint64), 4, 16) is None
    assert oracle.check_chunking(algo, np.zeros(10, np.uint8), np.zeros(0, np.uint64), 4, 16) is not None


@pytest.mark.parametrize("algo", ALGOS)
def test_check_batch_accepts_oracle_and_rejects_mutations(algo):
    data, offs = synth.many_files(300, seed=41, median=6000, sigma=1.2, cap=60000)
    sizes = np.diff(offs)
    sizes[[3, 50, 299]] = 0  # empty files (the byte ranges are re-packed below)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    data = data[:offs[-1]]
    w, mx = 500, 4000
    ends, bo = oracle.chunk_batch(algo, data, offs, w, mx)
    assert oracle.check_batch(algo, data, offs, ends, bo, w, mx, threads=5) is None
    for f in (0, 1, 137, 298):
        a, b = int(bo[f]), int(bo[f + 1])
        for bad in _mutations(ends[a:b], int(sizes[f])):
            e2 = np.concatenate([ends[:a], np.array(bad, dtype=np.uint64), ends[b:]])
            bo2 = bo.copy()
            bo2[f + 1:] += len(bad) - (b - a)
            r = oracle.check_batch(algo, data, offs, e2, bo2, w, mx, threads=4)
            assert r is not None and r[0] == f, (f, r)
    # a non-monotone bound-offset table is rejected
    bo3 = bo.copy()
    bo3[10], bo3[11] = bo3[11], bo3[10]
    if bo3[10] != bo3[11]:
        assert oracle.check_batch(algo, data, offs, ends, bo3, w, mx) is not None



# --------------------------------------------------------------------------
# MAXP (§2.1.2 l.173 and l.196, §4.3 l.361; readings M1-M4)
# --------------------------------------------------------------------------
def _bf_maxp_chunk(d, h, max_size):
    """Brute force from the definition with Python all(): the chunk from s ends
    right after the first t in [s+h, limit) whose h bytes before and h bytes
    after all lie in the stream and are all smaller than d[t]."""
    L, out, s = len(d), [], 0
    while s < L:
        limit = min(L, s + max_size)
        e = limit
        for t in range(s + h, limit):
            if t - h >= 0 and t + h <= L - 1 and all(x < d[t] for x in d[t - h:t]) and \
                    all(x < d[t] for x in d[t + 1:t + h + 1]):
                e = t + 1
                break
        out.append(e)
        s = e
    return out


def _local_maxima(d, h):
    """Every t in [h, L-h) with d[t] > max(d[t-h:t]) and d[t] > max(d[t+1:t+h+1]),
    from numpy sliding-window maxima (independent of the oracle's loops)."""
    d = np.asarray(d, dtype=np.int16)
    L = d.size
    if L < 2 * h + 1:
        return np.zeros(0, dtype=np.int64)
    win = np.lib.stride_tricks.sliding_window_view(d, h).max(axis=1)  # win[i] = max d[i:i+h]
    t = np.arange(h, L - h)
    ok = (d[t] > win[t - h]) & (d[t] > win[t + 1])
    return t[ok]


def test_maxp_single_peak_and_constant():
    d = np.zeros(100, np.uint8)
    d[30] = 255
    # the peak ends the first chunk; the zeros after it have no local maximum: caps, then the stream end
    assert oracle.chunk("maxp", d, 5, 40).tolist() == [31, 71, 100]
    assert pyref.chunk("maxp", d.tolist(), 5, 40) == [31, 71, 100]
    # a constant stream has no strict local maximum: every chunk is capped
    assert oracle.chunk("maxp", np.full(100, 0x42, np.uint8), 3, 10).tolist() == list(range(10, 101, 10))
    # a peak closer than h to the chunk start, or whose right window passes the stream end, is no boundary
    assert oracle.chunk("maxp", d, 31, 90).tolist() == [90, 100]
    d2 = np.zeros(40, np.uint8)
    d2[36] = 9
    assert oracle.chunk("maxp", d2, 4, 60).tolist() == [40]
    # two equal peaks within h of each other: neither is a strict local maximum
    d3 = np.zeros(100, np.uint8)
    d3[40] = d3[43] = 7
    assert oracle.chunk("maxp", d3, 5, 200).tolist() == [100]
    d3[43] = 6  # now 40 is one, 43 (within h of a larger byte) is not
    assert oracle.chunk("maxp", d3, 5, 200).tolist() == [41, 100]


def test_maxp_exhaustive_small_alphabet():
    count = 0
    for n in range(1, 8):
        for tup in itertools.product([0, 1, 2], repeat=n):
            d = list(tup)
            arr = np.array(d, dtype=np.uint8)
            for h in (1, 2, 3):
                for mx in (h + 1, h + 2, 7):
                    exp = _bf_maxp_chunk(d, h, mx)
                    assert oracle.chunk("maxp", arr, h, mx).tolist() == exp, (d, h, mx)
                    assert pyref.chunk("maxp", d, h, mx) == exp
                    count += 1
    assert count > 10000


def test_maxp_random_vs_bruteforce_and_pyref():
    rng = np.random.default_rng(17)
    for trial in range(60):
        n = int(rng.integers(1, 500))
        hi = int(rng.choice([2, 4, 16, 256]))
        d = rng.integers(0, hi, n).astype(np.uint8)
        h = int(rng.integers(1, 20))
        mx = int(h + 1 + rng.integers(0, 80))
        exp = _bf_maxp_chunk(d.tolist(), h, mx)
        assert oracle.chunk("maxp", d, h, mx).tolist() == exp, (n, h, mx)
        assert pyref.chunk("maxp", d.tolist(), h, mx) == exp


@pytest.mark.parametrize("gen", ["uniform", "zipf"])
def test_maxp_invariants_and_local_maxima(gen):
    L = 1 << 20
    d = synth.uniform(L, 21) if gen == "uniform" else synth.zipf_bytes(L, 1.1, 22)
    h, mx = 64, 2048
    ends = oracle.chunk("maxp", d, h, mx)
    lens = _lens(ends)
    assert int(ends[-1]) == L and (lens > 0).all()
    assert (lens[:-1] >= h + 1).all() and (lens <= mx).all()
    q = set(_local_maxima(d, h).tolist())
    s = 0
    for e in ends.tolist():
        if e - s < mx and e < L:          # a content boundary: its last byte is a local maximum ...
            assert e - 1 in q
        # ... and no earlier position of the chunk's candidate range is one
        assert not any(t in q for t in range(s + h, e - 1))
        s = e
    # without a cap the chain visits every local maximum (two are more than h apart)
    ends2 = oracle.chunk("maxp", d, h, L + 1)
    assert (ends2[:-1] - 1).tolist() == sorted(q)


def test_maxp_local_maximum_density_closed_form():
    """On i.i.d. uniform bytes a byte is a strict maximum of its 2h neighbours
    with probability P(h) = sum_v (1/256) (v/256)^(2h); with no cap the chain
    ends a chunk at every local maximum, so the boundary count is ~ (L - 2h) P(h).
    A non-strict test (>=), a one-sided window or a window of 2h bytes on one
    side move the count by far more than the sampling error."""
    L, h = 4 << 20, 64
    d = synth.uniform(L, 23)
    n = oracle.chunk("maxp", d, h, L + 1).size - 1
    p = sum((v / 256.0) ** (2 * h) for v in range(256)) / 256.0
    expect = (L - 2 * h) * p
    assert abs(n - expect) < 5 * math.sqrt(expect), (n, expect)


def test_maxp_check_chunking_accepts_oracle_and_rejects_mutations():
    for gen, h, mx in (("uniform", 100, 3000), ("zipf", 300, 8000), ("runs", 20, 600)):
        L = 300_001
        d = {"uniform": lambda: synth.uniform(L, 34), "zipf": lambda: synth.zipf_bytes(L, 1.1, 35),
             "runs": lambda: np.repeat(synth.uniform(L // 50 + 1, 36), 50)[:L]}[gen]()
        ends = oracle.chunk("maxp", d, h, mx)
        assert oracle.check_chunking("maxp", d, ends, h, mx, threads=4) is None
        for bad in _mutations(ends, L):
            assert oracle.check_chunking("maxp", d, np.array(bad, dtype=np.uint64), h, mx, threads=3) is not None
