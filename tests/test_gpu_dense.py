"""GPU parity of the dense-index mode (cdc_dense.cuh): small
single streams whose every window holds the saturating byte are resolved as
one recurrence over that byte's positions; anything else is handed to the
ordinary pipeline on the device.  Every comparison is bit-exact against the
oracle (RAM §2.1.2 l.198, AE l.169)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

DENSE = 4  # cdc_stats fast_path code of the dense-index mode


@pytest.fixture(scope="module")
def cdc(cuda_ok):
    import paper_2508_05797_b200 as m
    m.set_dense(-1)
    return m


def _run(cdc, d, p, t=None):
    t = torch.from_numpy(d).cuda() if t is None else t
    n = t.numel()
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    b = torch.full((cdc.max_boundaries(p, n),), -1, dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    cdc.chunk_async(t, p, b, c, ws)
    got = b[:int(c.item())].cpu().numpy().astype(np.uint64)
    return got, cdc.stats(p, ws, 1, n, n)


def _check(cdc, algo, d, p, dense):
    exp = oracle.chunk(algo, d, p.window, p.max_size)
    got, st = _run(cdc, d, p)
    if dense is not None:
        assert (st["fast_path"] == DENSE) == dense, st
    assert got.size == exp.size and (got == exp).all(), (algo, d.size, st)


@pytest.mark.parametrize("algo", ["ram", "ae_max", "ae_min"])
@pytest.mark.parametrize("avg", [8192, 16384])
def test_dense_uniform(cdc, algo, avg):
    """configs[0]-shape streams (16 MiB of uniform bytes, plus a ragged tail)."""
    d = synth.uniform((16 << 20) + 777, 10)
    _check(cdc, algo, d, cdc.params(algo, avg_size=avg), True)


@pytest.mark.parametrize("n", [1 << 20, (1 << 20) + 1, (3 << 20) + 12345, (9 << 20) - 4097, (33 << 20) + 5, 64 << 20])
@pytest.mark.parametrize("algo", ["ram", "ae_max"])
def test_dense_sizes(cdc, algo, n):
    """Both ends of the mode's size range, ragged tails, several segments per CTA."""
    d = synth.uniform(n, 20 + (n & 7))
    _check(cdc, algo, d, cdc.params(algo, avg_size=8192), True)


@pytest.mark.parametrize("algo,window", [("ram", 4096), ("ae_max", 4096), ("ae_min", 5000), ("ram", 20000),
                                         ("ae_max", 24576), ("ram", 24576)])
def test_dense_windows(cdc, algo, window):
    d = synth.uniform((8 << 20) + 333, 31)
    p = cdc.params(algo, window=window, max_size=4 * window)
    _check(cdc, algo, d, p, None)  # (the widest windows may exceed the candidate capacity: either path)


@pytest.mark.parametrize("algo", ["ram", "ae_max", "ae_min"])
@pytest.mark.parametrize("off", [1, 7, 16, 4095])
def test_dense_unaligned(cdc, algo, off):
    d = synth.uniform((4 << 20) + 4096 + 99, 41)
    t = torch.from_numpy(d).cuda()[off:]
    p = cdc.params(algo, avg_size=8192)
    exp = oracle.chunk(algo, d[off:], p.window, p.max_size)
    got, st = _run(cdc, d[off:], p, t)
    assert st["fast_path"] == DENSE, st
    assert got.size == exp.size and (got == exp).all()


def _hole(d, at, n, algo):
    """a stretch without the saturating byte"""
    sat = 0 if algo == "ae_min" else 255
    seg = d[at:at + n]
    seg[seg == sat] = 7
    return d


@pytest.mark.parametrize("algo", ["ram", "ae_max", "ae_min"])
@pytest.mark.parametrize("where", ["start", "middle", "seg_edge", "end"])
def test_dense_falls_back_on_a_hole(cdc, algo, where):
    """One window-sized stretch without the saturating byte anywhere in the
    stream: the kernels notice and the ordinary pipeline produces the output."""
    n = (6 << 20) + 1000
    d = synth.uniform(n, 51).copy()
    p = cdc.params(algo, avg_size=8192)
    w = p.window
    at = {"start": 0, "middle": 3 << 20, "seg_edge": 2 * 65536 - w // 2, "end": n - w - 3}[where]
    _hole(d, at, w + 2, algo)
    _check(cdc, algo, d, p, False)


@pytest.mark.parametrize("algo", ["ram", "ae_max"])
def test_dense_hole_just_short_enough(cdc, algo):
    """Gaps of exactly w between saturating bytes still satisfy the condition;
    w + 1 does not.  Either way the output equals the oracle's."""
    n = 4 << 20
    for gap, dense in ((0, True), (1, False)):
        d = synth.uniform(n, 52).copy()
        p = cdc.params(algo, avg_size=8192)
        w = p.window
        a = 1 << 20
        d[a] = 255
        _hole(d, a + 1, w - 1 + gap, algo)
        d[a + w + gap] = 255
        _check(cdc, algo, d, p, dense)


@pytest.mark.parametrize("algo", ["ram", "ae_max", "ae_min"])
def test_dense_stream_ends(cdc, algo):
    """The saturating byte as the very last byte, right before it, and a tail of exactly w bytes after the last one."""
    sat = 0 if algo == "ae_min" else 255
    p = cdc.params(algo, avg_size=8192)
    w = p.window
    for k, tail in enumerate((0, 1, 2, w - 1, w)):
        n = (2 << 20) + 17 * k
        d = synth.uniform(n, 60 + k).copy()
        last = n - 1 - tail
        d[last] = sat
        _hole(d, last + 1, tail, algo)
        _check(cdc, algo, d, p, True)


def test_dense_other_data(cdc):
    """Streams the mode must refuse or hand over: skewed bytes (the saturating
    byte is rare), far too many saturating bytes, constant streams, caps below 2w + 2."""
    n = 5 << 20
    p = cdc.params("ram", avg_size=8192)
    _check(cdc, "ram", synth.zipf_bytes(n, 1.1, 3), p, None)
    rng = np.random.default_rng(7)
    many = rng.integers(0, 256, n, dtype=np.uint8)
    many[rng.random(n) < 1 / 16] = 255
    _check(cdc, "ram", many, p, False)
    _check(cdc, "ae_max", many, cdc.params("ae_max", avg_size=8192), False)
    _check(cdc, "ram", np.full(n, 255, dtype=np.uint8), p, False)
    _check(cdc, "ae_min", np.zeros(n, dtype=np.uint8), cdc.params("ae_min", avg_size=8192), False)
    d = synth.uniform(n, 8)
    for algo in ("ram", "ae_max"):
        q = cdc.params(algo, avg_size=8192)
        q.max_size = 2 * q.window + 1
        _check(cdc, algo, d, q, False)
        q.max_size = 2 * q.window + 2
        _check(cdc, algo, d, q, True)


def test_dense_off_switch_and_repeats(cdc):
    d = synth.uniform(16 << 20, 0)  # configs[0]
    p = cdc.params("ram", avg_size=8192)
    exp = oracle.chunk("ram", d, p.window, p.max_size)
    t = torch.from_numpy(d).cuda()
    n = d.size
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(5):  # the same workspace again and again
        b.fill_(-1)
        cdc.chunk_async(t, p, b, c, ws)
        got = b[:int(c.item())].cpu().numpy().astype(np.uint64)
        assert got.size == exp.size and (got == exp).all()
    assert cdc.stats(p, ws, 1, n, n)["fast_path"] == DENSE
    # CUDA graph of the call
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        cdc.chunk_async(t, p, b, c, ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        cdc.chunk_async(t, p, b, c, ws)
    for _ in range(3):
        b.fill_(-1)
        c.zero_()
        g.replay()
        torch.cuda.synchronize()
        got = b[:int(c.item())].cpu().numpy().astype(np.uint64)
        assert got.size == exp.size and (got == exp).all()
    cdc.set_dense(0)
    try:
        got, st = _run(cdc, d, p)
        assert st["fast_path"] != DENSE
        assert got.size == exp.size and (got == exp).all()
    finally:
        cdc.set_dense(-1)


@pytest.mark.parametrize("algo,avg", [("ram", 8192), ("ram", 16384), ("ae_max", 8192), ("ae_min", 16384)])
def test_dense_then_kphase_on_versioned(cdc, algo, avg):
    """configs[2]'s recipe at 16 MiB (uniform bytes with zero-filled regions): the dense attempt gives up,
    K-phase speculation behind its gate produces the output (its three resolution levels in one CTA)."""
    d = synth.versioned(16 << 20, 0, seed=5)[0]
    p = cdc.params(algo, avg_size=avg)
    exp = oracle.chunk(algo, d, p.window, p.max_size)
    got, st = _run(cdc, d, p)
    assert st["fast_path"] == 3, st
    assert got.size == exp.size and (got == exp).all()


def test_dense_hands_over_constant_streams(cdc):
    """A constant stream is not saturated (the dense gate opens); whichever path behind it resolves the
    chain (K-phase when one of its chains coincides with the true one, else the ordinary pipeline, whose
    lists K-phase's resolver then resets: tests/test_gpu_kphase.py forces that), the output is the oracle's."""
    for algo, val in (("ram", 0), ("ae_max", 7), ("ae_min", 255)):
        d = np.full((6 << 20) + 321, val, dtype=np.uint8)
        p = cdc.params(algo, avg_size=8192)
        exp = oracle.chunk(algo, d, p.window, p.max_size)
        got, st = _run(cdc, d, p)
        assert st["fast_path"] != DENSE, st
        assert got.size == exp.size and (got == exp).all()
