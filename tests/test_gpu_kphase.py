"""GPU parity of K-phase speculation (cdc_kphase.cuh): a single
stream with a window the sparse walk takes (w >= 4096) and segments longer
than the transfer tables take (> 256 KiB) is chunked with K chains per
segment.  Chains meet siblings in their segment and the chains of later
segments in their halos; k_kres1-3 follow node 0's path.  A halo that gives
up on the true chain opens the gate of the ordinary pipeline, which then does
the work.  Every comparison is element-wise against oracle.chunk (bit-exact);
expected values come only from oracle/.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ALGOS = ["ram", "ae_max", "ae_min"]
SEG = 512 << 10  # > T_MAX_SEG: no transfer tables, so K-phase speculation


@pytest.fixture(scope="module")
def cdc(cuda_ok):
    import paper_2508_05797_b200 as m
    yield m
    m.set_kphase(-1)


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _run(cdc, d, algo, w, mx, seg=SEG, halo=0, ws=None):
    p = cdc.params(algo, window=w, max_size=mx, seg_bytes=seg, halo_bytes=halo)
    n = d.size
    t = _dev(d)
    if ws is None:
        ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    cdc.chunk_async(t, p, b, c, ws)
    torch.cuda.synchronize()
    got = b[: int(c.item())].cpu().numpy().astype(np.uint64)
    return got, cdc.stats(p, ws, 1, n, n), ws


def _check(cdc, d, algo, w, mx, seg=SEG, halo=0, want_kphase=True):
    got, st, _ = _run(cdc, d, algo, w, mx, seg, halo)
    exp = oracle.chunk(algo, d, w, mx)
    assert got.size == exp.size, (got.size, exp.size, st)
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, (int(bad[0]), int(got[bad[0]]), int(exp[bad[0]]), st)
    if want_kphase:
        assert st["fast_path"] == 3, st
    return st


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("w", [4096, 7936, 16128])
def test_kphase_uniform(cdc, algo, w):
    """Saturated bytes: siblings meet inside segments, halos meet later segments' chains."""
    cdc.set_kphase(-1)
    d = synth.uniform((24 << 20) + 4321, 31 + w)
    _check(cdc, d, algo, w, 4 * (w + 256))


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("k", [1, 2, 3, 5, 8])
def test_kphase_forced_k(cdc, algo, k):
    """Every chain count, including K = 1 (one chain per segment through the K-phase resolver)."""
    cdc.set_kphase(k)
    try:
        d = synth.uniform((12 << 20) + 999, 40 + k)
        # (one chain per segment: halos on uniform bytes may outrun the cap, and
        # then the ordinary pipeline writes the output)
        _check(cdc, d, algo, 7936, 32768, want_kphase=k >= 2)
    finally:
        cdc.set_kphase(-1)


@pytest.mark.parametrize("algo", ["ram", "ae_max"])
@pytest.mark.parametrize("w", [7936, 16128])
def test_kphase_versioned(cdc, algo, w):
    """configs[2]'s shape (uniform base with zero-filled 64 KiB regions, and a snapshot)."""
    cdc.set_kphase(-1)
    snaps = synth.versioned(32 << 20, 1, seed=7)
    for d in snaps:
        _check(cdc, d, algo, w, 4 * (w + 256))


@pytest.mark.parametrize("algo", ALGOS)
def test_kphase_mixed_content(cdc, algo):
    """configs[4]'s alternating shape, Zipf bytes, and patchwork switching between
    saturated and unsaturated stretches (sparse <-> ring hand-overs inside nodes)."""
    cdc.set_kphase(-1)
    for d in (synth.alternating((32 << 20) + 5, region=4 << 20, seed=9),
              synth.zipf_bytes((16 << 20) + 3, 1.1, 5),
              synth.patchwork((16 << 20) + 17, seed=6)):
        _check(cdc, d, algo, 8192, 32768)


@pytest.mark.parametrize("algo", ALGOS)
def test_kphase_constant_stream_falls_back(cdc, algo):
    """Chains in a constant stream never meet (every chunk is w+1 long): the
    halos on the true chain give up and the ordinary pipeline writes the output."""
    cdc.set_kphase(-1)
    d = np.full((6 << 20) + 11, 7, dtype=np.uint8)
    st = _check(cdc, d, algo, 4096, 16384, halo=64 << 10, want_kphase=False)
    assert st["fast_path"] != 3, st


@pytest.mark.parametrize("algo", ["ram", "ae_max"])
def test_kphase_short_halo_cap(cdc, algo):
    """A halo cap of a few windows: some halos give up (the gate opens when one
    is on the true chain), others still meet; the output is exact either way."""
    cdc.set_kphase(-1)
    d = synth.uniform((16 << 20) + 1, 77)
    for halo in (2 * 8192, 8 * 8192):
        _check(cdc, d, algo, 7936, 32768, halo=halo, want_kphase=False)


@pytest.mark.parametrize("algo", ALGOS)
def test_kphase_tight_cap_and_ragged(cdc, algo):
    """Caps just above the window (capped chunks in bodies and halos) and a stream
    whose length is not a multiple of anything.  With most chunks capped at
    nearly w+1 bytes chains keep their phases and rarely meet, so the gate may
    send the call to the ordinary pipeline; the output is exact either way."""
    cdc.set_kphase(-1)
    d = synth.uniform((9 << 20) + 12345, 3)
    for w, mx in [(4096, 4097), (4096, 4200), (9000, 9000 + 33), (4096, 8192)]:
        _check(cdc, d, algo, w, mx, want_kphase=False)


def test_kphase_workspace_reuse(cdc):
    """Two calls on one workspace: the second sees none of the first call's lists."""
    cdc.set_kphase(-1)
    a = synth.uniform((8 << 20) + 5, 1)
    b = synth.versioned(8 << 20, 0, seed=3)[0]
    p = cdc.params("ram", window=7936, max_size=32768, seg_bytes=SEG)
    n = max(a.size, b.size)
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    for d in (a, b, a):
        got, st, _ = _run(cdc, d, "ram", 7936, 32768, ws=ws)
        exp = oracle.chunk("ram", d, 7936, 32768)
        assert got.size == exp.size and (got == exp).all()
        assert st["fast_path"] == 3


def test_kphase_default_segments_and_graph(cdc):
    """Default geometry on a 640 MiB stream (segments over 256 KiB: K-phase without
    seg_bytes) captured in a CUDA graph and replayed; every chunk checked against
    the oracle (oracle.check_chunking: each end equals chunk_end of the previous)."""
    cdc.set_kphase(-1)
    n = (640 << 20) + 7
    d = synth.versioned(n, 0, seed=11)[0]
    p = cdc.params("ram", avg_size=16384)
    t = _dev(d)
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        cdc.chunk_async(t, p, b, c, ws)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        cdc.chunk_async(t, p, b, c, ws)
    b.fill_(0)
    g.replay()
    torch.cuda.synchronize()
    assert cdc.stats(p, ws, 1, n, n)["fast_path"] == 3
    got = b[: int(c.item())].cpu().numpy().astype(np.uint64)
    assert oracle.check_chunking("ram", d, got, p.window, p.max_size) is None
