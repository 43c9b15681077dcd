"""GPU parity of the transfer-table path (T-mode): saturated
streams (uniform bytes at w >> 256) whose chains are resolved in index space
instead of by halo walks, and the fallback when a stream is not saturated
everywhere.  Every comparison is bit-exact against the oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cdc(cuda_ok):
    import paper_2508_05797_b200 as m
    m.set_dense(0)  # (the dense-index mode would take these streams first: tests/test_gpu_dense.py)
    yield m
    m.set_dense(-1)


def _run(cdc, d, p):
    t = torch.from_numpy(d).cuda()
    n = d.size
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    b = torch.full((cdc.max_boundaries(p, n),), -1, dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    cdc.chunk_async(t, p, b, c, ws)
    got = b[:int(c.item())].cpu().numpy().astype(np.uint64)
    return got, cdc.stats(p, ws, 1, n, n)


@pytest.mark.parametrize("algo,avg", [("ram", 8192), ("ae_max", 8192), ("ae_min", 8192),
                                      ("ram", 16384), ("ae_max", 16384)])
def test_tables_uniform(cdc, algo, avg):
    """configs[0]-shape streams (16 MiB of uniform bytes, plus a ragged tail):
    the tables produce the output and it equals the oracle's."""
    d = synth.uniform((16 << 20) + 777, 10)
    p = cdc.params(algo, avg_size=avg)
    exp = oracle.chunk(algo, d, p.window, p.max_size)
    got, st = _run(cdc, d, p)
    assert st["fast_path"] == 2, st
    assert got.size == exp.size and (got == exp).all()


def test_tables_many_small_segments(cdc):
    """Forced 64 KiB segments: many tables, each with links into the next."""
    d = synth.uniform(6 << 20, 11)
    p = cdc.params("ram", avg_size=8192, seg_bytes=65536)
    exp = oracle.chunk("ram", d, p.window, p.max_size)
    got, st = _run(cdc, d, p)
    assert st["fast_path"] == 2, st
    assert got.size == exp.size and (got == exp).all()


@pytest.mark.parametrize("algo,slack", [("ram", 1), ("ram", 2), ("ram", 301), ("ae_max", 2), ("ae_min", 3)])
def test_tables_tight_cap(cdc, algo, slack):
    """max_size just above the window: nearly every chunk is cut by the cap, so
    chain exits are rarely candidates, and RAM's candidates of a segment reach
    past seg_end + max_size.  Both neighbours must agree on a segment's
    candidate set (regression: an index too short to decide it read as "no
    candidates" on one side only).  16 KiB segments, many hand-overs."""
    d = synth.uniform((2 << 20) + 123, 40)
    w = 5000
    p = cdc.params(algo, window=w, max_size=w + slack, seg_bytes=16384)
    exp = oracle.chunk(algo, d, w, w + slack)
    got, st = _run(cdc, d, p)
    assert got.size == exp.size and (got == exp).all(), st


@pytest.mark.parametrize("algo", ["ram", "ae_max"])
def test_tables_zero_region(cdc, algo):
    """A zero-filled region: steps inside it are not saturated and are read from
    the bytes, and chains that leave a segment through it are handed to the
    next segment as extra entries.  Same boundaries as the oracle."""
    d = synth.uniform(16 << 20, 12)
    d[5 << 20:(5 << 20) + 300_000] = 0
    d[(9 << 20) - 70_000:(9 << 20) + 70_000] = 0  # across a segment boundary
    p = cdc.params(algo, avg_size=8192)
    exp = oracle.chunk(algo, d, p.window, p.max_size)
    got, st = _run(cdc, d, p)
    assert got.size == exp.size and (got == exp).all(), st


@pytest.mark.parametrize("algo", ["ram", "ae_max", "ae_min"])
def test_tables_short_unsaturated_runs(cdc, algo):
    """Short runs without the saturating byte (a few KiB of 0x01 bytes, some
    across segment boundaries): those steps are read from the bytes, chains
    that leave a segment through one are handed to the next segment as extra
    entries, and the tables still resolve the stream."""
    d = synth.uniform(16 << 20, 16)
    rng = np.random.default_rng(16)
    starts = list(rng.integers(0, (16 << 20) - 20000, 40)) + [k * (1 << 17) - 3000 for k in range(1, 128, 9)]
    for a in starts:
        d[a:a + int(rng.integers(2000, 9000))] = 1
    p = cdc.params(algo, avg_size=8192)
    exp = oracle.chunk(algo, d, p.window, p.max_size)
    got, st = _run(cdc, d, p)
    assert st["fast_path"] == 2, st
    assert got.size == exp.size and (got == exp).all()


@pytest.mark.parametrize("algo,avg", [("ram", 8192), ("ram", 16384), ("ae_max", 8192)])
def test_tables_versioned(cdc, algo, avg):
    """configs[2]-like bytes (uniform with 10 % zero-filled 64 KiB regions, a
    snapshot with edits) at a size the oracle finishes quickly."""
    base, snap = synth.versioned(24 << 20, 1, seed=14)
    for d in (base, snap):
        p = cdc.params(algo, avg_size=avg)
        exp = oracle.chunk(algo, d, p.window, p.max_size)
        got, st = _run(cdc, d, p)
        assert got.size == exp.size and (got == exp).all(), st


@pytest.mark.parametrize("algo", ["ram", "ae_max"])
def test_tables_fallback(cdc, algo):
    """Half the stream never holds the saturating byte (bytes 1..254): its
    segments are not dense, the attempt fails and the speculative walk
    resolves the stream."""
    d = synth.uniform(16 << 20, 15)
    d[8 << 20:] = (d[8 << 20:] % 254 + 1).astype(np.uint8)
    p = cdc.params(algo, avg_size=8192)
    exp = oracle.chunk(algo, d, p.window, p.max_size)
    got, st = _run(cdc, d, p)
    assert st["fast_path"] != 2, st
    assert got.size == exp.size and (got == exp).all()


def test_tables_graph_replay(cdc):
    """The table path captured in a CUDA graph replays exactly."""
    d = synth.uniform(16 << 20, 13)
    p = cdc.params("ram", avg_size=8192)
    exp = oracle.chunk("ram", d, p.window, p.max_size)
    t = torch.from_numpy(d).cuda()
    n = d.size
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    b = torch.empty(cdc.max_boundaries(p, n), dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
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
    assert cdc.stats(p, ws, 1, n, n)["fast_path"] == 2
