"""GPU parity of MAXP (§2.1.2 l.173/l.196, §4.3 l.361; readings M1-M5):
the CUDA path (k_maxp_scan / link / path / write through the C ABI) against the
CPU oracle, element by element.  Inputs come from synth/ and seeded numpy;
expected values come only from oracle/.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TILE = 32768  # k_maxp_scan's tile (cdc_maxp.cuh MX_TILE): sizes below span several tiles and a ragged tail


@pytest.fixture(scope="module")
def cdc(cuda_ok):
    import paper_2508_05797_b200 as m
    return m


def _gpu(cdc, data, h, mx, offset=0):
    p = cdc.params("maxp", window=h, max_size=mx)
    if offset:
        buf = torch.zeros(data.size + offset + 32, dtype=torch.uint8, device="cuda")
        buf[offset:offset + data.size] = torch.from_numpy(np.ascontiguousarray(data)).cuda()
        t = buf[offset:offset + data.size]
    else:
        t = torch.from_numpy(np.ascontiguousarray(data)).cuda()
    return cdc.chunk(t, p).cpu().numpy().astype(np.uint64)


def _check(cdc, data, h, mx, offset=0):
    got = _gpu(cdc, data, h, mx, offset)
    exp = oracle.chunk("maxp", data, h, mx)
    assert got.size == exp.size and (got == exp).all(), (
        h, mx, offset, got.size, exp.size, int(np.argmax(got[:min(got.size, exp.size)] != exp[:min(got.size, exp.size)])))


def _sparse_peaks(n, seed, density, top=256):
    """Zeros with rare random bytes: long stretches without a local maximum, so
    chunks are capped and maxima near a cap start are skipped (k_maxp_path)."""
    rng = np.random.default_rng(seed)
    d = np.zeros(n, np.uint8)
    k = max(1, int(n * density))
    d[rng.integers(0, n, k)] = rng.integers(1, top, k).astype(np.uint8)
    return d


GENS = {
    "uniform": lambda n: synth.uniform(n, 3),
    "zipf": lambda n: synth.zipf_bytes(n, 1.1, 4),
    "zeros": lambda n: np.zeros(n, np.uint8),
    "ff": lambda n: np.full(n, 255, np.uint8),
    "ramp": lambda n: (np.arange(n) % 256).astype(np.uint8),
    "runs": lambda n: np.repeat(synth.uniform(n // 37 + 1, 5), 37)[:n],
    "versioned": lambda n: synth.versioned(n, 0, seed=2)[0],
    "sparse": lambda n: _sparse_peaks(n, 6, 1 / 3000),
}


@pytest.mark.parametrize("gen", sorted(GENS))
@pytest.mark.parametrize("h", [1, 5, 31, 447, 3000])
def test_maxp_generators(cdc, gen, h):
    n = 5 * TILE + 12345
    _check(cdc, GENS[gen](n), h, 4 * 8192 if h >= 31 else 64 * h + 1)


@pytest.mark.parametrize("h", [1, 2, 3, 14, 15, 16, 17, 30, 31, 32, 33, 46, 47, 48, 63, 100, 447, 1000, 4095, 4096,
                               20000, 65536])
def test_maxp_windows(cdc, h):
    n = 3 * TILE + 2 * h + 777
    d = synth.uniform(n, h)
    for mx in (h + 1, h + 2, 3 * h + 5, 1 << 40):
        _check(cdc, d, h, mx)


@pytest.mark.parametrize("h,mx", [(4, 40), (10, 40), (10, 11), (60, 600), (200, 1000), (447, 2000)])
@pytest.mark.parametrize("density", [1 / 50, 1 / 400, 1 / 5000])
def test_maxp_capped_stretches_skip_maxima(cdc, h, mx, density):
    """Capped runs whose next local maximum lies within h of a cap start skip it:
    many such runs, some skipping more than one maximum."""
    for seed in range(3):
        _check(cdc, _sparse_peaks(4 * TILE + 999, 100 + seed, density, top=8), h, mx)


@pytest.mark.parametrize("n", [0, 1, 2, 15, 16, 17, 447, 894, 895, 896, TILE - 1, TILE, TILE + 1, 2 * TILE + 447])
def test_maxp_sizes(cdc, n):
    d = synth.uniform(max(n, 1), 9)[:n]
    _check(cdc, d, 447, 4 * 8192)
    _check(cdc, d, 3, 40)


@pytest.mark.parametrize("offset", [1, 7, 15])
def test_maxp_unaligned(cdc, offset):
    d = synth.zipf_bytes(2 * TILE + 4321, 1.1, 11)
    _check(cdc, d, 447, 32768, offset)
    _check(cdc, d, 20, 2000, offset)


def test_maxp_full_256mib_uniform_and_zipf(cdc):
    """256 MiB at the 8 KiB default (h = 447, max_size 32 KiB): every chunk
    verified against the oracle (check_chunking over the host's cores)."""
    p = cdc.params("maxp", avg_size=8192)
    assert p.window == 447
    for d in (synth.uniform(256 << 20, 1), synth.zipf_bytes(256 << 20, 1.1, 1)):
        t = torch.from_numpy(d).cuda()
        got = cdc.chunk(t, p).cpu().numpy().astype(np.uint64)
        assert oracle.check_chunking("maxp", d, got, p.window, p.max_size) is None
        for _ in range(4):  # repeated calls give the same boundaries (no race between tiles or threads)
            assert np.array_equal(cdc.chunk(t, p).cpu().numpy().astype(np.uint64), got)


def test_maxp_host_entry_and_graph(cdc):
    d = synth.uniform(3 * TILE + 5, 12)
    p = cdc.params("maxp", avg_size=4096)
    exp = oracle.chunk("maxp", d, p.window, p.max_size)
    got = cdc.chunk_host(d, p)
    assert np.array_equal(np.asarray(got, dtype=np.uint64), exp)
    # CUDA-graph replay of the call on preallocated buffers
    t = torch.from_numpy(d).cuda()
    n = d.size
    cap = cdc.max_boundaries(p, n)
    bounds = torch.zeros(cap, dtype=torch.int64, device="cuda")
    count = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        cdc.chunk_async(t, p, bounds, count, ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        cdc.chunk_async(t, p, bounds, count, ws)
    for _ in range(3):
        bounds.zero_()
        g.replay()
        torch.cuda.synchronize()
        m = int(count.item())
        assert m == exp.size and np.array_equal(bounds[:m].cpu().numpy().astype(np.uint64), exp)


def test_maxp_rejected_where_undefined(cdc):
    p = cdc.params("maxp", avg_size=8192)
    d = torch.from_numpy(synth.uniform(100000, 2)).cuda()
    with pytest.raises(cdc.CdcError):
        cdc.chunk(d, cdc.params("maxp", window=65537, max_size=1 << 20))
    with pytest.raises(cdc.CdcError):
        cdc.stats(p, torch.empty(1 << 20, dtype=torch.uint8, device="cuda"), 1, 100000, 100000)


def _check_batch(cdc, data, offs, h, mx):
    p = cdc.params("maxp", window=h, max_size=mx)
    b, bo = cdc.chunk_batch(torch.from_numpy(np.ascontiguousarray(data)).cuda(), offs, p)
    got, gbo = b.cpu().numpy().astype(np.uint64), bo.cpu().numpy().astype(np.int64)
    exp, ebo = oracle.chunk_batch("maxp", data, offs, h, mx)
    assert np.array_equal(gbo, ebo), (h, mx, np.nonzero(gbo != ebo)[0][:5])
    assert np.array_equal(got, exp), (h, mx)


@pytest.mark.parametrize("h,mx", [(3, 40), (31, 700), (447, 32768), (2000, 9000)])
def test_maxp_batch_random(cdc, h, mx):
    """Packed batches: empty files, files shorter than h or 2h+1, files of several
    tiles with ragged tails, each file chunked on its own (file-relative ends)."""
    rng = np.random.default_rng(h)
    for trial in range(4):
        n = int(rng.integers(1, 300))
        sizes = rng.choice([0, 1, 5, h, 2 * h, 2 * h + 1, 3000, TILE - 1, TILE + 7, 3 * TILE + 555], n)
        sizes = np.where(rng.random(n) < 0.3, rng.integers(0, 200000, n), sizes)
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        gen = [lambda m: synth.uniform(m, 40 + trial), lambda m: synth.zipf_bytes(m, 1.1, 41 + trial),
               lambda m: _sparse_peaks(m, 42 + trial, 1 / 300, top=8)][trial % 3]
        data = gen(int(max(offs[-1], 1)))[:offs[-1]]
        _check_batch(cdc, data, offs, h, mx)


def test_maxp_batch_all_empty_and_single(cdc):
    _check_batch(cdc, np.zeros(0, np.uint8), np.zeros(4, np.int64), 447, 32768)
    d = synth.uniform(5 * TILE + 3, 44)
    _check_batch(cdc, d, np.array([0, d.size], np.int64), 447, 32768)


def test_maxp_batch_many_files_configs3_shape(cdc):
    """12,500 files of configs[3]'s size distribution and content mix at 8 KiB,
    every chunk of every file verified (check_batch), and the host entry point."""
    data, offs = synth.many_files(12500, seed=3)
    p = cdc.params("maxp", avg_size=8192)
    b, bo = cdc.chunk_batch(torch.from_numpy(data).cuda(), offs, p)
    got, gbo = b.cpu().numpy().astype(np.uint64), bo.cpu().numpy().astype(np.uint64)
    assert oracle.check_batch("maxp", data, offs, got, gbo, p.window, p.max_size) is None
    hb, hbo = cdc.chunk_batch_host(data[:offs[2000]], offs[:2001], p)
    assert np.array_equal(np.asarray(hb, dtype=np.uint64), got[:gbo[2000]])
    assert np.array_equal(np.asarray(hbo, dtype=np.uint64), gbo[:2001])
