"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Integer/index work: every comparison is bit-exact (boundary offsets, counts,
extreme values and positions).  Inputs come from synth/ (seeded); expected
values come only from oracle/.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import dedup

pytestmark = pytest.mark.gpu

ALGOS = ["ram", "ae_max", "ae_min"]


@pytest.fixture(scope="module")
def cdc(cuda_ok):
    import paper_2508_05797_b200 as m
    return m


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _gpu_chunk(cdc, data, algo, w, mx, seg=0, halo=0, offset=0):
    p = cdc.params(algo, window=w, max_size=mx, seg_bytes=seg, halo_bytes=halo)
    if offset:
        buf = torch.zeros(data.size + offset + 32, dtype=torch.uint8, device="cuda")
        buf[offset:offset + data.size] = _dev(data)
        t = buf[offset:offset + data.size]
    else:
        t = _dev(data)
    return cdc.chunk(t, p).cpu().numpy().astype(np.uint64)


# ---------------------------------------------------------------- primitives
@pytest.mark.parametrize("mode", ["max", "min"])
def test_extreme_byte_search(cdc, mode):
    rng = np.random.default_rng(0)
    data = rng.integers(0, 256, 1 << 20, dtype=np.uint8)
    data[5000:9000] = 7                       # plateau: leftmost tie-break
    offs = rng.integers(0, (1 << 20) - 9000, 500)
    lens = rng.integers(1, 9000, 500)
    offs[:4], lens[:4] = [5000, 5001, 0, 17], [4000, 1, 1, 8192]
    val, pos = cdc.extreme_byte_search(_dev(data), offs, lens, mode)
    val, pos = val.cpu().numpy(), pos.cpu().numpy()
    for i in range(offs.size):
        v, p = oracle.extreme_byte_search(data[offs[i]:offs[i] + lens[i]], mode)
        assert (val[i], pos[i]) == (v, p), i


@pytest.mark.parametrize("cmp", ["gt", "geq", "lt", "leq", "eq"])
def test_range_scan(cdc, cmp):
    rng = np.random.default_rng(1)
    data = rng.integers(0, 256, 1 << 20, dtype=np.uint8)
    offs = rng.integers(0, (1 << 20) - 5000, 400)
    lens = rng.integers(0, 5000, 400)
    tg = rng.choice([0, 1, 127, 128, 200, 250, 254, 255], 400).astype(np.uint8)
    got = cdc.range_scan(_dev(data), offs, lens, tg, cmp).cpu().numpy()
    for i in range(offs.size):
        r = oracle.range_scan(data[offs[i]:offs[i] + lens[i]], int(tg[i]), cmp)
        assert got[i] == (lens[i] if r is None else r), i


# ---------------------------------------------------------------- whole-stream chunking
GENS = {
    "uniform": lambda n, s: synth.uniform(n, s),
    "zipf": lambda n, s: synth.zipf_bytes(n, 1.1, s),
    "zeros": lambda n, s: synth.constant(n, 0),
    "ff": lambda n, s: synth.constant(n, 255),
    "inc": lambda n, s: (np.arange(n) % 256).astype(np.uint8),
    "dec": lambda n, s: (255 - np.arange(n) % 256).astype(np.uint8),
    "runs": lambda n, s: synth.alternating(n, region=1 << 16, seed=s),
    "versioned": lambda n, s: synth.versioned(n, 1, seed=s, region=1 << 14)[1][:n],
    "satedge": lambda n, s: synth.saturation_edges(n, s),
    "satedge_dense": lambda n, s: synth.saturation_edges(n, s, p=1 / 40),
}


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("gen", list(GENS))
def test_chunk_small_segments(cdc, algo, gen):
    """Many small segments force speculation, halos across segments and fix-ups."""
    n = 3 * (1 << 20) + 777        # ragged tail
    d = GENS[gen](n, 7)
    w, mx = 600, 4000
    exp = oracle.chunk(algo, d, w, mx)
    for seg, halo in [(16384, 0), (4096, 8192), (65536, 4096)]:
        got = _gpu_chunk(cdc, d, algo, w, mx, seg=seg, halo=halo)
        assert got.size == exp.size and (got == exp).all(), (seg, halo)


@pytest.mark.parametrize("algo", ALGOS)
def test_chunk_default_params_many_sizes(cdc, algo):
    rng = np.random.default_rng(3)
    for n in [0, 1, 2, 15, 16, 17, 511, 512, 2047, 2048, 2049, 100000, 1 << 20, (1 << 21) + 13]:
        d = rng.integers(0, 256, n, dtype=np.uint8)
        for avg in [256, 1024, 4096]:
            p = cdc.params(algo, avg_size=avg)
            exp = oracle.chunk(algo, d, p.window, p.max_size)
            got = cdc.chunk(_dev(d), p).cpu().numpy().astype(np.uint64) if n else np.zeros(0, np.uint64)
            if n == 0:
                got = cdc.chunk(torch.zeros(0, dtype=torch.uint8, device="cuda"), p).cpu().numpy()
            assert got.size == exp.size and (got == exp).all(), (n, avg)


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("offset", [1, 3, 8, 15])
def test_unaligned_input(cdc, algo, offset):
    d = synth.zipf_bytes(300001, 1.1, 4)
    exp = oracle.chunk(algo, d, 300, 2000)
    got = _gpu_chunk(cdc, d, algo, 300, 2000, seg=8192, offset=offset)
    assert (got == exp).all() and got.size == exp.size


@pytest.mark.parametrize("algo", ALGOS)
def test_edge_windows(cdc, algo):
    rng = np.random.default_rng(5)
    d = rng.integers(0, 4, 200000).astype(np.uint8)
    for w, mx in [(1, 2), (1, 3), (2, 3), (5, 6), (31, 33), (2047, 2048), (2048, 9000)]:
        exp = oracle.chunk(algo, d, w, mx)
        got = _gpu_chunk(cdc, d, algo, w, mx, seg=32768)
        assert got.size == exp.size and (got == exp).all(), (w, mx)


# ---------------------------------------------------------------- BASELINE configs
def test_config0_ram_8k_16mib_uniform(cdc):
    """BASELINE configs[0]: RAM, avg 8 KiB, 16 MiB uniform, seed 0 (bench launch config)."""
    d = synth.uniform(16 << 20, 0)
    p = cdc.params("ram", avg_size=8192)
    exp = oracle.chunk("ram", d, p.window, p.max_size)
    got = cdc.chunk(_dev(d), p).cpu().numpy().astype(np.uint64)
    assert got.size == exp.size and (got == exp).all()


def test_config1_ae_4k_256mib_zipf(cdc):
    """BASELINE configs[1] (the bench workload): AE-Max, avg 4 KiB, 256 MiB Zipf(1.1), seed 1."""
    d = synth.zipf_bytes(256 << 20, 1.1, 1)
    p = cdc.params("ae_max", avg_size=4096)
    exp = oracle.chunk("ae_max", d, p.window, p.max_size)
    got = cdc.chunk(_dev(d), p).cpu().numpy().astype(np.uint64)
    assert got.size == exp.size and (got == exp).all()


@pytest.mark.parametrize("avg", [4096, 8192, 16384])
def test_config2_versioned_dedup(cdc, avg):
    """BASELINE configs[2] (scaled: 64 MiB base, 3 snapshots): AE and RAM; boundaries
    and the Eq. (1) space savings from exact chunk equality match the oracle."""
    snaps = synth.versioned(64 << 20, 3, seed=2)
    for algo in ["ae_max", "ram"]:
        p = cdc.params(algo, avg_size=avg)
        g_ends, o_ends = [], []
        for s in snaps:
            e = oracle.chunk(algo, s, p.window, p.max_size)
            g = cdc.chunk(_dev(s), p).cpu().numpy().astype(np.uint64)
            assert g.size == e.size and (g == e).all()
            g_ends.append(g)
            o_ends.append(e)
        assert dedup.unique_bytes(snaps, g_ends) == dedup.unique_bytes(snaps, o_ends)


def test_config3_many_files(cdc):
    """BASELINE configs[3] (scaled to 2000 files): RAM 8 KiB over a packed batch."""
    data, offs = synth.many_files(2000, seed=3)
    p = cdc.params("ram", avg_size=8192)
    exp, exp_bo = oracle.chunk_batch("ram", data, offs, p.window, p.max_size)
    got, bo = cdc.chunk_batch(_dev(data), offs, p)
    assert (bo.cpu().numpy() == exp_bo).all()
    assert (got.cpu().numpy().astype(np.uint64) == exp).all()
    # the same call on preallocated device buffers, twice with one workspace
    total, max_len = int(offs[-1]), int(np.diff(offs).max())
    b = torch.full((exp.size + 8,), -1, dtype=torch.int64, device="cuda")
    bo2 = torch.zeros(offs.size, dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = torch.empty(cdc.workspace_size(p, offs.size - 1, total, max_len), dtype=torch.uint8, device="cuda")
    for _ in range(2):
        cdc.chunk_batch_async(_dev(data), _dev(offs), total, max_len, p, b, bo2, c, ws)
        assert int(c.item()) == exp.size and (bo2.cpu().numpy() == exp_bo).all()
        assert (b[:exp.size].cpu().numpy().astype(np.uint64) == exp).all()


@pytest.mark.parametrize("algo", ["ae_max", "ram"])
def test_config4_alternating_regions(cdc, algo):
    """BASELINE configs[4] shape on one GPU (scaled): alternating uniform / low-entropy regions."""
    d = synth.alternating(96 << 20, region=16 << 20, seed=5)
    p = cdc.params(algo, avg_size=8192)
    exp = oracle.chunk(algo, d, p.window, p.max_size)
    got = cdc.chunk(_dev(d), p).cpu().numpy().astype(np.uint64)
    assert got.size == exp.size and (got == exp).all()


# ---------------------------------------------------------------- batch edge cases, chain, host API
@pytest.mark.parametrize("algo", ALGOS)
def test_batch_edge_cases(cdc, algo):
    rng = np.random.default_rng(9)
    sizes = [0, 1, 5, 0, 700, 4096, 0, 100000, 3, 65536 * 3 + 5, 0]
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    data = rng.integers(0, 256, int(offs[-1]), dtype=np.uint8)
    p = cdc.params(algo, window=300, max_size=1200, seg_bytes=8192)
    exp, exp_bo = oracle.chunk_batch(algo, data, offs, 300, 1200)
    got, bo = cdc.chunk_batch(_dev(data), offs, p)
    assert (bo.cpu().numpy() == exp_bo).all()
    assert (got.cpu().numpy().astype(np.uint64) == exp).all()


@pytest.mark.parametrize("algo", ALGOS)
def test_chain_api(cdc, algo):
    d = synth.uniform(1 << 20, 13)
    p = cdc.params(algo, window=500, max_size=3000)
    t = _dev(d)
    for start, stop in [(0, 1 << 20), (12345, 400000), (999999, 1 << 20), (5, 5)]:
        exp = oracle.chain_from(algo, d, start, stop, 500, 3000)
        got = cdc.chain(t, p, start, stop).cpu().numpy().astype(np.uint64)
        assert (got == exp).all() and got.size == exp.size


@pytest.mark.parametrize("algo", ALGOS)
def test_host_api(cdc, algo):
    d = synth.zipf_bytes((8 << 20) + 5, 1.1, 21)
    p = cdc.params(algo, avg_size=4096)
    exp = oracle.chunk(algo, d, p.window, p.max_size)
    got = cdc.chunk_host(d, p)
    assert (got == exp).all() and got.size == exp.size


def test_repeated_calls_same_workspace(cdc):
    """Published-list epochs: back-to-back calls reusing one workspace stay exact."""
    p = cdc.params("ae_max", avg_size=4096)
    d1, d2 = synth.zipf_bytes(8 << 20, 1.1, 31), synth.uniform(8 << 20, 32)
    t1, t2 = _dev(d1), _dev(d2)
    n = d1.size
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    cap = cdc.max_boundaries(p, n)
    b = torch.empty(cap, dtype=torch.int64, device="cuda")
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    for t, d in [(t1, d1), (t2, d2), (t1, d1), (t2, d2)]:
        cdc.chunk_async(t, p, b, c, ws)
        got = b[:int(c.item())].cpu().numpy().astype(np.uint64)
        exp = oracle.chunk("ae_max", d, p.window, p.max_size)
        assert (got == exp).all() and got.size == exp.size


def test_invalid_params(cdc):
    with pytest.raises(cdc.CdcError):
        cdc.chunk(torch.zeros(10, dtype=torch.uint8, device="cuda"), cdc.params("ram", window=4, max_size=4))
    with pytest.raises(cdc.CdcError):
        cdc.chunk(torch.zeros(10, dtype=torch.uint8, device="cuda"), cdc.params("ram", window=0, max_size=4))


@pytest.mark.parametrize("case", ["fast", "fixup"])
def test_cuda_graph_capture(cdc, case):
    """cdc_chunk captured into a CUDA graph (as bench.py times it): replays stay
    exact whether the fused fast path holds or the fix-up kernel has to resolve."""
    if case == "fast":
        d = synth.zipf_bytes(16 << 20, 1.1, 41)
        p = cdc.params("ae_max", avg_size=4096)
    else:  # constant bytes never re-synchronise: every halo gives up, the fix-up runs
        d = synth.constant((3 << 20) + 5, 0)
        p = cdc.params("ram", window=600, max_size=4000, seg_bytes=16384, halo_bytes=8192)
    exp = oracle.chunk(["ram", "ae_max", "ae_min"][p.algo], d, p.window, p.max_size)
    t = _dev(d)
    n = d.size
    ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
    cap = cdc.max_boundaries(p, n)
    b = torch.empty(cap, dtype=torch.int64, device="cuda")
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
    if case == "fixup":
        assert cdc.stats(p, ws, 1, n, n)["fast_path"] == 0


def test_concurrent_streams(cdc):
    """Two calls in flight at once on two CUDA streams, each with its own
    workspace (the device state of a call lives in its workspace): both exact."""
    d1 = synth.zipf_bytes((6 << 20) + 11, 1.1, 31)
    d2 = synth.uniform((16 << 20) + 5, 32)
    jobs = []
    for d, algo, avg in ((d1, "ae_max", 4096), (d2, "ram", 8192)):
        p = cdc.params(algo, avg_size=avg)
        t = _dev(d)
        n = d.size
        ws = torch.empty(cdc.workspace_size(p, 1, n, n), dtype=torch.uint8, device="cuda")
        b = torch.full((cdc.max_boundaries(p, n),), -1, dtype=torch.int64, device="cuda")
        c = torch.zeros(1, dtype=torch.int64, device="cuda")
        jobs.append((d, algo, p, t, ws, b, c, torch.cuda.Stream()))
    torch.cuda.synchronize()
    for _ in range(3):
        for d, algo, p, t, ws, b, c, s in jobs:
            with torch.cuda.stream(s):
                cdc.chunk_async(t, p, b, c, ws, s)
    torch.cuda.synchronize()
    for d, algo, p, t, ws, b, c, s in jobs:
        exp = oracle.chunk(algo, d, p.window, p.max_size)
        got = b[:int(c.item())].cpu().numpy().astype(np.uint64)
        assert got.size == exp.size and (got == exp).all(), algo
