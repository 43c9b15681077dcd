"""GPU parity of the sparse walk (sparse_chain / walk_chain) and
of the round-2 batch pipeline (multi-CTA segment table, largest-first tickets,
half-share segments, batch_resolve) against the CPU oracle.

The sparse walk runs for windows of at least 4096 bytes; these cases use such
windows on streams that switch between saturated and unsaturated stretches
(every sparse -> ring -> sparse hand-over), caps at and just above the window
(capped chunks inside the sparse walk), files whose ends fall inside a
speculative copy, and batches whose long files are cut into segments whose
halos jump over segments or reach the file's end.  Every comparison is
bit-exact; expected values come only from oracle/.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ALGOS = ["ram", "ae_max", "ae_min"]


@pytest.fixture(scope="module")
def cdc(cuda_ok):
    import paper_2508_05797_b200 as m
    return m


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _check_stream(cdc, d, algo, w, mx, seg=0, halo=0):
    p = cdc.params(algo, window=w, max_size=mx, seg_bytes=seg, halo_bytes=halo)
    exp = oracle.chunk(algo, d, w, mx)
    got = cdc.chunk(_dev(d), p).cpu().numpy().astype(np.uint64)
    assert got.size == exp.size, (got.size, exp.size)
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, (int(bad[0]), int(got[bad[0]]), int(exp[bad[0]]))


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("w", [4096, 6000, 9000])
def test_sparse_switching(cdc, algo, w):
    """Saturated and unsaturated stretches of 2-64 KiB: the walk hands over to
    the ring walker and back many times per segment, in bodies and in halos."""
    d = synth.patchwork((6 << 20) + 333, seed=w)
    for mx, seg, halo in [(4 * w, 0, 0), (w + 300, 65536, 0), (2 * w, 131072, 4 * w)]:
        _check_stream(cdc, d, algo, w, mx, seg, halo)


@pytest.mark.parametrize("algo", ALGOS)
def test_sparse_tight_caps(cdc, algo):
    """Caps at w+1 .. w+64 on saturated bytes: most chunks end at the cap."""
    d = synth.uniform((3 << 20) + 77, 21)
    for w, mx in [(4096, 4097), (4096, 4100), (5000, 5064), (8192, 8192 + 17)]:
        _check_stream(cdc, d, algo, w, mx)


@pytest.mark.parametrize("algo", ALGOS)
def test_sparse_saturating_constant(cdc, algo):
    """Constant 0xFF / 0x00 stretches (every byte saturating for one side) and
    streams shorter than a few windows."""
    for d in (synth.constant(1 << 20, 255), synth.constant(1 << 20, 0),
              np.concatenate([synth.uniform(50000, 3), synth.constant(70000, 255), synth.uniform(90000, 4)])):
        for w, mx in [(4096, 16384), (4096, 4097), (10000, 40001)]:
            _check_stream(cdc, d, algo, w, mx)
    for n in [0, 1, 4095, 4096, 4097, 8193, 12289]:
        _check_stream(cdc, synth.uniform(n, n + 1), algo, 4096, 16384)


@pytest.mark.parametrize("algo", ALGOS)
def test_sparse_file_ends(cdc, algo):
    """A batch of saturated files whose ends fall at every offset of a
    speculative copy (lengths around w, 2w+1, and the copy size), the last one
    ending at the end of the buffer."""
    w, mx = 4096, 16384
    sizes = []
    for base in (w - 1, w, w + 1, 2 * w, 2 * w + 1, 2 * w + 2048, 3 * w + 100):
        sizes += [base + k for k in (0, 1, 15, 16, 17, 511, 1024, 2047)]
    sizes = np.array(sizes, dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    data = synth.uniform(int(offs[-1]), 31)
    p = cdc.params(algo, window=w, max_size=mx)
    exp, exp_bo = oracle.chunk_batch(algo, data, offs, w, mx)
    got, bo = cdc.chunk_batch(_dev(data), offs, p)
    assert (bo.cpu().numpy() == exp_bo).all()
    assert (got.cpu().numpy().astype(np.uint64) == exp).all()


@pytest.mark.parametrize("algo", ALGOS)
def test_sparse_chain_api(cdc, algo):
    """cdc_chain from interior starts (its single warp takes the sparse walk)."""
    d = synth.patchwork(2 << 20, seed=5)
    p = cdc.params(algo, window=5000, max_size=20000)
    t = _dev(d)
    for start, stop in [(0, d.size), (12345, 1 << 20), (777777, d.size), (d.size - 9000, d.size)]:
        exp = oracle.chain_from(algo, d, start, stop, 5000, 20000)
        got = cdc.chain(t, p, start, stop).cpu().numpy().astype(np.uint64)
        assert got.size == exp.size and (got == exp).all(), (start, stop)


def _batch(cdc, algo, data, offs, p):
    exp, exp_bo = oracle.chunk_batch(algo, data, offs, p.window, p.max_size)
    got, bo = cdc.chunk_batch(_dev(data), offs, p)
    assert (bo.cpu().numpy() == exp_bo).all()
    got = got.cpu().numpy().astype(np.uint64)
    assert got.size == exp.size
    bad = np.nonzero(got != exp)[0]
    assert bad.size == 0, int(bad[0])


@pytest.mark.parametrize("algo", ["ram", "ae_max"])
def test_batch_long_files_split(cdc, algo):
    """Long uniform and Zipf files among small and empty ones, at 8 KiB: the
    long ones go first (size classes 1 .. >= 32 MiB) and are cut into segments
    whose halos re-synchronise slowly (saturated bytes), jump over segments or
    reach the file's end; with forced small segments too."""
    rng = np.random.default_rng(41)
    sizes = list(rng.integers(0, 70000, 300)) + [0] * 20
    sizes += [1 << 20, (3 << 20) + 5, (9 << 20) + 11, 17 << 20, (33 << 20) + 3, 5 << 20]
    sizes = np.array(rng.permutation(sizes), dtype=np.int64)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    data = np.empty(int(offs[-1]), dtype=np.uint8)
    for i in range(sizes.size):  # per-file content: uniform or Zipf, alternating
        a, b = int(offs[i]), int(offs[i + 1])
        data[a:b] = synth.uniform(b - a, 100 + i) if i % 2 else synth.zipf_bytes(b - a, 1.1, 2003)
    for seg in (0, 262144):
        _batch(cdc, algo, data, offs, cdc.params(algo, avg_size=8192, seg_bytes=seg))


@pytest.mark.parametrize("algo", ALGOS)
def test_batch_many_tiles(cdc, algo):
    """12,000 files (12 segment-table tiles, 6 resolve tiles) with a third
    empty: the multi-CTA segment table and batch_resolve's phases."""
    rng = np.random.default_rng(42)
    sizes = rng.integers(0, 20000, 12000)
    sizes[rng.random(12000) < 0.33] = 0
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    data = synth.patchwork(int(offs[-1]), seed=9, piece_lo=512, piece_hi=8192)
    _batch(cdc, algo, data, offs, cdc.params(algo, window=4500, max_size=18000))
    _batch(cdc, algo, data, offs, cdc.params(algo, window=700, max_size=3000))
