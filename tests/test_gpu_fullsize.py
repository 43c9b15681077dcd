"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
uses (default segmenting, one cdc_chunk / cdc_chunk_batch call per stream).

The oracle cannot chunk tens of GiB within a test, so each run is checked two
ways:
- **Properties over every chunk** (vectorised): the boundaries tile the stream,
  every chunk is at most max_size, and every content chunk is longer than the
  window (the only minimum the paper's rules imply).
- **The oracle on sampled chunks.** A chunk's end is a function of its start
  and the bytes after it (§2.1.2), so oracle.chunk_end(start) must
  reproduce the GPU's end exactly. The sample is random, plus the first and
  last chunks of every speculation segment's neighbourhood and of the stream.

configs[0] and configs[1] are compared element by element in
test_gpu_parity.py; configs[2]'s dedup savings are compared with the oracle's
at reduced size there as well.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cdc(cuda_ok):
    import paper_2508_05797_b200 as m
    return m


def _verify(algo, data, ends, w, mx, n_samples=3000, seed=0, extra_starts=()):
    ends = np.asarray(ends, dtype=np.int64)
    L = data.size
    assert ends.size > 0 and ends[-1] == L
    starts = np.concatenate([[0], ends[:-1]])
    lens = ends - starts
    assert (lens > 0).all() and (lens <= mx).all()
    assert (lens[:-1] >= w + 1).all()
    rng = np.random.default_rng(seed)
    pick = set(rng.integers(0, ends.size, min(n_samples, ends.size)).tolist())
    pick.update([0, ends.size - 1, max(0, ends.size - 2)])
    for x in extra_starts:  # chunks around segment boundaries (where the splice happens)
        i = int(np.searchsorted(starts, x, side="right")) - 1
        pick.update([max(0, i - 1), i, min(ends.size - 1, i + 1)])
    for i in sorted(pick):
        e = oracle.chunk_end(algo, data, int(starts[i]), w, mx)
        assert e == ends[i], (algo, i, int(starts[i]), int(ends[i]), e)


def _seg_edges(cdc, p, n, k=400):
    """Up to k speculation segment starts (where chains are spliced), evenly picked."""
    st = cdc.segment_starts(p, n)
    return st[:: max(1, len(st) // k)]


def test_config2_full_versioned(cdc):
    """BASELINE configs[2] at full size: 1 GiB base + 9 snapshots, AE and RAM at 4/8/16 KiB."""
    snaps = synth.versioned(1 << 30, 9, seed=2)
    for si, s in enumerate(snaps):
        t = torch.from_numpy(s).cuda()
        for algo in ("ae_max", "ram"):
            for avg in (4096, 8192, 16384):
                if si % 3 != (avg // 4096) % 3 and si not in (0, 9):
                    continue  # every snapshot with some average, the first and last with all
                p = cdc.params(algo, avg_size=avg)
                ends = cdc.chunk(t, p).cpu().numpy()
                _verify(algo, s, ends, p.window, p.max_size, n_samples=600, seed=si * 7 + avg,
                        extra_starts=_seg_edges(cdc, p, s.size))
        del t
        torch.cuda.empty_cache()


def test_config3_full_many_files(cdc):
    """BASELINE configs[3], one GPU's share at 8 GPUs: 12,500 of the 100,000 lognormal files
    (median 64 KiB, sigma 1.5, capped at 16 MiB: ~2.3 GiB; the stated distribution gives
    ~18.7 GiB for all 100,000, not the ~8 GiB BASELINE.json quotes), RAM 8 KiB, one batch call."""
    data, offs = synth.many_files(12_500, seed=3)
    p = cdc.params("ram", avg_size=8192)
    got, bo = cdc.chunk_batch(torch.from_numpy(data).cuda(), offs, p)
    got, bo = got.cpu().numpy(), bo.cpu().numpy()
    assert bo[0] == 0 and bo[-1] == got.size and (np.diff(bo) >= 0).all()
    rng = np.random.default_rng(3)
    files = set(rng.integers(0, offs.size - 1, 1500).tolist())
    files.update(np.argsort(np.diff(offs))[-20:].tolist())  # the largest files (multi-segment)
    files.update([0, offs.size - 2])
    for f in sorted(files):
        a, b = int(offs[f]), int(offs[f + 1])
        ends = got[bo[f]:bo[f + 1]]
        if b == a:
            assert ends.size == 0
            continue
        _verify("ram", data[a:b], ends, p.window, p.max_size, n_samples=40, seed=f)


@pytest.mark.parametrize("algo", ["ram", "ae_max"])
def test_config4_full_shard(cdc, algo):
    """BASELINE configs[4] per GPU: one 8 GiB range of the 64 GiB alternating stream
    (256 MiB regions of uniform and run-length bytes), chunked in one call."""
    data = synth.alternating(8 << 30, region=256 << 20, seed=5)
    p = cdc.params(algo, avg_size=8192)
    ends = cdc.chunk(torch.from_numpy(data).cuda(), p).cpu().numpy()
    _verify(algo, data, ends, p.window, p.max_size, n_samples=3000, seed=11,
            extra_starts=_seg_edges(cdc, p, data.size) + [r << 28 for r in range(1, 32)])
