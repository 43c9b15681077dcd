"""Seeded random parity sweep: algorithm, window, cap, segment and halo sizes,
data kind and length drawn at random (fixed seed), every case compared with the
oracle bit for bit.  Covers the corners the targeted tests do not combine:
odd windows, caps just above the window, segments of a few windows, halos
shorter than a chunk, and transfer-table candidates (w >= 4096 on uniform
bytes)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

ALGOS = ["ram", "ae_max", "ae_min"]


def _data(kind, n, seed):
    if kind == "uniform":
        return synth.uniform(n, seed)
    if kind == "zipf":
        return synth.zipf_bytes(n, 1.1, seed)
    if kind == "runs":
        return synth.alternating(n, region=1 << 16, seed=seed)
    if kind == "satedge":
        return synth.saturation_edges(n, seed)
    rng = np.random.default_rng(seed)  # "small": a 4-letter alphabet
    return rng.integers(0, 4, n).astype(np.uint8)


def _cases(count=48, seed=20261020):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        algo = ALGOS[rng.integers(0, 3)]
        kind = ["uniform", "zipf", "runs", "satedge", "small"][rng.integers(0, 5)]
        if i % 6 == 0:  # transfer-table candidates
            algo, kind = ALGOS[(i // 6) % 3], "uniform"
            w = int(rng.integers(4096, 12000))
        else:
            w = int(rng.choice([1, 3, 17, 255, 256, 511, 1000, 2047, 3840, 5000]))
        mx = w + 1 + int(rng.choice([0, 1, 7, 300, 4 * w]))
        n = int(rng.integers(1, 2 << 20))
        seg = int(rng.choice([0, 0, 4096, 16384, 65536, 262144]))
        halo = int(rng.choice([0, 0, 0, 8192, 100000]))
        out.append((i, algo, kind, w, mx, n, seg, halo))
    return out


@pytest.fixture(scope="module")
def cdc(cuda_ok):
    import paper_2508_05797_b200 as m
    return m


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"c{c[0]}-{c[1]}-{c[2]}-w{c[3]}")
def test_fuzz(cdc, case):
    i, algo, kind, w, mx, n, seg, halo = case
    d = _data(kind, n, 100 + i)
    p = cdc.params(algo, window=w, max_size=mx, seg_bytes=seg, halo_bytes=halo)
    exp = oracle.chunk(algo, d, w, mx)
    got = cdc.chunk(torch.from_numpy(d).cuda(), p).cpu().numpy().astype(np.uint64)
    assert got.size == exp.size and (got == exp).all(), case


def _batch_cases(count=16, seed=20261021):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        algo = ALGOS[i % 3]
        kind = ["uniform", "zipf", "runs", "satedge", "small"][rng.integers(0, 5)]
        w = int(rng.choice([1, 17, 256, 1000, 3840, 6000]))
        mx = w + 1 + int(rng.choice([0, 5, 3 * w]))
        nfiles = int(rng.integers(1, 400))
        # a length mix: empty, shorter than a window, a few chunks, long files
        sizes = rng.choice([0, 1, 7, w, w + 1, 5000, 70000, 300000], nfiles,
                           p=[.1, .05, .05, .05, .05, .3, .3, .1]).astype(np.int64)
        sizes = sizes + rng.integers(0, 3, nfiles) * (sizes > 0)
        seg = int(rng.choice([0, 0, 8192, 65536]))
        out.append((i, algo, kind, w, mx, seg, sizes))
    return out


@pytest.mark.parametrize("case", _batch_cases(), ids=lambda c: f"b{c[0]}-{c[1]}-{c[2]}-w{c[3]}")
def test_fuzz_batch(cdc, case):
    i, algo, kind, w, mx, seg, sizes = case
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    d = _data(kind, max(int(offs[-1]), 1), 500 + i)[:int(offs[-1])]
    p = cdc.params(algo, window=w, max_size=mx, seg_bytes=seg)
    exp, exp_bo = oracle.chunk_batch(algo, d, offs, w, mx)
    got, bo = cdc.chunk_batch(torch.from_numpy(d).cuda(), offs, p)
    assert (bo.cpu().numpy() == exp_bo).all()
    assert (got.cpu().numpy().astype(np.uint64) == exp).all()


@pytest.mark.parametrize("i", range(6))
def test_fuzz_large(cdc, i):
    """Streams of 24-64 MiB: many segments per CTA, fused look-back, halos."""
    rng = np.random.default_rng(7000 + i)
    algo = ALGOS[i % 3]
    kind = ["zipf", "uniform", "runs", "satedge", "zipf", "uniform"][i]
    n = int(rng.integers(24 << 20, 64 << 20))
    avg = int(rng.choice([512, 2048, 4096, 8192]))
    d = _data(kind, n, 900 + i)
    p = cdc.params(algo, avg_size=avg)
    exp = oracle.chunk(algo, d, p.window, p.max_size)
    got = cdc.chunk(torch.from_numpy(d).cuda(), p).cpu().numpy().astype(np.uint64)
    assert got.size == exp.size and (got == exp).all(), (i, algo, kind, n, avg)
