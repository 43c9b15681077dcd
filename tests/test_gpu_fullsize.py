"""Element-wise parity at BASELINE.json's full sizes, in the launch
configuration bench.py uses (default segmenting, one cdc_chunk /
cdc_chunk_batch call per stream or batch, or shard.chunk_sharded for the
range-sharded stream).

Every chunk of every output is checked against the oracle: each GPU boundary
must equal oracle.chunk_end(previous boundary) (oracle.check_chunking /
check_batch, split over the host's cores).  By induction from the stream
start that is exactly oracle.chunk's output -- a chunk's end is a function of
its start and the bytes after it (§2.1.2) -- so these are full
comparisons, not samples.  Dedup space savings (Eq. 1) of configs[2] follow
from the verified boundaries and are computed with oracle.dedup.

Sizes: configs[2] 1 GiB base + 9 snapshots, AE-Max and RAM at 4/8/16 KiB (60
streams); configs[3] all 100,000 files (~18.7 GiB: the stated lognormal gives
that, not the ~8 GiB BASELINE.json quotes); configs[4] one GPU's 8 GiB range,
and the whole 64 GiB stream range-sharded over 8 ranks emulated by host
threads on one B200 (their kernels never wait on one another).
"""
import multiprocessing as mp
import threading

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import dedup

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cdc(cuda_ok):
    import paper_2508_05797_b200 as m
    return m


def _ok(algo, data, ends, p):
    bad = oracle.check_chunking(algo, data, np.asarray(ends, dtype=np.uint64), p.window, p.max_size)
    assert bad is None, (algo, p.window, data.size, bad)


_DEDUP = {}


def _dedup_job(key):
    streams, ends = _DEDUP[key]
    return key, dedup.unique_bytes(streams, ends)


def test_config2_full_versioned(cdc):
    """BASELINE configs[2]: 1 GiB base + 9 snapshots; AE-Max and RAM at 4/8/16 KiB;
    every chunk of every snapshot verified; dedup savings from the verified chunks."""
    snaps = synth.versioned(1 << 30, 9, seed=2)
    ends = {}
    for si, s in enumerate(snaps):
        t = torch.from_numpy(s).cuda()
        for algo in ("ae_max", "ram"):
            for avg in (4096, 8192, 16384):
                p = cdc.params(algo, avg_size=avg)
                e = cdc.chunk(t, p).cpu().numpy().astype(np.uint64)
                _ok(algo, s, e, p)
                ends.setdefault((algo, avg), []).append(e)
        del t
        torch.cuda.empty_cache()
    # Eq. (1) over the 10 versions, one process per (algo, avg) (fork: the
    # arrays are shared copy-on-write)
    for k, v in ends.items():
        _DEDUP[k] = (snaps, v)
    with mp.get_context("fork").Pool(len(ends)) as pool:
        res = dict(pool.map(_dedup_job, list(ends)))
    _DEDUP.clear()
    for (algo, avg), (total, uniq) in sorted(res.items()):
        assert total == sum(s.size for s in snaps)
        sv = dedup.space_savings(total, uniq)
        # ten versions of one base, ~1 % edited per version: a large share of the
        # chunks recur (less at larger chunks: an edit spoils a whole chunk)
        assert 20.0 < sv < 90.0, (algo, avg, sv)
        print(f"configs[2] {algo} {avg}: savings {sv:.3f} % ({total} -> {uniq} bytes)")


def test_config3_full_many_files(cdc):
    """BASELINE configs[3] at full size: all 100,000 lognormal files (median 64 KiB,
    sigma 1.5, capped at 16 MiB; ~18.7 GiB), RAM 8 KiB, one cdc_chunk_batch call
    (bench.py's workload); every file's every chunk verified."""
    data, offs = synth.many_files(100_000, seed=3)
    p = cdc.params("ram", avg_size=8192)
    t = torch.from_numpy(data).cuda()
    got, bo = cdc.chunk_batch(t, offs, p)
    got, bo = got.cpu().numpy().astype(np.uint64), bo.cpu().numpy().astype(np.uint64)
    del t
    torch.cuda.empty_cache()
    assert bo[0] == 0 and int(bo[-1]) == got.size
    bad = oracle.check_batch("ram", data, offs, got, bo, p.window, p.max_size)
    assert bad is None, bad


def test_config3_full_host_entry(cdc):
    """configs[3] through the end-to-end host entry point (cdc_chunk_batch_host:
    grouped, pipelined copies) equals the oracle too."""
    data, offs = synth.many_files(100_000, seed=3)
    p = cdc.params("ram", avg_size=8192)
    got, bo = cdc.chunk_batch_host(data, offs, p)
    assert int(bo[-1]) == got.size
    bad = oracle.check_batch("ram", data, offs, got, bo, p.window, p.max_size)
    assert bad is None, bad


@pytest.mark.parametrize("algo", ["ram", "ae_max"])
def test_config4_full_range(cdc, algo):
    """BASELINE configs[4] per GPU: one 8 GiB range of the 64 GiB alternating stream
    (256 MiB regions of uniform and run-length bytes), chunked in one call."""
    data = synth.alternating(8 << 30, region=256 << 20, seed=5)
    p = cdc.params(algo, avg_size=8192)
    ends = cdc.chunk(torch.from_numpy(data).cuda(), p).cpu().numpy()
    torch.cuda.empty_cache()
    _ok(algo, data, ends, p)


def test_config4_full_sharded_64gib(cdc):
    """BASELINE configs[4] at full size: the whole 64 GiB stream split by byte range
    with a halo across 8 ranks (shard.chunk_sharded, north_star (4)), AE-Max and
    RAM at 8 KiB; the concatenated per-rank boundaries verified chunk by chunk."""
    from paper_2508_05797_b200 import shard
    L = 64 << 30
    data = synth.alternating(L, region=256 << 20, seed=5)
    world = 8
    for algo in ("ram", "ae_max"):
        p = cdc.params(algo, avg_size=8192)
        halo = shard.default_halo(p.max_size, p.window)
        comm = shard.ThreadComm(world)
        res = [None] * world
        errs = []

        def work(r):
            try:
                pl = shard.plan(L, world, r, halo)
                buf = torch.from_numpy(data[pl.a:pl.buf_end]).cuda()
                U, off, total = shard.chunk_sharded(buf, pl, p, shard.CudaBackend(), comm.for_rank(r))
                res[r] = (U.cpu().numpy(), off, total)
                del buf
            except BaseException as e:
                errs.append(e)
                comm._barrier.abort()

        th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        if errs:
            raise errs[0]
        torch.cuda.empty_cache()
        offs = [o for _, o, _ in res]
        assert offs == sorted(offs) and offs[0] == 0
        assert len({t for _, _, t in res}) == 1
        got = np.concatenate([u for u, _, _ in res]).astype(np.uint64)
        assert got.size == res[0][2]
        for r in range(world):
            assert res[r][1] == (res[r + 1][1] if r + 1 < world else got.size) - res[r][0].size
        _ok(algo, data, got, p)
