"""Range sharding of one stream across ranks (paper_2508_05797_b200/shard.py).

CPU: the host protocol over real torch.distributed gloo (world size 2) and over
threads (world size 4), with an oracle-backed backend standing in for the GPU
kernels.  GPU: the same protocol with the CUDA backend, ranks emulated by host
threads on one GPU (their kernels never wait on one another).  Expected
boundaries always come from oracle.chunk on the whole stream.
"""
import os
import socket
import threading
from types import SimpleNamespace

import numpy as np
import pytest
import torch

import oracle
import synth
from paper_2508_05797_b200 import shard


class OracleBackend:
    """Test-only stand-in for the CUDA kernels (CPU tensors)."""

    def chunk(self, buf, p):
        return torch.from_numpy(oracle.chunk(p.algo, buf.numpy(), p.window, p.max_size).astype(np.int64))

    def first_common(self, a, b):
        a, b = a.numpy(), b.numpy()
        hit = np.isin(a, b)
        if not hit.any():
            return a.size, -1
        i = int(np.argmax(hit))
        return i, int(np.searchsorted(b, a[i]))

    def chain(self, buf, p, start, stop):
        return torch.from_numpy(oracle.chain_from(p.algo, buf.numpy(), start, stop, p.window, p.max_size)
                                .astype(np.int64))


CASES = {
    # name: (algo, generator, n, w, max_size, halo)
    "ram_zipf": ("ram", lambda n: synth.zipf_bytes(n, 1.1, 3), 3 << 20, 300, 1200, 64 << 10),
    "ae_max_uniform": ("ae_max", lambda n: synth.uniform(n, 4), 3 << 20, 400, 1600, 96 << 10),
    "ae_min_runs": ("ae_min", lambda n: synth.alternating(n, region=1 << 18, seed=5), 3 << 20, 250, 1000,
                    64 << 10),
    # a halo too short for the chains to meet: exercises the fix-up walk
    "ram_uniform_fixup": ("ram", lambda n: synth.uniform(n, 6), 2 << 20, 2000, 8000, 12000),
}


def _expected(case):
    algo, gen, n, w, mx, halo = CASES[case]
    data = gen(n)
    return data, oracle.chunk(algo, data, w, mx).astype(np.int64), SimpleNamespace(algo=algo, window=w, max_size=mx)


def _run_rank(rank, world, data, p, halo, comm, backend, to=None):
    pl = shard.plan(data.size, world, rank, halo)
    buf = torch.from_numpy(np.ascontiguousarray(data[pl.a:pl.buf_end]))
    if to is not None:
        buf = buf.to(to)
    U, off, total = shard.chunk_sharded(buf, pl, p, backend, comm)
    return U.cpu().numpy(), off, total


def _check(parts, exp):
    totals = {t for _, _, t in parts}
    assert totals == {exp.size}
    got = np.concatenate([u for u, _, _ in parts])
    offs = [o for _, o, _ in parts]
    assert offs == sorted(offs) and offs[0] == 0
    assert got.size == exp.size and (got == exp).all()


def _gloo_worker(rank, world, port, case, out_dir):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        data, exp, p = _expected(case)
        halo = CASES[case][5]
        U, off, total = _run_rank(rank, world, data, p, halo, shard.DistComm(), OracleBackend())
        np.save(os.path.join(out_dir, f"r{rank}.npy"), np.concatenate([[off, total], U]))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", list(CASES))
def test_shard_gloo_world2(case, tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_gloo_worker, args=(world, _free_port(), case, str(tmp_path)), nprocs=world, join=True)
    _, exp, _ = _expected(case)
    parts = []
    for r in range(world):
        a = np.load(tmp_path / f"r{r}.npy")
        parts.append((a[2:], int(a[0]), int(a[1])))
    _check(parts, exp)


def _threads(world, data, p, halo, backend, to=None):
    comm = shard.ThreadComm(world)
    res = [None] * world
    errs = []

    def work(r):
        try:
            res[r] = _run_rank(r, world, data, p, halo, comm.for_rank(r), backend, to)
        except BaseException as e:  # surface worker failures
            errs.append(e)
            comm._barrier.abort()

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return res


class CountingBackend(OracleBackend):
    def __init__(self):
        self.walks = 0

    def chain(self, buf, p, start, stop):
        self.walks += 1
        return super().chain(buf, p, start, stop)


@pytest.mark.parametrize("world", [3, 4])
@pytest.mark.parametrize("case", ["ram_zipf", "ae_max_uniform", "ram_uniform_fixup"])
def test_shard_threads_oracle(case, world):
    data, exp, p = _expected(case)
    be = CountingBackend()
    _check(_threads(world, data, p, CASES[case][5], be), exp)
    if case.endswith("fixup"):
        assert be.walks > 0  # the fix-up walk ran


def test_shard_plan_rejects_short_shards():
    with pytest.raises(ValueError):
        shard.plan(1000, 4, 0, 300)


@pytest.mark.gpu
@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("world", [2, 4])
def test_shard_gpu_threads(case, world, cuda_ok):
    import paper_2508_05797_b200 as cdc
    data, exp, p0 = _expected(case)
    p = cdc.params(p0.algo, window=p0.window, max_size=p0.max_size)
    _check(_threads(world, data, p, CASES[case][5], shard.CudaBackend(), to="cuda"), exp)


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["ram", "ae_max"])
def test_shard_gpu_config4_shape(algo, cuda_ok):
    """BASELINE configs[4] shape, scaled: alternating uniform / low-entropy regions,
    8 KiB average, split across 8 emulated ranks with the default halo."""
    import paper_2508_05797_b200 as cdc
    data = synth.alternating(1 << 30, region=64 << 20, seed=5)
    p = cdc.params(algo, avg_size=8192)
    exp = oracle.chunk(algo, data, p.window, p.max_size).astype(np.int64)
    halo = shard.default_halo(p.max_size, p.window)
    _check(_threads(8, data, p, halo, shard.CudaBackend(), to="cuda"), exp)
