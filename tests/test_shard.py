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

    def chunk_batch(self, data, offs, p):
        e, bo = oracle.chunk_batch(p.algo, data.numpy(), offs, p.window, p.max_size)
        return torch.from_numpy(e.astype(np.int64)), torch.from_numpy(bo)


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


# --------------------------------------------------------------------------
# file sharding (north_star (4): "files shard directly")
# --------------------------------------------------------------------------
def _files():
    data, offs = synth.many_files(400, seed=43, median=20000, sigma=1.5, cap=1 << 20)
    return data, offs, SimpleNamespace(algo="ram", window=1000, max_size=8000)


def _file_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        data, offs, p = _files()
        f0, f1 = shard.file_range(offs, world, rank)
        local = offs[f0:f1 + 1] - offs[f0]
        buf = torch.from_numpy(np.ascontiguousarray(data[offs[f0]:offs[f1]]))
        b, bo, off, total = shard.chunk_files_sharded(buf, local, p, shard.DistComm(), OracleBackend())
        np.save(os.path.join(out_dir, f"f{rank}.npy"), np.concatenate([[f0, f1, off, total], bo.numpy(), b.numpy()]))
    finally:
        dist.destroy_process_group()


def test_file_range_partitions_byte_balanced():
    _, offs, _ = _files()
    for world in (1, 2, 3, 8):
        rs = [shard.file_range(offs, world, r) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == offs.size - 1
        assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
        total = offs[-1]
        for f0, f1 in rs:  # every rank's bytes are within one largest file of the share
            assert abs(int(offs[f1] - offs[f0]) - total / world) <= int(np.diff(offs).max()) + 1


def test_files_gloo_world2(tmp_path):
    import torch.multiprocessing as tmp
    world = 2
    tmp.spawn(_file_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    data, offs, p = _files()
    exp, exp_bo = oracle.chunk_batch(p.algo, data, offs, p.window, p.max_size)
    got = []
    for r in range(world):
        a = np.load(tmp_path / f"f{r}.npy")
        f0, f1, off, total = (int(x) for x in a[:4])
        nf = f1 - f0
        bo = a[4:4 + nf + 1]
        b = a[4 + nf + 1:]
        assert total == exp.size and off == int(exp_bo[f0])
        assert (bo + off == exp_bo[f0:f1 + 1]).all()
        got.append(b)
    assert (np.concatenate(got).astype(np.uint64) == exp).all()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
def test_files_gpu_threads(world, cuda_ok):
    """File sharding with the CUDA backend, ranks emulated by host threads."""
    import paper_2508_05797_b200 as cdc
    data, offs, p0 = _files()
    p = cdc.params("ram", window=p0.window, max_size=p0.max_size)
    exp, exp_bo = oracle.chunk_batch("ram", data, offs, p.window, p.max_size)
    comm = shard.ThreadComm(world)
    res = [None] * world

    def work(r):
        f0, f1 = shard.file_range(offs, world, r)
        buf = torch.from_numpy(np.ascontiguousarray(data[offs[f0]:offs[f1]])).cuda()
        b, bo, off, total = shard.chunk_files_sharded(buf, offs[f0:f1 + 1] - offs[f0], p, comm.for_rank(r))
        res[r] = (f0, f1, b.cpu().numpy(), bo.cpu().numpy(), off, total)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for f0, f1, b, bo, off, total in res:
        assert total == exp.size and off == int(exp_bo[f0]) and (bo + off == exp_bo[f0:f1 + 1]).all()
    assert (np.concatenate([r[2] for r in res]).astype(np.uint64) == exp).all()


def _nccl_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    import paper_2508_05797_b200 as cdc
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        comm = shard.DistComm()
        data, exp, p0 = _expected("ram_zipf")
        p = cdc.params("ram", window=p0.window, max_size=p0.max_size)
        pl = shard.plan(data.size, world, rank, CASES["ram_zipf"][5])
        U, off, total = shard.chunk_sharded(torch.from_numpy(data).cuda(), pl, p, shard.CudaBackend(), comm)
        # a real NCCL collective on the exchange's message shape
        x = torch.arange(5, dtype=torch.int64, device="cuda")
        parts = comm.all_gather(x)
        y = comm.all_reduce_sum(torch.ones(3, dtype=torch.int64, device="cuda"))
        fd, fo, fp = _files()
        pf = cdc.params("ram", window=fp.window, max_size=fp.max_size)
        b, bo, foff, ftotal = shard.chunk_files_sharded(torch.from_numpy(fd).cuda(), fo, pf, comm)
        np.save(os.path.join(out_dir, "nccl.npy"), np.concatenate(
            [[off, total, len(parts), int(parts[0].sum()), int(y.sum()), foff, ftotal], U.cpu().numpy(),
             b.cpu().numpy()]))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_distcomm_nccl_world1(cuda_ok, tmp_path):
    """DistComm over a real NCCL process group (world size 1: gpurun has one GPU)
    runs the range-sharded and file-sharded paths end to end."""
    import torch.multiprocessing as tmp
    tmp.spawn(_nccl_worker, args=(1, _free_port(), str(tmp_path)), nprocs=1, join=True)
    a = np.load(tmp_path / "nccl.npy")
    off, total, nparts, s, ysum, foff, ftotal = (int(x) for x in a[:7])
    _, exp, _ = _expected("ram_zipf")
    fd, fo, fp = _files()
    fexp, _ = oracle.chunk_batch("ram", fd, fo, fp.window, fp.max_size)
    assert (off, total, nparts, s, ysum, foff, ftotal) == (0, exp.size, 1, 10, 3, 0, fexp.size)
    assert (a[7:7 + total] == exp).all()
    assert (a[7 + total:].astype(np.uint64) == fexp).all()
