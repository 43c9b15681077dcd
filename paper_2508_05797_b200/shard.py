"""Range sharding of one stream across ranks (north_star (4)).

A stream too large for one GPU, or one that should use all GPUs of a box, is
cut into `world` contiguous byte ranges [a_r, b_r).  Rank r holds its range
plus a halo of H bytes of the next range.  The protocol has five steps.

1. **Local pass.** Rank r chunks its buffer [a_r, min(L, b_r + H)) with the
   single-GPU pipeline (`cdc_chunk`), as if a chunk started at a_r. This is
   speculation.
   - The chain starts inside the range are its list S_r.
   - The starts of the same chain past b_r are its halo chain T_r. Only
     starts below b_r + H - max_size count: every chunk that starts there
     ends inside the buffer, so the truncated buffer end cannot have moved
     them.
2. **Exchange.** Every rank all-gathers |S_r|, the head of S_r (its starts
   below a_r + H) and T_r. Only segment-edge chain states cross NVLink, never
   bytes, and the exchange is one all_gather.
3. **Re-synchronisation.** `cdc_first_common(T_{r-1}, head(S_r))` finds the
   first start that rank r-1's chain shares with rank r's chain.
   Content-defined boundaries depend only on the bytes after a chunk start,
   so from that start on the two chains coincide. Rank r-1 keeps T_{r-1}
   before it. Rank r drops the S_r entries before it. Every rank computes
   every pair, so all ranks agree on the counts.
4. **Fix-up.** This is rare: it runs only when T_{r-1} never meets S_r inside
   the halo. Rank r walks the chain from the last start of T_{r-1} over its
   own bytes (`cdc_chain`) until the chain meets S_r. The starts it passes
   before that point are extra true starts of rank r. A second all_gather
   carries their counts.
5. **Output.** Rank r's true starts are U_r = extra_r ++ S_r[e_r:] ++
   T_r[:t_r]. The global boundary list (exclusive chunk ends) is the
   concatenation over ranks of U_r without the stream start 0, followed by L.
   Rank r's part starts at output offset sum_{r'<r} |U_r'|.

Rank 0's chain is the true chain; by induction each rank's list from its
entry on is too.  The functions take a `backend` with `chunk(buf, p)`,
`first_common(a, b)` and `chain(buf, p, start, stop)`.  The CUDA backend
below runs the library's kernels; the CPU tests inject one built on the
oracle to exercise this host logic over gloo.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


@dataclass
class ShardPlan:
    total: int      # stream length L
    world: int
    rank: int
    a: int          # range [a, b)
    b: int
    buf_end: int    # rank holds bytes [a, buf_end) = range + halo
    halo: int

    @property
    def last(self) -> bool:
        return self.rank == self.world - 1


def plan(total: int, world: int, rank: int, halo: int) -> ShardPlan:
    """Equal byte ranges; every range must be at least as long as the halo."""
    a = total * rank // world
    b = total * (rank + 1) // world
    if world > 1 and min(total * (r + 1) // world - total * r // world for r in range(world)) < halo:
        raise ValueError(f"shards of a {total}-byte stream over {world} ranks are shorter than the halo {halo}")
    return ShardPlan(total, world, rank, a, b, min(total, b + halo) if rank < world - 1 else total, halo)


def default_halo(max_size: int, window: int) -> int:
    """H: 64 MiB, and at least 64 max-size chunks -- chains re-synchronise within a
    few chunks on typical data and within ~3 MB at the 99th percentile on
    uniform bytes at 8 KiB."""
    return max(64 << 20, 64 * max_size, 64 * (window + 1))


class CudaBackend:
    """The product backend: the library's kernels through the thin binding."""

    def __init__(self):
        from . import api
        self.api = api

    def chunk(self, buf: torch.Tensor, p) -> torch.Tensor:
        return self.api.chunk(buf, p)

    def first_common(self, a: torch.Tensor, b: torch.Tensor) -> tuple[int, int]:
        if a.numel() == 0 or b.numel() == 0:
            return a.numel(), -1
        out = self.api.first_common(a, b).cpu()
        return int(out[0]), int(out[1])

    def chain(self, buf: torch.Tensor, p, start: int, stop: int) -> torch.Tensor:
        return self.api.chain(buf, p, start, stop)

    def chunk_batch(self, data: torch.Tensor, file_offsets, p):
        return self.api.chunk_batch(data, file_offsets, p)


@dataclass
class LocalPass:
    S: torch.Tensor   # chain starts inside [a, b), absolute, ascending (S[0] = a)
    T: torch.Tensor   # the same chain's trusted starts past b, absolute


def local_pass(buf: torch.Tensor, pl: ShardPlan, p, backend) -> LocalPass:
    """Step 1: speculative chunking of the rank's range + halo."""
    if buf.numel() != pl.buf_end - pl.a:
        raise ValueError("buffer does not match the shard plan")
    ends = backend.chunk(buf, p).to(torch.int64)
    starts = torch.cat([torch.zeros(1, dtype=torch.int64, device=ends.device), ends[:-1]]) + pl.a
    S = starts[starts < pl.b]
    if pl.last:
        T = starts[:0]
    else:
        trusted = pl.buf_end - int(p.max_size)
        T = starts[(starts >= pl.b) & (starts < trusted)]
    return LocalPass(S.contiguous(), T.contiguous())


class DistComm:
    """Collectives of the exchange over torch.distributed (NCCL over NVLink on
    the GPU box, gloo in the CPU tests)."""

    def __init__(self, group=None):
        self.group = group

    def all_gather(self, x: torch.Tensor) -> list[torch.Tensor]:
        import torch.distributed as dist
        out = [torch.empty_like(x) for _ in range(dist.get_world_size(self.group))]
        dist.all_gather(out, x, group=self.group)
        return out

    def all_reduce_sum(self, x: torch.Tensor) -> torch.Tensor:
        import torch.distributed as dist
        dist.all_reduce(x, group=self.group)
        return x


class ThreadComm:
    """The same collectives between threads of one process (one thread per
    emulated rank): used to exercise the protocol on a single GPU, where the
    ranks' kernels never wait on one another -- only the host threads meet."""

    def __init__(self, world: int):
        import threading
        self.world = world
        self._barrier = threading.Barrier(world)
        self._slots = [None] * world

    def _swap(self, rank: int, x: torch.Tensor) -> list[torch.Tensor]:
        self._slots[rank] = x.clone()
        self._barrier.wait()
        out = [t.to(x.device) for t in self._slots]
        self._barrier.wait()
        return out

    def for_rank(self, rank: int):
        comm = self

        class _R:
            rank = None

            def all_gather(self, x):
                return comm._swap(rank, x)

            def all_reduce_sum(self, x):
                parts = comm._swap(rank, x)
                x.copy_(torch.stack(parts).sum(0))
                return x
        r = _R()
        r.rank = rank
        return r


def exchange(lp: LocalPass, pl: ShardPlan, K: int, comm):
    """Step 2: all_gather of (|S_r|, |head_r|, |T_r|, head_r padded to K, T_r padded to K)."""
    dev = lp.S.device
    head = lp.S[lp.S < pl.a + pl.halo]
    if head.numel() > K or lp.T.numel() > K:
        raise RuntimeError("edge lists exceed the exchange capacity")
    msg = torch.full((3 + 2 * K,), -1, dtype=torch.int64, device=dev)
    msg[0] = lp.S.numel()
    msg[1] = head.numel()
    msg[2] = lp.T.numel()
    msg[3:3 + head.numel()] = head
    msg[3 + K:3 + K + lp.T.numel()] = lp.T
    parts = comm.all_gather(msg)
    nS = [int(m[0]) for m in parts]
    heads = [m[3:3 + int(m[1])] for m in parts]
    Ts = [m[3 + K:3 + K + int(m[2])] for m in parts]
    return nS, heads, Ts


def chunk_sharded(buf: torch.Tensor, pl: ShardPlan, p, backend=None, comm=None):
    """Steps 1-5 on this rank.  Returns (this rank's boundaries: int64 exclusive
    chunk ends of the global stream, absolute, ascending; their output offset;
    the global boundary count)."""
    backend = backend or CudaBackend()
    lp = local_pass(buf, pl, p, backend)
    W = pl.world
    if W == 1:
        U = torch.cat([lp.S[1:], torch.tensor([pl.total], dtype=torch.int64, device=lp.S.device)])
        return (U, 0, U.numel()) if pl.total > 0 else (U[:0], 0, 0)
    comm = comm or DistComm()
    K = pl.halo // (int(p.window) + 1) + 2
    nS, heads, Ts = exchange(lp, pl, K, comm)
    # step 3: every pair (r-1, r), computed identically on every rank
    entry = [0] * W                # e_r: index in S_r where the true chain enters
    tail = [len(t) for t in Ts]    # t_r: T_r entries on the true chain
    broken = []                    # pairs whose chains did not meet inside the halo
    for r in range(1, W):
        ia, ib = backend.first_common(Ts[r - 1], heads[r])
        if ib >= 0:
            entry[r], tail[r - 1] = ib, ia
        else:
            broken.append(r)
    # step 4: fix-up walk on each rank entered through a broken pair
    extra = None
    if pl.rank in broken:
        prev_T = Ts[pl.rank - 1]
        if prev_T.numel() == 0:
            raise RuntimeError("no trusted halo chain to continue; use a larger halo")
        s_last = int(prev_T[-1]) - pl.a
        walk = backend.chain(buf, p, s_last, buf.numel()).to(torch.int64)[1:] + pl.a  # starts after s_last
        ia, ib = backend.first_common(walk, lp.S)
        if ib < 0:
            raise RuntimeError("chains did not re-synchronise within one shard; use a larger halo")
        extra = walk[:ia]
        entry[pl.rank] = ib
    # step 5: counts (a second collective only when a fix-up ran) and this rank's output
    mine = (0 if extra is None else extra.numel()) + nS[pl.rank] - entry[pl.rank] + tail[pl.rank]
    if broken:
        c = torch.zeros(W, dtype=torch.int64, device=lp.S.device)
        c[pl.rank] = mine
        counts = [int(x) for x in comm.all_reduce_sum(c).cpu()]
    else:
        counts = [nS[r] - entry[r] + tail[r] for r in range(W)]
    counts[0] -= 1           # the stream start 0 is not a boundary
    counts[-1] += 1          # the stream length is the last boundary
    parts = ([extra] if extra is not None else []) + [lp.S[entry[pl.rank]:], lp.T[:tail[pl.rank]]]
    U = torch.cat(parts)
    if pl.rank == 0:
        U = U[1:]
    if pl.last:
        U = torch.cat([U, torch.tensor([pl.total], dtype=torch.int64, device=U.device)])
    return U, sum(counts[:pl.rank]), sum(counts)


# ---------------------------------------------------------------------- files
def file_range(offsets, world: int, rank: int) -> tuple[int, int]:
    """Files shard directly (north_star (4)): rank r takes the contiguous files
    [f0, f1) whose first bytes fall in the r-th of `world` equal byte ranges of
    the packed batch (byte-balanced, no file split; no data-path collective)."""
    import numpy as np
    offs = np.asarray(offsets, dtype=np.int64)
    nf = offs.size - 1
    total = int(offs[-1] - offs[0])

    def cut(r):
        if r <= 0:
            return 0
        if r >= world:
            return nf
        # first file starting at or after the r-th byte cut
        return int(np.searchsorted(offs[:-1], offs[0] + total * r // world, side="left"))
    return cut(rank), cut(rank + 1)


def chunk_files_sharded(data: torch.Tensor, file_offsets, p, comm=None, backend=None):
    """Chunk this rank's files (data: its packed bytes on the device; file_offsets:
    host int64[nf+1] relative to data) with one cdc_chunk_batch call, then one
    all_gather of the per-rank counts places its boundaries in the global list.
    Returns (bounds int64[m] per-file ends, bound_offsets int64[nf+1] local,
    this rank's output offset, the global boundary count)."""
    backend = backend or CudaBackend()
    bounds, bo = backend.chunk_batch(data, file_offsets, p)
    m = bounds.numel()
    if comm is None:
        return bounds, bo, 0, m
    x = torch.tensor([m], dtype=torch.int64, device=bounds.device)
    counts = [int(t.item()) for t in comm.all_gather(x)]
    rank = counts_rank(comm)
    return bounds, bo, sum(counts[:rank]), sum(counts)


def counts_rank(comm) -> int:
    r = getattr(comm, "rank", None)
    if r is not None:
        return r
    import torch.distributed as dist
    return dist.get_rank(getattr(comm, "group", None))
