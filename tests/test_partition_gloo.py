"""CPU, world_size 2 over gloo: the multi-rank driver of the hash-partitioned
fixpoint (partition.run_partitioned + TorchExchange: counts all-to-all,
rows all-to-all-v, |Δ| all-reduce termination) is exercised end to end with
a host-side stand-in for the per-rank device engine.  The stand-in
implements the same begin/end protocol as gd_engine_partition_* with plain
set semantics (test-only), so the union of the ranks' relations must equal
the transitive closure computed directly."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


class HostShard:
    """Per-rank TC shard with the gd_engine_partition_* protocol."""

    def __init__(self, edges, rank, nranks):
        self.edges = {tuple(map(int, e)) for e in edges}
        self.by_dst = {}
        for a, b in self.edges:
            self.by_dst.setdefault(b, []).append(a)
        self.rank, self.P = rank, nranks
        mine = {e for e in self.edges if self.owner(e) == rank}
        self.full, self.delta = set(mine), set(mine)
        self.iterations = 0

    def owner(self, t):
        return (t[0] * 1000003 + t[1]) % self.P

    def exchange_words(self):
        return 1

    def partition_begin(self, P):
        new = {(a, c) for (b, c) in self.delta for a in self.by_dst.get(b, ())}
        groups = [sorted(t for t in new if self.owner(t) == k) for k in range(P)]
        self.send = np.array([(a << 32) | c for g in groups for (a, c) in g], dtype=np.int64)
        counts = np.array([len(g) for g in groups], dtype=np.uint64)
        return counts, (self.send.ctypes.data if len(self.send) else 0)

    def partition_end(self, ptr, rows):
        import ctypes
        got = set()
        if rows:
            arr = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_int64)), shape=(rows,))
            got = {(int(x) >> 32, int(x) & 0xFFFFFFFF) for x in arr}
        assert all(self.owner(t) == self.rank for t in got)
        self.delta = got - self.full
        self.full |= self.delta
        self.iterations += 1
        return len(self.delta)


def closure(edges):
    e = {tuple(map(int, x)) for x in edges}
    reach = set(e)
    while True:
        new = {(a, d) for (a, b) in e for (c, d) in reach if b == c} - reach
        if not new:
            return reach
        reach |= new


def _worker(rank, world, port, edges, out):
    import torch.distributed as dist

    from paper_2311_02206_b200.partition import TorchExchange, run_partitioned

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    shard = HostShard(edges, rank, world)
    it = run_partitioned(shard, TorchExchange(device="cpu"), world)
    out[rank] = (sorted(shard.full), it)
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("seed", [1, 2])
def test_partitioned_driver_gloo_world2(seed):
    rng = np.random.default_rng(seed)
    edges = rng.integers(0, 40, size=(90, 2))
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, free_port(), edges, out), nprocs=world, join=True,
                       start_method="spawn")
    union = set()
    for r in range(world):
        rows, it = out[r]
        union |= {tuple(x) for x in rows}
        assert it == out[0][1]  # all ranks stop on the same iteration
    assert union == closure(edges)
    # shards are disjoint
    assert sum(len(out[r][0]) for r in range(world)) == len(union)


def _id_worker(rank, world, port, out):
    import torch.distributed as dist

    from paper_2311_02206_b200.partition import share_unique_id

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    raw = bytes(range(128)) if rank == 0 else bytes(128)
    out[rank] = share_unique_id(raw)
    dist.destroy_process_group()


def test_share_unique_id_gloo():
    """The native driver's communicator setup: rank 0's NCCL id reaches
    every rank through torch.distributed (here gloo, 2 ranks on CPU)."""
    world = 2
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_id_worker, args=(world, free_port(), out), nprocs=world, join=True)
        assert out[0] == out[1] == bytes(range(128))
