"""Hash-partitioned multi-GPU fixpoint (component N1).

One process per GPU.  Every rank holds the EDB replicated and the IDB
tuples it owns (owner = hash(tuple) mod nranks, engine.cu keep_owned).  Per
iteration each rank:
  1. runs the recursive joins on its local Δ, sorts + dedups the derived
     rows and groups them by owner rank      (gd_engine_partition_begin);
  2. exchanges the groups with an all-to-all-v (NCCL over NVLink through
     torch.distributed: counts first, then the rows);
  3. merges what it received into its local full relation, producing its
     local Δ                                  (gd_engine_partition_end);
  4. sends its |Δ| with the next iteration's counts — the fixpoint is
     reached when the global sum is 0 (no separate all-reduce).

The exchange is abstracted (`Exchange`) so the same loop runs over NCCL,
over gloo (CPU tests) or over an in-process loopback of P logical shards on
one GPU (parity tests).
"""
from __future__ import annotations

import numpy as np


class CudaBuffer:
    """__cuda_array_interface__ view of a device pointer (zero-copy into
    torch.as_tensor)."""

    def __init__(self, ptr: int, nwords: int):
        self.__cuda_array_interface__ = {
            "shape": (nwords,), "typestr": "<u8", "data": (ptr, False), "version": 3, "strides": None}


class TorchExchange:
    """All-to-all-v through torch.distributed (NCCL on GPUs).  The
    collectives run on torch's current stream, which must be the engine
    context's stream (bench.py builds the Context on it): the engine's
    next kernels then read the received rows in stream order."""

    def __init__(self, device: str = "cuda"):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.device = torch, dist, device
        self.rank = dist.get_rank()
        self.size = dist.get_world_size()
        self._recv = None

    def _wrap(self, ptr: int, nwords: int):
        torch = self.torch
        if self.device == "cpu":  # host pointer (gloo tests)
            import ctypes

            arr = np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctypes.c_int64)), shape=(nwords,))
            return torch.from_numpy(arr)
        return torch.as_tensor(CudaBuffer(ptr, nwords), device=self.device).view(torch.int64)

    def exchange(self, send_counts: np.ndarray, send_ptr: int, words: int, delta: int = 1):
        """All-to-all-v of the owner groups.  Each rank's |Δ| rides along
        with its counts (one all-to-all instead of counts + an all-reduce);
        returns (recv_ptr, recv_rows, global |Δ|).  When the global |Δ| is 0
        every rank sent nothing and the row exchange is skipped."""
        torch, dist = self.torch, self.dist
        P = len(send_counts)
        meta = np.stack([send_counts.astype(np.int64), np.full(P, int(delta), dtype=np.int64)], 1).reshape(-1)
        cnt = torch.as_tensor(meta, device=self.device)
        rcnt = torch.empty_like(cnt)
        dist.all_to_all_single(rcnt, cnt)
        rm = rcnt.cpu().numpy().reshape(P, 2)
        rc, gdelta = rm[:, 0], int(rm[:, 1].sum())
        if gdelta == 0:
            return 0, 0, 0
        total_send = int(send_counts.sum())
        total_recv = int(rc.sum())
        if total_send:
            send = self._wrap(send_ptr, total_send * words)
        else:
            send = torch.empty(0, dtype=torch.int64, device=self.device)
        if self._recv is None or self._recv.numel() < max(total_recv * words, 1):
            self._recv = torch.empty(max(total_recv * words, 1) * 5 // 4 + 1024, dtype=torch.int64,
                                     device=self.device)
        recv = self._recv[: total_recv * words]
        dist.all_to_all_single(recv, send, [int(x) * words for x in rc], [int(x) * words for x in send_counts])
        return (recv.data_ptr() if total_recv else 0), total_recv, gdelta


def run_partitioned(eng, exchange, nranks: int, max_iters: int = 1 << 30) -> int:
    """Drives one rank's engine to the global fixpoint; returns iterations.
    `eng` must be seeded with set_partition(rank, nranks) applied.  The
    termination test uses the |Δ| each rank sends with its counts, so an
    iteration costs one counts all-to-all and one rows all-to-all; after the
    last productive iteration one more (empty) begin + counts exchange sees
    the global |Δ| = 0."""
    import os
    import time

    trace = os.environ.get("GD_PART_TRACE") == "1"
    tb = tx = te = 0.0
    words = eng.exchange_words()
    it = 0
    local = 1  # the seeded Δ: the first iteration always runs (engine.hpp:181-257)
    while it < max_iters:
        t0 = time.perf_counter()
        counts, ptr = eng.partition_begin(nranks)
        t1 = time.perf_counter()
        rptr, rrows, gdelta = exchange.exchange(counts, ptr, words, local)
        t2 = time.perf_counter()
        tb, tx = tb + t1 - t0, tx + t2 - t1
        if gdelta == 0:
            break
        local = eng.partition_end(rptr, rrows)
        te += time.perf_counter() - t2
        it += 1
    if trace:
        print(f"[partition] {it} iterations: begin {tb * 1e3:.1f} ms, exchange {tx * 1e3:.1f} ms, "
              f"end {te * 1e3:.1f} ms", flush=True)
    return it


def share_unique_id(raw: bytes) -> bytes:
    """Rank 0's 128-byte NCCL unique id to every rank of the default
    torch.distributed group (the other ranks pass any 128 bytes)."""
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(list(raw), dtype=torch.uint8, device=dev)
    dist.broadcast(t, 0)
    return bytes(t.cpu().tolist())


class NcclComm:
    """The native driver's NCCL communicator (gd_nccl_comm_create): rank 0's
    unique id is broadcast through the default torch.distributed group."""

    def __init__(self, ctx, rank: int, nranks: int):
        import ctypes as C

        import torch  # noqa: F401  (loads torch's NCCL before the library resolves it)

        self.ctx = ctx
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            ctx.check(ctx.lib.gd_nccl_unique_id(uid))
        if nranks > 1:
            uid = (C.c_uint8 * 128)(*share_unique_id(bytes(uid)))
        h = C.c_void_p()
        ctx.check(ctx.lib.gd_nccl_comm_create(ctx.h, uid, nranks, rank, C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            self.ctx.lib.gd_nccl_comm_destroy(self.h)
            self.h = None


class LoopbackComms:
    """Test transport of the native driver: `nranks` communicators whose
    ranks run as threads of this process on one GPU (gd_loopback_*)."""

    def __init__(self, ctx, nranks: int):
        import ctypes as C

        self.ctx = ctx
        hub = C.c_void_p()
        ctx.check(ctx.lib.gd_loopback_hub_create(nranks, C.byref(hub)))
        self.hub = hub
        self.comms = []
        for r in range(nranks):
            h = C.c_void_p()
            ctx.check(ctx.lib.gd_loopback_comm_create(hub, r, C.byref(h)))
            c = NcclComm.__new__(NcclComm)
            c.ctx, c.h = ctx, h
            self.comms.append(c)

    def close(self):
        for c in self.comms:
            c.close()
        if self.hub:
            self.ctx.lib.gd_loopback_hub_destroy(self.hub)
            self.hub = None


def run_partitioned_native(eng, comm: NcclComm, max_iters: int = 0) -> int:
    """The partitioned fixpoint with the library's own NCCL exchanges (one
    host synchronisation per iteration); same result as run_partitioned."""
    return eng.run_partitioned(comm, max_iters)


class LoopbackCluster:
    """P logical shards in one process (one GPU): the all-to-all is a
    device-to-device gather of every shard's send groups.  Used by the
    parity tests of the partitioned path on a single B200."""

    def __init__(self, engines):
        import torch

        self.torch = torch
        self.engines = engines
        self.P = len(engines)

    def run(self, max_iters: int = 1 << 30) -> int:
        torch = self.torch
        P = self.P
        words = self.engines[0].exchange_words()
        it = 0
        while it < max_iters:
            sends = [e.partition_begin(P) for e in self.engines]  # (counts, ptr)
            views = []
            for counts, ptr in sends:
                tot = int(counts.sum())
                if tot:
                    t = torch.as_tensor(CudaBuffer(ptr, tot * words), device="cuda").view(torch.int64).clone()
                else:
                    t = torch.empty(0, dtype=torch.int64, device="cuda")
                offs = np.concatenate([[0], np.cumsum(counts.astype(np.int64))]) * words
                views.append((t, offs))
            total = 0
            for dst, e in enumerate(self.engines):
                parts = [t[offs[dst]: offs[dst + 1]] for t, offs in views]
                recv = torch.cat(parts) if parts else torch.empty(0, dtype=torch.int64, device="cuda")
                torch.cuda.synchronize()  # the engine reads recv on its own stream
                n = recv.numel() // words
                total += e.partition_end(recv.data_ptr() if n else 0, n)
                del recv
            it += 1
            if total == 0:
                break
        return it
