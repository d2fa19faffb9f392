"""Data-parallel CTC step over torch.distributed (NCCL on B200, gloo in CPU tests).

The reference's only cross-worker interaction on the CTC path is the ring
all-reduce of the two scalars {local_loss, local_skipped}
(proj/src/trainer.cpp:174-180, allreduce.cpp:301-341). Here each rank
computes its shard of the global minibatch (H1: SortaGrad composition, LPT
deal) and the scalars cross NVLink in ONE tiny collective. For run-to-run
determinism like the reference ring's fixed fold order (allreduce.hpp:91-95),
the per-rank pairs are all-gathered and folded in rank order on every rank.
Empty shards still join the collective (trainer.cpp:141-155,173-180).
"""
from __future__ import annotations

import ctypes
from typing import Callable, Tuple

import numpy as np

from . import scheduler


def reduce_loss_skipped(local_loss: float, local_skipped: int, device=None) -> Tuple[float, int]:
    """Rank-order-deterministic sum of {loss, skipped} over the default process group."""
    import torch
    import torch.distributed as dist

    pair = torch.tensor([float(local_loss), float(local_skipped)], dtype=torch.float64, device=device)
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(pair[0]), int(pair[1])
    world = dist.get_world_size()
    out = torch.empty(world * 2, dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(out, pair)
    vals = out.view(world, 2).cpu().numpy()
    loss = 0.0
    skipped = 0.0
    for r in range(world):  # fixed rank order, like the ring's fold (allreduce.cpp:326)
        loss = loss + vals[r, 0]
        skipped = skipped + vals[r, 1]
    return float(loss), int(skipped)


def local_loss_skipped(costs: np.ndarray) -> Tuple[float, int]:
    """trainer.cpp:160-168: infeasible utterances (cost +inf) are skipped, the rest summed
    in order -- a NaN cost (diverged logits) is feasible in the reference and makes the sum NaN."""
    loss = 0.0
    skipped = 0
    for c in np.asarray(costs, dtype=np.float64):
        if np.isposinf(c):
            skipped += 1
        else:
            loss += float(c)
    return loss, skipped


def dp_ctc_step(batch_input_lengths, batch_label_lengths, alphabet_size: int, rank: int, world: int,
                compute: Callable[[np.ndarray], np.ndarray], device=None):
    """One data-parallel CTC step for a global minibatch.

    compute(indices) must return this rank's per-utterance costs for the
    given minibatch indices (the GPU path in bench.py; any function in tests).
    Returns (global loss sum, global skipped count, this rank's indices).
    """
    idx = scheduler.shard_batch(batch_input_lengths, batch_label_lengths, alphabet_size, world, rank)
    costs = compute(idx) if idx.size else np.zeros(0)
    loss, skipped = local_loss_skipped(costs)
    g_loss, g_skipped = reduce_loss_skipped(loss, skipped, device=device)
    return g_loss, g_skipped, idx


class PeerLossReducer:
    """The trainer's {loss, skipped} sums fused with their all-reduce over
    NVLink peer memory (ds2ctc_loss_sum_allreduce): one single-warp kernel per
    rank per step, rank-ordered fold, no NCCL call on the step. Setup exchanges
    CUDA IPC handles of the per-rank mailboxes over the default process group
    once; every collective of the setup runs on every rank even if a local
    step failed, and `ok` is the group's agreement (all ranks succeeded)."""

    def __init__(self, device):
        import torch
        import torch.distributed as dist

        from . import _lib

        self.lib = _lib.lib()
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.opened = []
        self.own = None
        self.seq = 0
        err = None
        own = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        if self.world > 8:
            err = "more than 8 ranks"
        elif self.lib.ds2ctc_mailbox_alloc(self.world, ctypes.byref(own), handle) != 0:
            err = "mailbox alloc / IPC handle failed"
        else:
            self.own = own.value
        handles = [None] * self.world
        dist.all_gather_object(handles, None if err else bytes(handle))
        self.ptrs = (ctypes.c_void_p * max(self.world, 1))()
        if err is None:
            for r in range(self.world):
                if r == self.rank:
                    self.ptrs[r] = self.own
                    continue
                if handles[r] is None:
                    err = f"rank {r} has no mailbox"
                    break
                p = ctypes.c_void_p()
                h = (ctypes.c_char * 64).from_buffer_copy(handles[r])
                if self.lib.ds2ctc_mailbox_open(h, ctypes.byref(p)) != 0:
                    err = f"IPC open of rank {r}'s mailbox failed"
                    break
                self.ptrs[r] = p.value
                self.opened.append(p.value)
        flag = torch.tensor([0 if err else 1], dtype=torch.int32, device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        self.ok = bool(flag.item())
        self.error = err
        if not self.ok:
            self.close()

    def reduce(self, costs_ptr: int, B: int, out2_ptr: int, stream_ptr: int) -> None:
        from . import _lib

        if self.own is None:
            raise RuntimeError("PeerLossReducer is closed (a peer was lost); rebuild it on every rank")
        self.seq += 1
        _lib.check(self.lib.ds2ctc_loss_sum_allreduce(ctypes.c_void_p(costs_ptr), B, ctypes.c_void_p(out2_ptr),
                                                      ctypes.cast(self.ptrs, ctypes.POINTER(ctypes.c_void_p)),
                                                      self.rank, self.world, self.seq,
                                                      ctypes.c_void_p(stream_ptr)),
                   "ds2ctc_loss_sum_allreduce")

    def check(self) -> None:
        """Raises (and closes the mailboxes) if a step's peer wait timed out. The
        kernel wrote NaN for that step instead of a stale fold; after a timeout
        the one-step-ahead invariant is gone, so the reducer must be rebuilt."""
        from . import _lib

        seq = _lib.reduce_fault()
        if seq is not None:
            self.close()
            raise RuntimeError(f"fused loss all-reduce: peer wait timed out at step {seq}")

    def close(self) -> None:
        for p in self.opened:
            self.lib.ds2ctc_mailbox_close(ctypes.c_void_p(p), 0)
        if self.own is not None:
            self.lib.ds2ctc_mailbox_close(ctypes.c_void_p(self.own), 1)
        self.opened = []
        self.own = None


class PeerVecReducer:
    """The parameter-gradient all-reduce of trainer.cpp:175 (ring_allreduce,
    allreduce.cpp:301-341) over NVLink peer memory (ds2ctc_vec_allreduce): one
    kernel per call, rank-ordered fold (bitwise identical on every rank), no
    NCCL call on the step. One exchange region per rank for vectors of `n`
    floats; setup exchanges CUDA IPC handles once over the default process
    group, and `ok` is the group's agreement (all ranks succeeded)."""

    def __init__(self, n: int, device):
        import torch
        import torch.distributed as dist

        from . import _lib

        self.lib = _lib.lib()
        self.n = int(n)
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.opened = []
        self.own = None
        self.seq = 0
        err = None
        own = ctypes.c_void_p()
        handle = (ctypes.c_char * 64)()
        size = ctypes.c_size_t()
        if self.world > 8:
            err = "more than 8 ranks"
        elif self.lib.ds2ctc_exchange_size(self.n, ctypes.byref(size)) != 0 or \
                self.lib.ds2ctc_exchange_alloc(size.value, ctypes.byref(own), handle) != 0:
            err = "exchange alloc / IPC handle failed"
        else:
            self.own = own.value
        handles = [None] * self.world
        dist.all_gather_object(handles, None if err else bytes(handle))
        self.ptrs = (ctypes.c_void_p * max(self.world, 1))()
        if err is None:
            for r in range(self.world):
                if r == self.rank:
                    self.ptrs[r] = self.own
                    continue
                if handles[r] is None:
                    err = f"rank {r} has no exchange region"
                    break
                p = ctypes.c_void_p()
                h = (ctypes.c_char * 64).from_buffer_copy(handles[r])
                if self.lib.ds2ctc_mailbox_open(h, ctypes.byref(p)) != 0:
                    err = f"IPC open of rank {r}'s exchange region failed"
                    break
                self.ptrs[r] = p.value
                self.opened.append(p.value)
        flag = torch.tensor([0 if err else 1], dtype=torch.int32, device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        self.ok = bool(flag.item())
        self.error = err
        if not self.ok:
            self.close()

    def reduce(self, data_ptr: int, stream_ptr: int) -> None:
        """In place: data[n] (fp32, device) <- sum over ranks in rank order."""
        from . import _lib

        if self.own is None:
            raise RuntimeError("PeerVecReducer is closed (a peer was lost); rebuild it on every rank")
        self.seq += 1
        _lib.check(self.lib.ds2ctc_vec_allreduce(ctypes.c_void_p(data_ptr), self.n,
                                                 ctypes.cast(self.ptrs, ctypes.POINTER(ctypes.c_void_p)),
                                                 self.rank, self.world, self.seq, ctypes.c_void_p(stream_ptr)),
                   "ds2ctc_vec_allreduce")

    def check(self) -> None:
        """Raises (and closes) if a peer wait of any peer-memory collective timed out."""
        from . import _lib

        seq = _lib.reduce_fault()
        if seq is not None:
            self.close()
            raise RuntimeError(f"peer-memory all-reduce: peer wait timed out at step {seq}")

    def close(self) -> None:
        for p in self.opened:
            self.lib.ds2ctc_mailbox_close(ctypes.c_void_p(p), 0)
        self.opened = []
        if self.own is not None:
            self.lib.ds2ctc_mailbox_close(ctypes.c_void_p(self.own), 1)
            self.own = None
