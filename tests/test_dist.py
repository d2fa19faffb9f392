"""Multi-process (gloo, world_size 2 and 3) check of the data-parallel CTC
step's host logic: LPT shards cover the global minibatch exactly once, an
empty shard still joins the collective, and the rank-ordered scalar reduce
of {loss, skipped} equals the single-process trainer sums
(trainer.cpp:160-180). Per-utterance costs come from the oracle (the
checker) -- the GPU path is exercised by bench.py / -m gpu tests."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_1512_02595_b200 import dist as ddist
from paper_1512_02595_b200.synth import make_batch


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, result_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        T = [30, 12, 25, 8, 20, 2, 16, 10][:n]
        L = [8, 3, 7, 2, 5, 4, 4, 3][:n]  # utterance 5 (T=2, L=4) is infeasible
        acts, flat, ll, il = make_batch(6, T, L, seed=21)
        offs = np.concatenate([[0], np.cumsum(ll)])

        def compute(idx):
            costs = []
            for b in idx:
                x = acts[:il[b], b, :].astype(np.float64)
                ok, loss, _ = oracle.oracle_loss(x, flat[offs[b]:offs[b + 1]], 5, want_grad=False)
                costs.append(loss if ok else np.inf)
            return np.asarray(costs)

        g_loss, g_skipped, idx = ddist.dp_ctc_step(il, ll, 6, rank, world, compute)
        result_q.put((rank, g_loss, g_skipped, sorted(int(i) for i in idx)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 8), (3, 2)])
def test_dp_step_matches_single_process(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    T = [30, 12, 25, 8, 20, 2, 16, 10][:n]
    L = [8, 3, 7, 2, 5, 4, 4, 3][:n]
    acts, flat, ll, il = make_batch(6, T, L, seed=21)
    costs, _ = oracle.oracle_batch(acts, flat, ll, il, want_grad=False)
    want_loss, want_skipped = ddist.local_loss_skipped(costs)
    covered = []
    for rank, g_loss, g_skipped, idx in results:
        assert g_skipped == want_skipped
        assert abs(g_loss - want_loss) <= 1e-9 * max(1.0, abs(want_loss))
        covered += idx
    assert sorted(covered) == list(range(n))
    # every rank saw the bitwise-identical reduced value (rank-order fold)
    assert len({r[1] for r in results}) == 1


def _peer_worker(rank, world, port, result_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # No GPU here: the mailbox allocation fails on every rank, every setup
        # collective still runs (no deadlock) and the group agrees to fall back.
        red = ddist.PeerLossReducer("cpu")
        result_q.put((rank, red.ok, red.error is not None))
    finally:
        dist.destroy_process_group()


def test_peer_reducer_setup_agrees_on_fallback_without_gpu():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(not ok and had_error for _, ok, had_error in results)
