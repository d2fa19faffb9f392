"""H1 host scheduler: SortaGrad order identical to the reference
(trainer.cpp:58-91), the reference's contiguous rank slice
(trainer.cpp:140-143), and the LPT re-deal used on B200."""
import numpy as np
import pytest

import oracle
from paper_1512_02595_b200 import scheduler
from paper_1512_02595_b200.synth import Rng, sortagrad_lengths


def test_sortagrad_matches_reference_golden(golden):
    lens = golden["sortagrad/lengths"]
    for epoch in range(4):
        for on in (0, 1):
            got = scheduler.sortagrad_order(lens, 16, epoch, 1234, bool(on))
            assert np.array_equal(got, golden[f"sortagrad/order_e{epoch}_s{on}"]), (epoch, on)


@pytest.mark.skipif(not oracle.ref_available(), reason="reference build not present")
def test_sortagrad_matches_live_reference():
    rng = Rng(3)
    for trial in range(20):
        n = 1 + int(rng.below(1, 200)[0])
        lens = (1 + rng.below(n, 50)).astype(np.int32)
        gb = 1 + int(rng.below(1, 32)[0])
        for epoch in range(3):
            for on in (False, True):
                assert np.array_equal(scheduler.sortagrad_order(lens, gb, epoch, 77 + trial, on),
                                      oracle.ref_sortagrad(lens, gb, epoch, 77 + trial, on))


def test_sortagrad_properties():
    # test_trainer.cpp:63-105: epoch-0 sort, stable ties, deterministic shuffles, permutation
    lens = np.array([5, 3, 3, 9, 1, 3, 7, 7], dtype=np.int32)
    o0 = scheduler.sortagrad_order(lens, 3, 0, 1)
    assert list(o0) == [4, 1, 2, 5, 0, 6, 7, 3]
    o1 = scheduler.sortagrad_order(lens, 3, 1, 1)
    assert sorted(o1) == list(range(8))
    assert np.array_equal(o1, scheduler.sortagrad_order(lens, 3, 1, 1))
    # later epochs visit whole epoch-0 minibatches (including the partial one) in a shuffled order
    batches = [tuple(o0[i:i + 3]) for i in range(0, 8, 3)]
    pos, seen = 0, []
    while pos < 8:
        match = [bt for bt in batches if tuple(o1[pos:pos + len(bt)]) == bt]
        assert len(match) == 1
        seen.append(match[0])
        pos += len(match[0])
    assert sorted(seen) == sorted(batches)


def test_rank_slice_matches_reference_formula():
    for batch_n in (0, 1, 7, 16, 17):
        for mb in (1, 4, 8):
            for rank in range(4):
                b, e = scheduler.rank_slice(batch_n, mb, rank)
                assert b == min(batch_n, rank * mb) and e == min(batch_n, (rank + 1) * mb)


def test_lpt_balances_sortagrad_batch():
    T, L = sortagrad_lengths(512, seed=7)
    order = np.argsort(T, kind="stable")
    T, L = T[order], L[order]
    for world in (2, 4, 8):
        ranks, load = scheduler.shard_lpt(T, L, 29, world)
        assert sorted(set(ranks.tolist())) == list(range(world))
        cost = T.astype(np.float64) * (1 + 29 / 1024)
        for r in range(world):
            assert abs(load[r] - cost[ranks == r].sum()) < 1e-6 * cost.sum()
        assert load.max() / load.mean() < 1.01
        # longest utterances spread across ranks (no straggler rank)
        top = np.argsort(-T, kind="stable")[:world]
        assert len(set(ranks[top].tolist())) == world
        # the reference's contiguous slices are badly imbalanced on a sorted batch
        mb = 512 // world
        contiguous = [cost[r * mb:(r + 1) * mb].sum() for r in range(world)]
        assert max(contiguous) / np.mean(contiguous) > load.max() / load.mean()


def test_shard_batch_partitions():
    T, L = sortagrad_lengths(100, seed=1)
    seen = []
    for r in range(4):
        idx = scheduler.shard_batch(T, L, 29, 4, r)
        assert np.all(np.diff(T[idx]) <= 0)  # longest first within a rank
        seen.extend(idx.tolist())
    assert sorted(seen) == list(range(100))
    # world larger than the batch: some ranks are empty but valid
    ranks, _ = scheduler.shard_lpt([10, 20], [2, 3], 29, 8)
    assert set(ranks.tolist()) <= set(range(8))
