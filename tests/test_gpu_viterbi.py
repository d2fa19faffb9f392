"""GPU forced alignment (ds2ctc_viterbi_align) vs the reference's
viterbi_align (proj/src/ctc.cpp:327-370): the oracle restatement (pinned
bitwise to the reference build in test_oracle.py) and, where present, the
reference build itself. Alignments are index sequences: the bar is exact
equality, including the tie rule (stay > advance > skip, terminal blank)."""
import math

import numpy as np
import pytest

import oracle
from paper_1512_02595_b200 import ctc as dctc
from paper_1512_02595_b200.synth import Rng, fixed_shape_batch, make_batch

pytestmark = pytest.mark.gpu


def gpu_align(acts, flat, ll, il, blank=None):
    import torch

    x = torch.from_numpy(np.ascontiguousarray(acts, dtype=np.float32)).cuda()
    align, status = dctc.viterbi_align_batch(x, flat, ll, il, blank=blank)
    torch.cuda.synchronize()
    return align.cpu().numpy(), status.cpu().numpy()


def check_batch(acts, flat, ll, il, blank):
    align, status = gpu_align(acts, flat, ll, il, blank)
    offs = np.concatenate([[0], np.cumsum(ll)]).astype(np.int64)
    n_aligned = 0
    for b in range(len(il)):
        T = int(il[b])
        label = [int(c) for c in flat[offs[b]:offs[b + 1]]]
        ref = oracle.oracle_viterbi(acts[:T, b, :].astype(np.float64), label, blank)
        if ref is None:
            assert status[b] == 1, f"utterance {b}: reference has no alignment, GPU status {status[b]}"
            assert np.all(align[b] == -1)
        else:
            assert status[b] == 0, f"utterance {b}: GPU found no alignment"
            assert np.array_equal(align[b, :T], ref), f"utterance {b}: alignment differs"
            assert np.all(align[b, T:] == -1)
            n_aligned += 1
            if oracle.ref_available():
                assert np.array_equal(oracle.ref_viterbi(acts[:T, b, :].astype(np.float64), label, blank), ref)
    return n_aligned


def test_known_answers(cuda):
    # test_ctc.cpp:233-240 (forced alignment) and :257-266 (tie rule)
    lp = np.full((3, 4), math.log(0.02), dtype=np.float32)
    label = [2, 0, 1]
    for t in range(3):
        lp[t, label[t]] = math.log(0.94)
    assert dctc.viterbi_align(lp, label, 3) == label
    assert dctc.viterbi_align(np.full((2, 2), math.log(0.5), dtype=np.float32), [0], 1) == [0, 1]
    with pytest.raises(ValueError):
        dctc.viterbi_align(np.zeros((2, 3), dtype=np.float32), [0, 0], 2)  # T < min_frames = 3


def test_random_small_with_repeats_and_infeasible(cuda):
    rng = Rng(777)
    T = [int(v) for v in rng.below(48, 40) + 1]
    L = [int(v) for v in rng.below(48, 12)]
    for i in range(0, 48, 7):
        L[i] = 0  # empty labels
    for i in range(3, 48, 11):
        T[i] = max(1, L[i] - 2)  # infeasible lengths
    acts, flat, ll, il = make_batch(6, T, L, seed=31)
    flat = flat.copy()
    flat[::3] = flat[::3] % 2  # many repeats -> blank-separated runs
    assert check_batch(acts, flat, ll, il, 5) > 20


def test_uniform_logits_tie_rule(cuda):
    # every path ties: the reference's rule alone decides
    T, A = 9, 4
    acts = np.zeros((T, 3, A), dtype=np.float32)
    flat = np.array([0, 1, 0, 2, 2, 1], dtype=np.int32)
    ll = np.array([2, 3, 1], dtype=np.int32)
    il = np.array([T, T, 5], dtype=np.int32)
    assert check_batch(acts, flat, ll, il, A - 1) == 3


def test_english_shape_and_peaked(cuda):
    acts, flat, ll, il = fixed_shape_batch(29, 700, 150, 16, seed=12)
    assert check_batch(acts, flat, ll, il, 28) == 16
    acts8 = (acts * 8.0).astype(np.float32)
    assert check_batch(acts8, flat, ll, il, 28) == 16


def test_large_alphabet(cuda):
    acts, flat, ll, il = fixed_shape_batch(300, 120, 40, 4, seed=5)
    assert check_batch(acts, flat, ll, il, 299) == 4
