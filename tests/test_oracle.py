"""The oracle restatement (oracle/ctc_oracle.c) pinned against the reference.

* against the golden fixtures produced by the reference's own fp64 build
  (tests/golden/make_golden.py) -- works anywhere;
* bit-for-bit against the live reference build (oracle/_ref) when present;
* against the reference's known-answer tests (proj/tests/test_ctc.cpp) and
  its brute-force / finite-difference oracles (proj/tests/oracles.hpp);
* the reference's own test_ctc.cpp, compiled unchanged (oracle/_ref/test_ctc).
"""
import itertools
import math
import os
import subprocess

import numpy as np
import pytest

import oracle
from conftest import golden_cases
from paper_1512_02595_b200.synth import Rng

need_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference build (oracle/_ref) not present")


def test_oracle_matches_golden(golden):
    for name in golden_cases(golden):
        costs, grads = oracle.oracle_batch(golden[f"{name}/acts"], golden[f"{name}/labels"],
                                           golden[f"{name}/label_lengths"], golden[f"{name}/input_lengths"],
                                           blank=int(golden[f"{name}/blank"]))
        ref_c = golden[f"{name}/costs"]
        assert np.array_equal(np.isfinite(costs), np.isfinite(ref_c)), name
        fin = np.isfinite(ref_c)
        assert np.array_equal(costs[fin], ref_c[fin]), f"{name}: cost not bit-identical to the reference"
        assert np.array_equal(grads.astype(np.float32), golden[f"{name}/grads"]), f"{name}: grads differ"


@need_ref
def test_oracle_bitwise_vs_live_reference():
    rng = Rng(123)
    for it in range(60):
        A = 2 + int(rng.below(1, 30)[0])
        T = int(rng.below(1, 40)[0])
        L = int(rng.below(1, 12)[0])
        label = [int(c) for c in rng.below(L, A)] if L else []  # may include the blank id
        logits = rng.normal(T * A).reshape(T, A) * (1 + 4 * (it % 3))
        if T == 0:
            continue
        f1, l1, g1 = oracle.oracle_loss(logits, label, A - 1)
        f2, l2, g2 = oracle.ref_loss(logits, label, A - 1)
        assert f1 == f2
        if f1:
            assert l1 == l2
            assert np.array_equal(g1, g2)
        a1, b1, p1 = oracle.oracle_lattice(logits, label, A - 1)
        a2, b2, p2 = oracle.ref_lattice(logits, label, A - 1)
        assert np.array_equal(a1, a2) and np.array_equal(b1, b2) and (p1 == p2 or (math.isnan(p1) and math.isnan(p2)))


def test_known_answers():
    half = math.log(0.5)
    ok, loss, _ = oracle.oracle_loss(np.full((1, 2), half), [0], 1)  # test_ctc.cpp:71-79
    assert ok and abs(loss - (-math.log(0.5))) < 1e-12
    ok, loss, _ = oracle.oracle_loss(np.full((2, 2), half), [0], 1)  # test_ctc.cpp:81-93
    assert ok and abs(math.exp(-loss) - 0.75) < 1e-12
    ok, loss, g = oracle.oracle_loss(np.full((2, 2), half), [0, 0], 1)  # test_ctc.cpp:95-105
    assert not ok and math.isinf(loss)
    assert oracle.oracle_min_frames([0, 0]) == 3
    assert oracle.oracle_loss(np.full((3, 2), half), [0, 0], 1)[0]
    ok, loss, _ = oracle.oracle_loss(np.full((4, 3), math.log(1 / 3)), [], 2)  # test_ctc.cpp:268-275
    assert ok and abs(loss - 4 * math.log(3)) < 1e-12
    lse = oracle.oracle_lib().orc_log_sum_exp_guarded  # test_ctc.cpp:60-69
    assert lse(-math.inf, -1.5) == -1.5 and lse(-1.5, -math.inf) == -1.5
    assert lse(-math.inf, -math.inf) == -math.inf
    assert abs(lse(-3.0, -3.0) - (-3.0 + math.log(2))) < 1e-14


def _collapse(path, blank):  # oracles.hpp:35-42
    out = []
    for t, c in enumerate(path):
        if t > 0 and c == path[t - 1]:
            continue
        if c != blank:
            out.append(c)
    return out


def _brute(probs, label, blank):  # oracles.hpp:46-63
    T, C = probs.shape
    total = 0.0
    for path in itertools.product(range(C), repeat=T):
        if _collapse(path, blank) == list(label):
            total += float(np.prod([probs[t, path[t]] for t in range(T)]))
    return total


def test_brute_force_path_sum():
    # acceptance_main.cpp:90-109 (criterion 1) style, smaller count
    rng = Rng(101)
    done = 0
    while done < 60:
        alphabet = 1 + int(rng.below(1, 3)[0])
        frames = 1 + int(rng.below(1, 5)[0])
        L = int(rng.below(1, 4)[0])
        label = [int(c) for c in rng.below(L, alphabet)] if L else []
        u = 0.05 + rng.uniform(frames * (alphabet + 1)).reshape(frames, alphabet + 1)
        lp = np.log(u / u.sum(axis=1, keepdims=True))
        brute = _brute(np.exp(lp), label, alphabet)
        ok, loss, _ = oracle.oracle_loss(lp, label, alphabet)
        if frames < oracle.oracle_min_frames(label):
            assert not ok and brute < 1e-15
            continue
        done += 1
        assert ok and abs(math.exp(-loss) - brute) <= 1e-9


def test_finite_difference_gradient():
    # test_ctc.cpp:126-147 / oracles.hpp:124-138
    rng = Rng(7)
    for _ in range(10):
        alphabet = 1 + int(rng.below(1, 3)[0])
        frames = 2 + int(rng.below(1, 4)[0])
        L = int(rng.below(1, 3)[0])
        label = [int(c) for c in rng.below(L, alphabet)] if L else []
        while label and frames < oracle.oracle_min_frames(label):
            label.pop()
        x = rng.uniform(frames * (alphabet + 1)).reshape(frames, alphabet + 1) * 2 - 1
        ok, loss, g = oracle.oracle_loss(x, label, alphabet)
        assert ok
        h = 1e-6
        for t in range(frames):
            for k in range(alphabet + 1):
                xp = x.copy()
                xp[t, k] += h
                xm = x.copy()
                xm[t, k] -= h
                fd = (oracle.oracle_loss(xp, label, alphabet, False)[1] -
                      oracle.oracle_loss(xm, label, alphabet, False)[1]) / (2 * h)
                assert abs(g[t, k] - fd) / max(1.0, abs(fd)) < 1e-6


def test_lattice_cancellation():
    # test_ctc.cpp:172-199: invalid cells are -inf after alpha+beta, valid cells finite
    rng = Rng(31337)
    for _ in range(30):
        alphabet = 1 + int(rng.below(1, 3)[0])
        frames = 1 + int(rng.below(1, 6)[0])
        L = int(rng.below(1, 4)[0])
        label = [int(c) for c in rng.below(L, alphabet)] if L else []
        if frames < oracle.oracle_min_frames(label):
            continue
        x = rng.normal(frames * (alphabet + 1)).reshape(frames, alphabet + 1)
        alpha, beta, _ = oracle.oracle_lattice(x, label, alphabet)
        aug = [alphabet]
        for c in label:
            aug += [c, alphabet]
        S = len(aug)
        skip = [s >= 2 and aug[s] != alphabet and aug[s] != aug[s - 2] for s in range(S)]
        fwd = np.zeros((S, frames), bool)
        bwd = np.zeros((S, frames), bool)
        fwd[0, 0] = True
        if S > 1:
            fwd[1, 0] = True
        for t in range(1, frames):
            for s in range(S):
                fwd[s, t] = fwd[s, t - 1] or (s >= 1 and fwd[s - 1, t - 1]) or (skip[s] and fwd[s - 2, t - 1])
        bwd[S - 1, frames - 1] = True
        if S > 1:
            bwd[S - 2, frames - 1] = True
        for t in range(frames - 2, -1, -1):
            for s in range(S):
                bwd[s, t] = bwd[s, t + 1] or (s + 1 < S and bwd[s + 1, t + 1]) or (
                    s + 2 < S and skip[s + 2] and bwd[s + 2, t + 1])
        comb = alpha + beta
        valid = fwd & bwd
        assert np.all(np.isneginf(comb[~valid]))
        assert np.all(np.isfinite(comb[valid]))


def test_viterbi_matches_reference_semantics():
    # test_ctc.cpp:233-240 forced alignment and :257-266 tie rule
    lp = np.full((3, 4), math.log(0.02))
    label = [2, 0, 1]
    for t in range(3):
        lp[t, label[t]] = math.log(0.94)
    assert list(oracle.oracle_viterbi(lp, label, 3)) == label
    assert list(oracle.oracle_viterbi(np.full((2, 2), math.log(0.5)), [0], 1)) == [0, 1]


@need_ref
def test_viterbi_bitwise_vs_reference():
    rng = Rng(4242)
    for _ in range(40):
        A = 2 + int(rng.below(1, 6)[0])
        T = 1 + int(rng.below(1, 20)[0])
        L = int(rng.below(1, 6)[0])
        label = [int(c) for c in rng.below(L, A - 1)] if L else []
        x = rng.normal(T * A).reshape(T, A)
        a = oracle.oracle_viterbi(x, label, A - 1)
        b = oracle.ref_viterbi(x, label, A - 1)
        assert (a is None and b is None) or np.array_equal(a, b)


@need_ref
def test_reference_parallel_equals_reference():
    # ctc_loss_parallel is bitwise equal to the sequential one (test_ctc.cpp:149-170)
    rng = Rng(99)
    for _ in range(10):
        x = rng.normal(12 * 5).reshape(12, 5)
        label = [int(c) for c in rng.below(3, 4)]
        a = oracle.ref_loss(x, label, 4)
        b = oracle.ref_loss_parallel(x, label, 4, 3)
        assert a[0] == b[0] and a[1] == b[1] and np.array_equal(a[2], b[2])


def test_reference_unit_tests_pass_unchanged():
    exe = os.path.join(oracle.HERE, "_ref", "test_ctc")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/test_ctc not built")
    res = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "15 passed | 0 failed" in res.stdout


def test_sortagrad_golden(golden):
    lens = golden["sortagrad/lengths"]
    for epoch in range(4):
        for on in (0, 1):
            want = golden[f"sortagrad/order_e{epoch}_s{on}"]
            assert np.array_equal(oracle.oracle_sortagrad(lens, 16, epoch, 1234, bool(on)), want)
