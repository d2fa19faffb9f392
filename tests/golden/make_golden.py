"""Generates tests/golden/ctc_golden.npz from the REFERENCE's own fp64 build.

Run here (the container that has /root/reference):

    make -C oracle && python tests/golden/make_golden.py

Every cost / gradient in the fixture comes from ``asr::ctc::ctc_loss_reference``
(proj/src/ctc.cpp:171-207) compiled from the reference sources by
oracle/Makefile into oracle/_ref/libasr_ref.so, driven with the trainer's
convention (infeasible -> +inf cost, zero gradient rows; proj/src/trainer.cpp:
158-169). Inputs are fp32 ``[T_max][B][A]`` batches; the reference sees each
slice widened exactly to fp64. The fixture travels to the GPU box (where the
reference does not exist) and pins both the oracle restatement and the CUDA
path.

Cases
-----
* ``ka_*``       known answers from proj/tests/test_ctc.cpp:71-105,268-275
* ``fuzz_A{n}``  tiny fuzzed utterances in the style of test_ctc.cpp:107-124
                 (A <= 4+blank, T <= 6, L <= 3), grouped by alphabet size
* ``config1``    BASELINE.json configs[0]: A=29, T=150, L=40, B=16, seed 1234
* ``peaked``     A=29, variable T <= 200, logits N(0,1) x 8 (dynamic-range case)
* ``edge``       repeats (min_frames = 2L-1), empty labels, T < min_frames,
                 T = 0, zero-probability rows (-inf logits), a label that
                 contains the blank id, and logits shifted by +1e4
* ``sortagrad``  asr::trainer::sortagrad_order (trainer.cpp:58-91) orders
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1512_02595_b200.synth import Rng, make_batch  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ctc_golden.npz")


def pack(utts, alphabet):
    """utts: list of (logits T x A float array, label list). Returns batch arrays."""
    B = len(utts)
    t_max = max([u[0].shape[0] for u in utts] + [0])
    acts = np.zeros((t_max, B, alphabet), dtype=np.float32)
    il = np.zeros(B, dtype=np.int32)
    ll = np.zeros(B, dtype=np.int32)
    flat = []
    for b, (x, lab) in enumerate(utts):
        T = x.shape[0]
        acts[:T, b, :] = x.astype(np.float32)
        il[b] = T
        ll[b] = len(lab)
        flat.extend(int(c) for c in lab)
    return acts, np.asarray(flat, dtype=np.int32), ll, il


def add_case(store, name, acts, flat, ll, il, blank):
    costs, grads = oracle.ref_batch(acts, flat, ll, il, blank=blank, want_grad=True)
    store[f"{name}/acts"] = acts
    store[f"{name}/labels"] = flat
    store[f"{name}/label_lengths"] = ll
    store[f"{name}/input_lengths"] = il
    store[f"{name}/blank"] = np.int32(blank)
    store[f"{name}/costs"] = costs
    store[f"{name}/grads"] = grads
    print(f"{name:12s} A={acts.shape[2]:5d} B={ll.shape[0]:4d} Tmax={acts.shape[0]:5d} "
          f"feasible={int(np.isfinite(costs).sum())}/{costs.size}")


def main():
    store = {}

    # Known answers (test_ctc.cpp). Log-probabilities are valid logits (softmax is a no-op on them).
    half = math.log(0.5)
    add_case(store, "ka_single", *pack([(np.full((1, 2), half), [0])], 2), blank=1)
    add_case(store, "ka_two", *pack([(np.full((2, 2), half), [0])], 2), blank=1)
    add_case(store, "ka_repeat", *pack([(np.full((2, 2), half), [0, 0]), (np.full((3, 2), half), [0, 0])], 2),
             blank=1)
    add_case(store, "ka_empty", *pack([(np.full((4, 3), math.log(1.0 / 3)), [])], 3), blank=2)

    # Fuzzed tiny utterances, grouped by alphabet size (blank = alphabet index, as the tests use).
    rng = Rng(20260808)
    groups = {}
    for _ in range(160):
        alphabet = 1 + int(rng.below(1, 4)[0])
        frames = 1 + int(rng.below(1, 6)[0])
        L = int(rng.below(1, 4)[0])
        label = [int(c) for c in rng.below(L, alphabet)] if L else []
        logits = rng.uniform(frames * (alphabet + 1)).reshape(frames, alphabet + 1) * 4.0 - 2.0
        groups.setdefault(alphabet, []).append((logits, label))
    for alphabet, utts in sorted(groups.items()):
        add_case(store, f"fuzz_A{alphabet + 1}", *pack(utts, alphabet + 1), blank=alphabet)

    # BASELINE configs[0].
    acts, flat, ll, il = make_batch(29, [150] * 16, [40] * 16, seed=1234)
    add_case(store, "config1", acts, flat, ll, il, blank=28)

    # Peaked logits, variable lengths.
    T = [200, 180, 150, 120, 90, 60, 40, 25]
    L = [60, 50, 40, 35, 20, 15, 10, 5]
    acts, flat, ll, il = make_batch(29, T, L, seed=99, scale=8.0)
    add_case(store, "peaked", acts, flat, ll, il, blank=28)

    # Edge sweep (A=6, blank 5).
    A, blank = 6, 5
    r = Rng(4242)

    def rnd(T):
        return r.normal(T * A).reshape(T, A)

    edge = [
        (rnd(9), [1, 1, 1, 1, 1]),        # all repeats: min_frames = 2L-1 = 9, exactly feasible
        (rnd(8), [1, 1, 1, 1, 1]),        # one frame short: infeasible
        (rnd(7), []),                      # empty label
        (np.zeros((0, A)), []),            # T = 0, empty label (reference UB; defined as loss 0)
        (np.zeros((0, A)), [2]),           # T = 0, non-empty label: infeasible
        (rnd(3), [0, 1, 2]),               # T == L: single forced path
        (rnd(12), [0, 5, 2]),              # label containing the blank id (accepted, no validation)
        (rnd(10) + 1e4, [3, 1, 3]),        # shifted logits (shift invariance)
        (rnd(11), [2, 2, 3, 3, 4]),        # mixed repeats
        (rnd(1), []),                      # single frame, empty label
        (rnd(1), [4]),                     # single frame, single symbol
    ]
    zp = rnd(6)
    zp[:, :blank] = -np.inf                # only blank possible -> label {0,1} has p = 0
    edge.append((zp, [0, 1]))
    add_case(store, "edge", *pack(edge, A), blank=blank)

    # SortaGrad orders (trainer.cpp:58-91).
    lens = (50 + Rng(5).below(97, 1451)).astype(np.int32)
    lens[10:20] = 700  # ties exercise stability
    store["sortagrad/lengths"] = lens
    for epoch in range(4):
        for on in (0, 1):
            store[f"sortagrad/order_e{epoch}_s{on}"] = oracle.ref_sortagrad(lens, 16, epoch, 1234, bool(on))

    np.savez_compressed(OUT, **store)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
