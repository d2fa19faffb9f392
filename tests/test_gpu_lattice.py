"""GPU lattice export (ds2ctc_ctc_lattice) vs the reference's ctc_lattice
(proj/src/ctc.cpp:145-169) through the oracle restatement (pinned to the
reference build in test_oracle.py): same -inf pattern, finite cells within
1e-9 (fp64, CUDA vs libm exp/log1p differ by ulps), and the cancellation
property the column-parallel scheme relies on (test_ctc.cpp:172-199):
log_sum_exp_s(alpha(s, t) + beta(s, t)) = log p for every frame t."""
import numpy as np
import pytest

import oracle
from paper_1512_02595_b200 import ctc as dctc
from paper_1512_02595_b200.synth import fixed_shape_batch, make_batch

pytestmark = pytest.mark.gpu


def check(acts, flat, ll, il, blank):
    import torch

    x = torch.from_numpy(np.ascontiguousarray(acts, dtype=np.float32)).cuda()
    alpha, beta, lp = dctc.ctc_lattice_batch(x, flat, ll, il, blank=blank)
    alpha, beta, lp = alpha.cpu().numpy(), beta.cpu().numpy(), lp.cpu().numpy()
    offs = np.concatenate([[0], np.cumsum(ll)]).astype(np.int64)
    cell = 0
    for b in range(len(il)):
        T, L = int(il[b]), int(ll[b])
        S = 2 * L + 1
        label = [int(c) for c in flat[offs[b]:offs[b + 1]]]
        ra, rb, rlp = oracle.oracle_lattice(acts[:T, b, :].astype(np.float64), label, blank)
        ga = alpha[cell:cell + S * T].reshape(S, T)
        gb = beta[cell:cell + S * T].reshape(S, T)
        cell += S * T
        for g, r in ((ga, ra), (gb, rb)):
            assert np.array_equal(np.isneginf(g), np.isneginf(r))
            fin = np.isfinite(r)
            assert np.allclose(g[fin], r[fin], rtol=1e-12, atol=1e-9)
        assert (np.isneginf(lp[b]) and np.isneginf(rlp)) or abs(lp[b] - rlp) <= 1e-9 * max(1.0, abs(rlp))
        if np.isfinite(rlp):
            comb = ga + gb
            m = comb.max(axis=0)
            per_t = m + np.log(np.exp(comb - m).sum(axis=0))
            assert np.allclose(per_t, lp[b], atol=1e-8)


def test_lattice_small_random(cuda):
    T = [1, 2, 5, 9, 17, 30, 3, 12]
    L = [0, 1, 2, 4, 6, 8, 3, 0]
    acts, flat, ll, il = make_batch(7, T, L, seed=99)
    check(acts, flat, ll, il, 6)


def test_lattice_config1(cuda):
    acts, flat, ll, il = fixed_shape_batch(29, 150, 40, 4, seed=1)
    check(acts, flat, ll, il, 28)


def test_lattice_rejects_empty_input(cuda):
    import torch

    x = torch.zeros((1, 2, 5), dtype=torch.float32, device="cuda")
    with pytest.raises(Exception):
        dctc.ctc_lattice_batch(x, [1], [1, 0], [1, 0], blank=4)
