"""The CTC gradient's consumer: the output fully connected
layer's backward on tcgen05 tensor cores (ds2ctc_fc_backward), checked
against the reference's OWN FullyConnectedLayer::backward (nn.cpp:874-899,
built from the reference sources into oracle/_ref, fp64), and the
device-resident trainer step: ds2ctc_compute_loss -> ds2ctc_fc_backward with
no host round trip, against the reference's ctc_loss_reference ->
FullyConnectedLayer::backward (trainer.cpp:155-171).

Tolerance (tf32 products: 10-bit mantissa, fp32 accumulation): per output
|err| <= 4e-3 * max|ref| of that output and relative Frobenius error <= 2e-3.
"""
import numpy as np
import pytest

import oracle
from paper_1512_02595_b200 import ctc as dctc
from paper_1512_02595_b200.synth import make_batch, sortagrad_lengths

pytestmark = pytest.mark.gpu


def close_tf32(got, ref, what):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    scale = max(np.abs(ref).max(), 1e-30)
    err = np.abs(got - ref).max() / scale
    fro = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-30)
    print(f"FC {what}: max err / max|ref| {err:.2e}, frobenius rel {fro:.2e}")
    assert err <= 4e-3 and fro <= 2e-3, (what, err, fro)


@pytest.mark.parametrize("A,H,B,seed", [(29, 256, 8, 1), (29, 2560, 4, 2), (600, 384, 4, 3), (6000, 128, 2, 4)])
def test_fc_backward_matches_reference(cuda, A, H, B, seed):
    import torch

    rng = np.random.default_rng(seed)
    T = rng.integers(20, 160, size=B).astype(np.int32)
    T[0] = 160
    Tm = int(T.max())
    x = rng.standard_normal((Tm, B, H)).astype(np.float32)
    g = (rng.standard_normal((Tm, B, A)) * 0.05).astype(np.float32)
    for b in range(B):
        g[T[b]:, b] = 0.0  # padded frames are zero rows (the CTC contract)
    w = (rng.standard_normal((A, H)) * 0.02).astype(np.float32)
    dw, db, dx = dctc.fc_backward(torch.from_numpy(g).cuda(), torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda())
    torch.cuda.synchronize()
    rdw, rdb, rdx = oracle.ref_fc_backward(x, g, T, w)
    close_tf32(dw.cpu().numpy(), rdw, f"dW A{A} H{H}")
    close_tf32(db.cpu().numpy(), rdb, f"db A{A}")
    mask = (np.arange(Tm)[:, None] < T[None, :])
    close_tf32(dx.cpu().numpy()[mask], rdx[mask], f"dx A{A} H{H}")


def test_trainer_step_device_resident(cuda):
    # one data-parallel shard's CTC + output-FC backward, the gradient never
    # leaving the device, vs the reference trainer's per-utterance loop
    import torch

    A, H = 29, 512
    T, L = sortagrad_lengths(24, seed=5)
    acts, flat, ll, il = make_batch(A, T, L, seed=8)
    rng = np.random.default_rng(9)
    x = rng.standard_normal((acts.shape[0], acts.shape[1], H)).astype(np.float32)
    w = (rng.standard_normal((A, H)) * 0.02).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    costs, grads = dctc.compute_ctc_loss(torch.from_numpy(acts).cuda(), flat, ll, il)
    dw, db, dx = dctc.fc_backward(grads, xd, torch.from_numpy(w).cuda())
    torch.cuda.synchronize()
    rc, rg = oracle.ref_batch(acts, flat, ll, il, nthreads=8)
    rdw, rdb, rdx = oracle.ref_fc_backward(x, rg, il, w)
    assert np.allclose(costs.cpu().numpy(), rc, rtol=1e-4)
    close_tf32(dw.cpu().numpy(), rdw, "step dW")
    close_tf32(db.cpu().numpy(), rdb, "step db")
    mask = (np.arange(acts.shape[0])[:, None] < il[None, :])
    close_tf32(dx.cpu().numpy()[mask], rdx[mask], "step dx")
