"""Debug probe for ds2ctc_fc_backward on the GPU box: prints errors and output stats."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1512_02595_b200 import ctc as dctc  # noqa: E402

for (A, H, T, B) in [(32, 128, 32, 1), (29, 256, 160, 8), (128, 128, 128, 1)]:
    rng = np.random.default_rng(0)
    x = rng.standard_normal((T, B, H)).astype(np.float32)
    g = rng.standard_normal((T, B, A)).astype(np.float32)
    w = rng.standard_normal((A, H)).astype(np.float32)
    try:
        dw, db, dx = dctc.fc_backward(torch.from_numpy(g).cuda(), torch.from_numpy(x).cuda(),
                                      torch.from_numpy(w).cuda())
        torch.cuda.synchronize()
    except Exception as e:  # noqa: BLE001
        print("ERROR", A, H, T, B, repr(e))
        continue
    G = g.reshape(-1, A).astype(np.float64)
    X = x.reshape(-1, H).astype(np.float64)
    rdw = G.T @ X
    rdx = G @ w.astype(np.float64)
    gdw = dw.cpu().numpy()
    gdx = dx.cpu().numpy().reshape(-1, H)
    print(f"A{A} H{H} rows{T*B}: db err {np.abs(db.cpu().numpy() - G.sum(0)).max():.3e}  "
          f"dW err {np.abs(gdw - rdw).max():.3e} (max {np.abs(rdw).max():.2e}, nonzero {np.count_nonzero(gdw)})  "
          f"dx err {np.abs(gdx - rdx).max():.3e} (max {np.abs(rdx).max():.2e}, nonzero {np.count_nonzero(gdx)})")
    # ratio patterns
    if np.count_nonzero(gdw):
        nz = np.abs(rdw) > 1
        print("   dW ratio sample", (gdw[nz] / rdw[nz])[:8])
        # check transposition hypotheses
        print("   dW vs transposed? ", np.abs(gdw[:min(A, H), :min(A, H)] - rdw[:min(A, H), :min(A, H)].T).max())
    if np.count_nonzero(gdx):
        print("   dx[0,:8]", gdx[0, :8], "ref", rdx[0, :8])
        print("   dx[1,:8]", gdx[1, :8], "ref", rdx[1, :8])
