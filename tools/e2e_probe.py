"""Host-path (ds2ctc_compute_loss_host) time split: full call, cost-only, and
a tiny batch (fixed overheads); evidence for the e2e number."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1512_02595_b200 import ctc  # noqa: E402
from paper_1512_02595_b200.synth import fixed_shape_batch  # noqa: E402


def t(fn, n=30):
    for _ in range(5):
        fn()
    a = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - a) / n * 1e6


def main():
    import torch

    acts, flat, ll, il = fixed_shape_batch(29, 700, 150, 64, seed=3)
    pa = torch.from_numpy(acts).pin_memory().numpy()
    g = torch.empty(acts.shape, dtype=torch.float32).pin_memory().numpy()
    c = torch.empty(64, dtype=torch.float32).pin_memory().numpy()
    print(f"full (grads)   {t(lambda: ctc.compute_ctc_loss_host(pa, flat, ll, il, gradients=g, costs=c)):8.1f} us")
    print(f"cost only      {t(lambda: ctc.compute_ctc_loss_host(pa, flat, ll, il, want_grad=False, costs=c)):8.1f} us")
    a1, f1, l1, i1 = fixed_shape_batch(29, 700, 150, 1, seed=3)
    print(f"B=1            {t(lambda: ctc.compute_ctc_loss_host(a1, f1, l1, i1)):8.1f} us")
    a2, f2, l2, i2 = fixed_shape_batch(29, 20, 5, 1, seed=3)
    print(f"B=1 T=20       {t(lambda: ctc.compute_ctc_loss_host(a2, f2, l2, i2)):8.1f} us")


if __name__ == "__main__":
    main()
