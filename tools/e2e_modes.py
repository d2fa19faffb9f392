"""Per-call host-path times (ds2ctc_compute_loss_host, English, pinned buffers):
prints a histogram of call times so a bimodal process state shows up, plus the
H2D / D2H copy bandwidth of this process's pinned buffers."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1512_02595_b200 import ctc  # noqa: E402
from paper_1512_02595_b200.synth import fixed_shape_batch  # noqa: E402


def main():
    import torch

    acts, flat, ll, il = fixed_shape_batch(29, 700, 150, 64, seed=3)
    pa = torch.from_numpy(acts).pin_memory()
    g = torch.empty(acts.shape, dtype=torch.float32).pin_memory()
    c = torch.empty(64, dtype=torch.float32).pin_memory()
    d = torch.empty(acts.shape, dtype=torch.float32, device="cuda")
    for _ in range(10):
        ctc.compute_ctc_loss_host(pa.numpy(), flat, ll, il, gradients=g.numpy(), costs=c.numpy())
    ts = []
    for _ in range(60):
        a = time.perf_counter()
        ctc.compute_ctc_loss_host(pa.numpy(), flat, ll, il, gradients=g.numpy(), costs=c.numpy())
        ts.append((time.perf_counter() - a) * 1e6)
    ts = np.array(ts)
    def bw(fn):
        torch.cuda.synchronize()
        a = time.perf_counter()
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        return acts.nbytes * 20 / (time.perf_counter() - a) / 1e9
    h2d = bw(lambda: d.copy_(pa, non_blocking=True))
    d2h = bw(lambda: g.copy_(d, non_blocking=True))
    print(f"cpu {os.sched_getaffinity(0) if len(os.sched_getaffinity(0)) < 16 else 'all'} "
          f"call us: min {ts.min():.0f} p50 {np.median(ts):.0f} p90 {np.percentile(ts, 90):.0f} max {ts.max():.0f} | "
          f"H2D {h2d:.1f} GB/s D2H {d2h:.1f} GB/s")


if __name__ == "__main__":
    main()
