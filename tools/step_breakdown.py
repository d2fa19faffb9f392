"""Where the English step's time goes outside k_pair (evidence for DESIGN.md):
CUDA-event time of back-to-back calls of (a) ds2ctc_compute_loss alone,
(b) + ds2ctc_loss_sum, (c) a bare pinned H2D copy of the metadata size, with
the library's own stage events for k_pair."""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1512_02595_b200 import _lib, ctc  # noqa: E402
from paper_1512_02595_b200.synth import fixed_shape_batch  # noqa: E402


def main():
    import torch

    A, T, L, B = 29, 700, 150, 64
    acts, flat, ll, il = fixed_shape_batch(A, T, L, B, seed=3)
    x = torch.from_numpy(acts).cuda()
    g = torch.empty_like(x)
    costs = torch.empty(B, device="cuda")
    pair = torch.empty(2, dtype=torch.float64, device="cuda")
    ws = ctc.Workspace(torch.device("cuda", 0))
    ws_ptr, ws_bytes = ws.get(ctc.workspace_size(ll, il, A))
    lib = _lib.lib()
    s = torch.cuda.current_stream()
    P = ctypes.POINTER(ctypes.c_int)
    lab, lla, ila = [np.ascontiguousarray(v, dtype=np.int32) for v in (flat, ll, il)]

    def call(with_sum):
        lib.ds2ctc_compute_loss_checked(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(g.data_ptr()),
                                        lab.ctypes.data_as(P), lla.ctypes.data_as(P), ila.ctypes.data_as(P), A, B,
                                        A - 1, ctypes.c_void_p(costs.data_ptr()), ctypes.c_void_p(ws_ptr), ws_bytes,
                                        ctypes.c_void_p(s.cuda_stream))
        if with_sum:
            lib.ds2ctc_loss_sum(ctypes.c_void_p(costs.data_ptr()), B, ctypes.c_void_p(pair.data_ptr()),
                                ctypes.c_void_p(s.cuda_stream))

    def timed(fn, n=50):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def per_step_flushed(n=30):
        st = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        en = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        for k in range(n):
            flush.zero_()
            st[k].record()
            call(True)
            en[k].record()
        torch.cuda.synchronize()
        return float(np.mean([a.elapsed_time(b) for a, b in zip(st, en)])) * 1e3

    per_step_flushed(5)
    print(f"bench-style step (L2 flushed) {per_step_flushed():8.1f} us")
    meta = 64 * 64 + 4 * (5 * int(ll.sum()) + 3 * B)
    h = torch.empty(meta, dtype=torch.uint8).pin_memory()
    d = torch.empty(meta, dtype=torch.uint8, device="cuda")
    print(f"compute_loss alone          {timed(lambda: call(False)):8.1f} us/call")
    print(f"compute_loss + loss_sum     {timed(lambda: call(True)):8.1f} us/call")
    print(f"pinned H2D of {meta} B       {timed(lambda: d.copy_(h, non_blocking=True)):8.1f} us/copy")
    lib.ds2ctc_profile_enable(20)
    for _ in range(20):
        call(False)
    ms = (ctypes.c_float * 4)()
    vals = []
    for k in range(20):
        lib.ds2ctc_profile_read(k, ms)
        vals.append(ms[0])
    lib.ds2ctc_profile_enable(0)
    print(f"k_pair (library events)     {1e3 * float(np.mean(vals)):8.1f} us")


if __name__ == "__main__":
    main()
