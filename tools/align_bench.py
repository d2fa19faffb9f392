"""Timing of the f2/f3 paths (forced alignment, lattice export) on the English
shape, GPU (device-resident activations, CUDA events) beside the reference's
own viterbi_align / ctc_lattice (oracle/_ref build, one thread). Evidence for
DESIGN.md; not part of bench.py's contract."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_1512_02595_b200 import ctc  # noqa: E402
from paper_1512_02595_b200.synth import fixed_shape_batch  # noqa: E402


def gpu_ms(fn, reps=10):
    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    import torch

    A, T, L, B = 29, 700, 150, 64
    acts, flat, ll, il = fixed_shape_batch(A, T, L, B, seed=3)
    x = torch.from_numpy(acts).cuda()
    v_ms = gpu_ms(lambda: ctc.viterbi_align_batch(x, flat, ll, il))
    l_ms = gpu_ms(lambda: ctc.ctc_lattice_batch(x, flat, ll, il))
    print(f"GPU viterbi_align  B={B} T={T} L={L}: {v_ms:.3f} ms/batch = {B / v_ms * 1e3:.0f} utt/s")
    print(f"GPU ctc_lattice    B={B} T={T} L={L}: {l_ms:.3f} ms/batch = {B / l_ms * 1e3:.0f} utt/s")
    if oracle.ref_available():
        n = 8
        t0 = time.perf_counter()
        for b in range(n):
            oracle.ref_viterbi(acts[:, b, :].astype(np.float64), flat[b * L:(b + 1) * L], A - 1)
        v_cpu = (time.perf_counter() - t0) / n
        t0 = time.perf_counter()
        for b in range(n):
            oracle.ref_lattice(acts[:, b, :].astype(np.float64), flat[b * L:(b + 1) * L], A - 1)
        l_cpu = (time.perf_counter() - t0) / n
        print(f"CPU reference viterbi_align (1 thread): {1 / v_cpu:.0f} utt/s; ctc_lattice: {1 / l_cpu:.0f} utt/s")


if __name__ == "__main__":
    main()
