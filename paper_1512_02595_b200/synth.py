"""Synthetic CTC batches with the reference's own random stream.

The reference seeds everything through ``asr::Rng`` (SplitMix64 +
Box-Muller, proj/include/asr/common.hpp:92-118). SplitMix64's n-th output
is a pure function of ``seed + n * gamma``, so the stream vectorises: this
module reproduces it in numpy (uint64 wrap-around arithmetic) and draws

* logits ``x[t][b][k] ~ N(0, 1) * scale`` rounded to fp32 (time-major
  ``[T_max][B][A]``, the layout of the C-ABI), and
* labels ``y_b[i] ~ U{0 .. A-2}`` (blank is ``A-1``, trainer.cpp:127).

It is data plumbing for tests and the benchmark, not a CTC implementation.
"""
from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


class Rng:
    """Vectorised ``asr::Rng`` (common.hpp:92-131). Stream-identical to the C++ one."""

    def __init__(self, seed: int):
        self.state = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)

    def next_u64(self, n: int) -> np.ndarray:
        with np.errstate(over="ignore"):
            k = np.arange(1, n + 1, dtype=np.uint64)
            z = self.state + k * _GAMMA
            self.state = self.state + np.uint64(n) * _GAMMA
            z = (z ^ (z >> np.uint64(30))) * _M1
            z = (z ^ (z >> np.uint64(27))) * _M2
            return z ^ (z >> np.uint64(31))

    def uniform(self, n: int) -> np.ndarray:
        return (self.next_u64(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def below(self, n: int, bound: int) -> np.ndarray:
        return (self.next_u64(n) % np.uint64(bound)).astype(np.int64)

    def normal(self, n: int) -> np.ndarray:
        u = self.uniform(2 * n).reshape(n, 2)
        u1 = np.maximum(u[:, 0], 1e-300)
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * 3.14159265358979323846 * u[:, 1])


def make_batch(alphabet: int, input_lengths, label_lengths, seed: int = 1234, scale: float = 1.0):
    """Returns (acts fp32 [T_max][B][A], flat_labels int32, label_lengths int32, input_lengths int32)."""
    input_lengths = np.asarray(input_lengths, dtype=np.int32)
    label_lengths = np.asarray(label_lengths, dtype=np.int32)
    B = int(input_lengths.shape[0])
    t_max = int(input_lengths.max()) if B else 0
    rng = Rng(seed)
    acts = (rng.normal(t_max * B * alphabet) * scale).astype(np.float32).reshape(t_max, B, alphabet)
    flat = rng.below(int(label_lengths.sum()), max(alphabet - 1, 1)).astype(np.int32)
    return np.ascontiguousarray(acts), flat, label_lengths, input_lengths


def fixed_shape_batch(alphabet: int, T: int, L: int, B: int, seed: int = 1234, scale: float = 1.0):
    """The BASELINE.json fixed shapes (config 1, English, Mandarin)."""
    return make_batch(alphabet, [T] * B, [L] * B, seed=seed, scale=scale)


def sortagrad_lengths(n: int, seed: int = 7, t_lo: int = 50, t_hi: int = 1500, l_lo: int = 5, l_hi: int = 300):
    """Config 4 lengths: T_b ~ U[t_lo, t_hi], L_b ~ U[l_lo, min(l_hi, T_b // 2)]."""
    rng = Rng(seed)
    T = t_lo + rng.below(n, t_hi - t_lo + 1)
    hi = np.minimum(l_hi, T // 2)
    L = l_lo + (rng.next_u64(n) % (hi - l_lo + 1).astype(np.uint64)).astype(np.int64)
    return T.astype(np.int32), L.astype(np.int32)
