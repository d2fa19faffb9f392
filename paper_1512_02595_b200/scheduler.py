"""H1 host scheduler (C++ in libds2ctc.so; these are thin ctypes wrappers).

* ``sortagrad_order``  -- asr::trainer::sortagrad_order (trainer.cpp:58-91)
* ``rank_slice``       -- the reference's contiguous per-rank slice (trainer.cpp:140-143)
* ``shard_lpt``        -- the B200 re-deal of one global minibatch across GPUs,
                          longest-processing-time first on estimated cost
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def _i32(a):
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))
    return arr if arr.size else np.zeros(1, dtype=np.int32)


def sortagrad_order(lengths, global_batch: int, epoch: int, seed: int, sortagrad_on: bool = True) -> np.ndarray:
    lens = _i32(lengths)
    n = int(np.asarray(lengths).size)
    out = np.zeros(max(n, 1), dtype=np.int64)
    _lib.check(_lib.lib().ds2ctc_sortagrad_order(lens.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), n, global_batch,
                                                 epoch, seed, 1 if sortagrad_on else 0,
                                                 out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))),
               "ds2ctc_sortagrad_order")
    return out[:n]


def rank_slice(batch_n: int, minibatch_size: int, rank: int):
    b = ctypes.c_int()
    e = ctypes.c_int()
    _lib.check(_lib.lib().ds2ctc_rank_slice(batch_n, minibatch_size, rank, ctypes.byref(b), ctypes.byref(e)),
               "ds2ctc_rank_slice")
    return b.value, e.value


def shard_lpt(input_lengths, label_lengths, alphabet_size: int, world: int):
    """Returns (rank per utterance int32 [n], estimated load per rank float64 [world])."""
    il = _i32(input_lengths)
    ll = _i32(label_lengths)
    n = int(np.asarray(input_lengths).size)
    ranks = np.zeros(max(n, 1), dtype=np.int32)
    load = np.zeros(world, dtype=np.float64)
    P = ctypes.POINTER(ctypes.c_int)
    _lib.check(_lib.lib().ds2ctc_shard_lpt(il.ctypes.data_as(P), ll.ctypes.data_as(P), n, alphabet_size, world,
                                           ranks.ctypes.data_as(P),
                                           load.ctypes.data_as(ctypes.POINTER(ctypes.c_double))),
               "ds2ctc_shard_lpt")
    return ranks[:n], load


def shard_batch(input_lengths, label_lengths, alphabet_size: int, world: int, rank: int):
    """Indices (into the global minibatch) this rank computes, longest first."""
    ranks, _ = shard_lpt(input_lengths, label_lengths, alphabet_size, world)
    mine = np.where(ranks == rank)[0]
    il = np.asarray(input_lengths)
    return mine[np.argsort(-il[mine], kind="stable")] if mine.size else mine
