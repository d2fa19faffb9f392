"""ctypes front-end of the CPU parity checkers (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` arm may import this package. It loads

* ``oracle/liboracle_ctc.so`` -- the plain-C fp64 restatement of the
  reference CTC (oracle/ctc_oracle.c), and
* ``oracle/_ref/libasr_ref.so`` -- the reference's own fp64 build
  (oracle/Makefile compiles it from /root/reference sources in place).

Neither is ever on the product path; the product (``paper_1512_02595_b200``)
does not import this package.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle_ctc.so")
REF_SO = os.path.join(HERE, "_ref", "libasr_ref.so")

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_float_p = ctypes.POINTER(ctypes.c_float)
_c_int_p = ctypes.POINTER(ctypes.c_int)
_c_i64_p = ctypes.POINTER(ctypes.c_int64)

_oracle = None
_ref = None


def build():
    """Compile the oracle (and the reference build when its sources are present)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a, ctype):
    return a.ctypes.data_as(ctype) if a is not None else None


def oracle_lib():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            build()
        lib = ctypes.CDLL(ORACLE_SO)
        lib.orc_log_sum_exp_guarded.restype = ctypes.c_double
        lib.orc_log_sum_exp_guarded.argtypes = [ctypes.c_double, ctypes.c_double]
        lib.orc_ctc_loss.restype = ctypes.c_int
        lib.orc_ctc_loss.argtypes = [_c_double_p, ctypes.c_int, ctypes.c_int, _c_int_p, ctypes.c_int, ctypes.c_int,
                                     _c_double_p, _c_double_p]
        lib.orc_ctc_lattice.restype = None
        lib.orc_ctc_lattice.argtypes = [_c_double_p, ctypes.c_int, ctypes.c_int, _c_int_p, ctypes.c_int,
                                        ctypes.c_int, _c_double_p, _c_double_p, _c_double_p]
        lib.orc_viterbi_align.restype = ctypes.c_int
        lib.orc_viterbi_align.argtypes = [_c_double_p, ctypes.c_int, ctypes.c_int, _c_int_p, ctypes.c_int,
                                          ctypes.c_int, _c_int_p]
        lib.orc_min_frames.restype = ctypes.c_int
        lib.orc_min_frames.argtypes = [_c_int_p, ctypes.c_int]
        lib.orc_ctc_batch.restype = None
        lib.orc_ctc_batch.argtypes = [_c_float_p, _c_int_p, _c_int_p, _c_int_p, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, _c_double_p, _c_double_p, ctypes.c_int]
        lib.orc_sortagrad_order.restype = None
        lib.orc_sortagrad_order.argtypes = [_c_int_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                            ctypes.c_int, _c_i64_p]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference sources; run make -C oracle)")
        lib = ctypes.CDLL(REF_SO)
        lib.ref_ctc_loss.restype = ctypes.c_int
        lib.ref_ctc_loss.argtypes = [_c_double_p, ctypes.c_int, ctypes.c_int, _c_int_p, ctypes.c_int, ctypes.c_int,
                                     _c_double_p, _c_double_p]
        lib.ref_ctc_loss_parallel.restype = ctypes.c_int
        lib.ref_ctc_loss_parallel.argtypes = [_c_double_p, ctypes.c_int, ctypes.c_int, _c_int_p, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, _c_double_p, _c_double_p]
        lib.ref_ctc_lattice.restype = None
        lib.ref_ctc_lattice.argtypes = [_c_double_p, ctypes.c_int, ctypes.c_int, _c_int_p, ctypes.c_int,
                                        ctypes.c_int, _c_double_p, _c_double_p, _c_double_p]
        lib.ref_viterbi_align.restype = ctypes.c_int
        lib.ref_viterbi_align.argtypes = [_c_double_p, ctypes.c_int, ctypes.c_int, _c_int_p, ctypes.c_int,
                                          ctypes.c_int, _c_int_p]
        lib.ref_min_frames.restype = ctypes.c_int
        lib.ref_min_frames.argtypes = [_c_int_p, ctypes.c_int]
        lib.ref_sortagrad_order.restype = None
        lib.ref_sortagrad_order.argtypes = [_c_int_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                            ctypes.c_int, _c_i64_p]
        lib.ref_fc_backward.restype = None
        lib.ref_fc_backward.argtypes = [_c_float_p, _c_float_p, _c_int_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_int, _c_float_p, _c_double_p, _c_double_p, _c_double_p]
        lib.ref_ctc_batch.restype = None
        lib.ref_ctc_batch.argtypes = [_c_float_p, _c_int_p, _c_int_p, _c_int_p, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, _c_double_p, _c_float_p, ctypes.c_int]
        _ref = lib
    return _ref


# ---------------------------------------------------------------- per utterance

def _utt_args(logits, label):
    x = np.ascontiguousarray(logits, dtype=np.float64)
    lab = np.ascontiguousarray(np.asarray(label, dtype=np.int32).reshape(-1))
    if lab.size == 0:
        lab = np.zeros(1, dtype=np.int32)
        L = 0
    else:
        L = int(np.asarray(label).size)
    return x, lab, L


def _loss(fn, logits, label, blank, want_grad=True):
    x, lab, L = _utt_args(logits, label)
    T, C = x.shape
    loss = ctypes.c_double()
    grad = np.zeros((max(T, 1), C), dtype=np.float64) if want_grad else None
    ok = fn(_ptr(x, _c_double_p), T, C, _ptr(lab, _c_int_p), L, blank, ctypes.byref(loss),
            _ptr(grad, _c_double_p))
    return bool(ok), loss.value, (grad[:T] if (ok and want_grad) else None)


def oracle_loss(logits, label, blank, want_grad=True):
    """Oracle restatement of ctc_loss_reference -> (feasible, loss, grad T x C or None)."""
    return _loss(oracle_lib().orc_ctc_loss, logits, label, blank, want_grad)


def ref_loss(logits, label, blank, want_grad=True):
    """The reference's own ctc_loss_reference -> (feasible, loss, grad T x C or None)."""
    return _loss(ref_lib().ref_ctc_loss, logits, label, blank, want_grad)


def ref_loss_parallel(logits, label, blank, workers, want_grad=True):
    x, lab, L = _utt_args(logits, label)
    T, C = x.shape
    loss = ctypes.c_double()
    grad = np.zeros((max(T, 1), C), dtype=np.float64) if want_grad else None
    ok = ref_lib().ref_ctc_loss_parallel(_ptr(x, _c_double_p), T, C, _ptr(lab, _c_int_p), L, blank, workers,
                                         ctypes.byref(loss), _ptr(grad, _c_double_p))
    return bool(ok), loss.value, (grad[:T] if (ok and want_grad) else None)


def _lattice(fn, logits, label, blank):
    x, lab, L = _utt_args(logits, label)
    T, C = x.shape
    S = 2 * L + 1
    alpha = np.zeros((S, T), dtype=np.float64)
    beta = np.zeros((S, T), dtype=np.float64)
    lp = ctypes.c_double()
    fn(_ptr(x, _c_double_p), T, C, _ptr(lab, _c_int_p), L, blank, _ptr(alpha, _c_double_p),
       _ptr(beta, _c_double_p), ctypes.byref(lp))
    return alpha, beta, lp.value


def oracle_lattice(logits, label, blank):
    return _lattice(oracle_lib().orc_ctc_lattice, logits, label, blank)


def ref_lattice(logits, label, blank):
    return _lattice(ref_lib().ref_ctc_lattice, logits, label, blank)


def _viterbi(fn, logits, label, blank):
    x, lab, L = _utt_args(logits, label)
    T, C = x.shape
    out = np.zeros(max(T, 1), dtype=np.int32)
    rc = fn(_ptr(x, _c_double_p), T, C, _ptr(lab, _c_int_p), L, blank, _ptr(out, _c_int_p))
    return None if rc != 0 else out[:T]


def oracle_viterbi(logits, label, blank):
    return _viterbi(oracle_lib().orc_viterbi_align, logits, label, blank)


def ref_viterbi(logits, label, blank):
    return _viterbi(ref_lib().ref_viterbi_align, logits, label, blank)


def oracle_min_frames(label):
    lab = np.ascontiguousarray(np.asarray(label, dtype=np.int32).reshape(-1))
    if lab.size == 0:
        return 0
    return oracle_lib().orc_min_frames(_ptr(lab, _c_int_p), int(lab.size))


# ---------------------------------------------------------------- batched

def _batch_args(acts, flat_labels, label_lengths, input_lengths):
    acts = np.ascontiguousarray(acts, dtype=np.float32)
    flat = np.ascontiguousarray(flat_labels, dtype=np.int32)
    if flat.size == 0:
        flat = np.zeros(1, dtype=np.int32)
    ll = np.ascontiguousarray(label_lengths, dtype=np.int32)
    il = np.ascontiguousarray(input_lengths, dtype=np.int32)
    return acts, flat, ll, il


def oracle_batch(acts, flat_labels, label_lengths, input_lengths, blank=None, want_grad=True, nthreads=1):
    """Oracle over [T_max][B][A] fp32 -> (costs fp64 [B], grads fp64 [T_max][B][A] or None)."""
    acts, flat, ll, il = _batch_args(acts, flat_labels, label_lengths, input_lengths)
    A = acts.shape[2]
    B = ll.shape[0]
    blank = A - 1 if blank is None else blank
    costs = np.zeros(max(B, 1), dtype=np.float64)
    grads = np.zeros(acts.shape, dtype=np.float64) if want_grad else None
    oracle_lib().orc_ctc_batch(_ptr(acts, _c_float_p), _ptr(flat, _c_int_p), _ptr(ll, _c_int_p),
                               _ptr(il, _c_int_p), A, B, blank, _ptr(costs, _c_double_p),
                               _ptr(grads, _c_double_p), nthreads)
    return costs[:B], grads


def ref_batch(acts, flat_labels, label_lengths, input_lengths, blank=None, want_grad=True, nthreads=1):
    """Reference build over [T_max][B][A] fp32 -> (costs fp64 [B], grads fp32 [T_max][B][A] or None)."""
    acts, flat, ll, il = _batch_args(acts, flat_labels, label_lengths, input_lengths)
    A = acts.shape[2]
    B = ll.shape[0]
    blank = A - 1 if blank is None else blank
    costs = np.zeros(max(B, 1), dtype=np.float64)
    grads = np.zeros(acts.shape, dtype=np.float32) if want_grad else None
    ref_lib().ref_ctc_batch(_ptr(acts, _c_float_p), _ptr(flat, _c_int_p), _ptr(ll, _c_int_p), _ptr(il, _c_int_p),
                            A, B, blank, _ptr(costs, _c_double_p), _ptr(grads, _c_float_p), nthreads)
    return costs[:B], grads


def _sortagrad(fn, lengths, global_batch, epoch, seed, sortagrad_on=True):
    lens = np.ascontiguousarray(lengths, dtype=np.int32)
    out = np.zeros(max(lens.size, 1), dtype=np.int64)
    fn(_ptr(lens, _c_int_p), int(lens.size), global_batch, epoch, seed, 1 if sortagrad_on else 0,
       _ptr(out, _c_i64_p))
    return out[:lens.size]


def oracle_sortagrad(lengths, global_batch, epoch, seed, sortagrad_on=True):
    return _sortagrad(oracle_lib().orc_sortagrad_order, lengths, global_batch, epoch, seed, sortagrad_on)


def ref_sortagrad(lengths, global_batch, epoch, seed, sortagrad_on=True):
    return _sortagrad(ref_lib().ref_sortagrad_order, lengths, global_batch, epoch, seed, sortagrad_on)


def ref_fc_backward(x, dlogits, input_lengths, w):
    """The reference's output-layer backward (asr::nn FullyConnectedLayer, nn.cpp:874-899) on
    batched [T_max][B][H] inputs and [T_max][B][A] gradients -> (dw A x H, db A, dx [T_max][B][H]), fp64."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    g = np.ascontiguousarray(dlogits, dtype=np.float32)
    w = np.ascontiguousarray(w, dtype=np.float32)
    il = np.ascontiguousarray(input_lengths, dtype=np.int32)
    Tmax, B, H = x.shape
    A = g.shape[2]
    dw = np.zeros((A, H), np.float64)
    db = np.zeros(A, np.float64)
    dx = np.zeros((Tmax, B, H), np.float64)
    ref_lib().ref_fc_backward(_ptr(x, _c_float_p), _ptr(g, _c_float_p), _ptr(il, _c_int_p), B, Tmax, H, A,
                              _ptr(w, _c_float_p), _ptr(dw, _c_double_p), _ptr(db, _c_double_p),
                              _ptr(dx, _c_double_p))
    return dw, db, dx
