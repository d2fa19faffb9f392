"""Host-side mirror of the reference CTC interface, over the C-ABI.

Reference interface (proj/include/asr/ctc.hpp:62-87):

    struct CtcResult { bool feasible; real loss; Matrix logit_grad; };
    CtcResult ctc_loss_reference(const Matrix& frame_logits,
                                 const std::vector<int>& label, int blank);

``ctc_loss`` keeps that signature and meaning (one utterance, T x A logits,
blank passed explicitly, loss = -log p, gradient w.r.t. pre-softmax logits,
infeasible -> feasible=False, loss=+inf, empty gradient), computed on the
B200 through ``ds2ctc_compute_loss_host``. ``compute_ctc_loss`` is the
batched device entry point the trainer loop (trainer.cpp:155-171) maps onto:
``[T_max][B][A]`` fp32 CUDA activations in, per-utterance costs and
``[T_max][B][A]`` gradients out, all on the caller's CUDA stream.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib

_ip = ctypes.POINTER(ctypes.c_int)


@dataclass
class CtcResult:
    """asr::ctc::CtcResult (ctc.hpp:62-66)."""

    feasible: bool
    loss: float
    logit_grad: np.ndarray  # T x A; empty (0 x 0) when infeasible


def _i32(a) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))
    return arr if arr.size else np.zeros(1, dtype=np.int32)


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(_ip)


def workspace_size(label_lengths, input_lengths, alphabet_size: int) -> int:
    """ds2ctc_get_workspace_size: device bytes needed for one call."""
    ll = _i32(label_lengths)
    il = _i32(input_lengths)
    B = int(np.asarray(label_lengths).size)
    out = ctypes.c_size_t()
    _lib.check(_lib.lib().ds2ctc_get_workspace_size(_iptr(ll), _iptr(il), alphabet_size, B, ctypes.byref(out)),
               "ds2ctc_get_workspace_size")
    return int(out.value)


class Workspace:
    """Grow-only device workspace (a torch uint8 buffer, 256-byte aligned)."""

    def __init__(self, device=None):
        self.device = device
        self.buf = None

    def get(self, nbytes: int):
        import torch

        if self.buf is None or self.buf.numel() < nbytes + 256:
            self.buf = torch.empty(max(nbytes + 256, 1 << 20), dtype=torch.uint8, device=self.device)
        ptr = self.buf.data_ptr()
        return (ptr + 255) // 256 * 256, self.buf.numel() - ((ptr + 255) // 256 * 256 - ptr)


_default_ws = {}


def compute_ctc_loss(activations, flat_labels, label_lengths, input_lengths, blank: Optional[int] = None,
                     want_grad: bool = True, gradients=None, costs=None, workspace: Optional[Workspace] = None,
                     stream=None):
    """Batched CTC on the GPU via ds2ctc_compute_loss_checked.

    activations: torch.float32 CUDA tensor [T_max, B, A] (time-major, contiguous),
    T_max == max(input_lengths). flat_labels / label_lengths / input_lengths are host
    int sequences. Returns (costs [B] fp32 CUDA, gradients [T_max, B, A] or None).
    Asynchronous on `stream` (default: torch's current stream).
    """
    import torch

    if not (activations.is_cuda and activations.dtype == torch.float32 and activations.is_contiguous()):
        raise ValueError("activations must be a contiguous float32 CUDA tensor [T, B, A]")
    T_max, B, A = activations.shape
    ll = _i32(label_lengths)
    il = _i32(input_lengths)
    labels = _i32(flat_labels)
    if int(np.asarray(input_lengths).size) != B or int(np.asarray(label_lengths).size) != B:
        raise ValueError("label_lengths / input_lengths must have B entries")
    if B and int(np.max(np.asarray(input_lengths))) != T_max:
        raise ValueError("activations.shape[0] must equal max(input_lengths)")
    blank = A - 1 if blank is None else int(blank)
    dev = activations.device
    if costs is None:
        costs = torch.empty(B, dtype=torch.float32, device=dev)
    if want_grad and gradients is None:
        gradients = torch.empty_like(activations)
    if not want_grad:
        gradients = None
    if workspace is None:
        workspace = _default_ws.setdefault(dev.index, Workspace(dev))
    need = workspace_size(label_lengths, input_lengths, A)
    ws_ptr, ws_bytes = workspace.get(need)
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    st = _lib.lib().ds2ctc_compute_loss_checked(
        ctypes.c_void_p(activations.data_ptr()),
        ctypes.c_void_p(gradients.data_ptr()) if gradients is not None else None,
        _iptr(labels), _iptr(ll), _iptr(il), A, B, blank, ctypes.c_void_p(costs.data_ptr()),
        ctypes.c_void_p(ws_ptr), ws_bytes, ctypes.c_void_p(stream.cuda_stream))
    _lib.check(st, "ds2ctc_compute_loss")
    return costs, gradients


def compute_ctc_loss_host(activations: np.ndarray, flat_labels, label_lengths, input_lengths,
                          blank: Optional[int] = None, want_grad: bool = True, device: int = 0,
                          gradients: Optional[np.ndarray] = None, costs: Optional[np.ndarray] = None):
    """Host buffers in, host buffers out (ds2ctc_compute_loss_host); synchronous."""
    acts = np.ascontiguousarray(activations, dtype=np.float32)
    T_max, B, A = acts.shape
    blank = A - 1 if blank is None else int(blank)
    if costs is None:
        costs = np.empty(max(B, 1), dtype=np.float32)
    if want_grad and gradients is None:
        gradients = np.empty_like(acts)
    st = _lib.lib().ds2ctc_compute_loss_host(
        ctypes.c_void_p(acts.ctypes.data),
        ctypes.c_void_p(gradients.ctypes.data) if want_grad else None,
        _iptr(_i32(flat_labels)), _iptr(_i32(label_lengths)), _iptr(_i32(input_lengths)), A, B, blank,
        ctypes.c_void_p(costs.ctypes.data), device)
    _lib.check(st, "ds2ctc_compute_loss_host")
    return costs[:B], (gradients if want_grad else None)


def ctc_loss(frame_logits, label: Sequence[int], blank: int, device: int = 0) -> CtcResult:
    """Drop-in for asr::ctc::ctc_loss_reference (ctc.cpp:171-207) on one utterance."""
    x = np.ascontiguousarray(np.asarray(frame_logits, dtype=np.float32))
    T, A = x.shape
    lab = list(int(c) for c in label)
    costs, grads = compute_ctc_loss_host(x.reshape(T, 1, A), lab, [len(lab)], [T], blank=blank, device=device)
    loss = float(costs[0])
    if np.isposinf(loss):  # infeasible (ctc.cpp:173,189-193); a NaN loss is feasible, as in the reference
        return CtcResult(False, float("inf"), np.zeros((0, 0), dtype=np.float32))
    return CtcResult(True, loss, grads.reshape(T, A))


def viterbi_workspace_size(label_lengths, input_lengths, alphabet_size: int) -> int:
    """ds2ctc_viterbi_get_workspace_size: device bytes for one alignment call."""
    ll = _i32(label_lengths)
    il = _i32(input_lengths)
    B = int(np.asarray(label_lengths).size)
    out = ctypes.c_size_t()
    _lib.check(_lib.lib().ds2ctc_viterbi_get_workspace_size(_iptr(ll), _iptr(il), alphabet_size, B,
                                                            ctypes.byref(out)),
               "ds2ctc_viterbi_get_workspace_size")
    return int(out.value)


def viterbi_align_batch(activations, flat_labels, label_lengths, input_lengths, blank: Optional[int] = None,
                        workspace: Optional[Workspace] = None, stream=None):
    """Batched forced alignment on the GPU (ds2ctc_viterbi_align).

    activations: contiguous float32 CUDA tensor [T_max, B, A]. Returns
    (alignments int32 CUDA [B, T_max] with -1 past T_b, status int32 CUDA [B]:
    0 aligned, 1 no alignment -- where the reference throws)."""
    import torch

    if not (activations.is_cuda and activations.dtype == torch.float32 and activations.is_contiguous()):
        raise ValueError("activations must be a contiguous float32 CUDA tensor [T, B, A]")
    T_max, B, A = activations.shape
    blank = A - 1 if blank is None else int(blank)
    dev = activations.device
    align = torch.empty((max(B, 1), max(T_max, 1)), dtype=torch.int32, device=dev)
    status = torch.empty(max(B, 1), dtype=torch.int32, device=dev)
    if workspace is None:
        workspace = _default_ws.setdefault(dev.index, Workspace(dev))
    ws_ptr, ws_bytes = workspace.get(viterbi_workspace_size(label_lengths, input_lengths, A))
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    st = _lib.lib().ds2ctc_viterbi_align(
        ctypes.c_void_p(activations.data_ptr()), _iptr(_i32(flat_labels)), _iptr(_i32(label_lengths)),
        _iptr(_i32(input_lengths)), A, B, blank, ctypes.c_void_p(align.data_ptr()),
        ctypes.c_void_p(status.data_ptr()), ctypes.c_void_p(ws_ptr), ws_bytes, ctypes.c_void_p(stream.cuda_stream))
    _lib.check(st, "ds2ctc_viterbi_align")
    return align[:B, :T_max], status[:B]


def viterbi_align(frame_logits, label: Sequence[int], blank: int, device: int = 0):
    """Drop-in for asr::ctc::viterbi_align (ctc.cpp:327-370) on one utterance:
    the frame symbols of the best alignment; raises ValueError where the
    reference throws (label infeasible for T, or no path of nonzero probability)."""
    import torch

    x = np.ascontiguousarray(np.asarray(frame_logits, dtype=np.float32))
    T, A = x.shape
    lab = [int(c) for c in label]
    xt = torch.from_numpy(x.reshape(T, 1, A)).to(torch.device("cuda", device))
    align, status = viterbi_align_batch(xt, lab, [len(lab)], [T], blank=blank)
    if int(status[0].item()) != 0:
        raise ValueError("viterbi_align: label infeasible for frame count or no feasible path")
    return align[0].cpu().numpy().astype(np.int64).tolist()


@dataclass
class CtcLattice:
    """asr::ctc::CtcLattice (ctc.hpp:55-60): augmented label, alpha and the
    emission-exclusive beta as (2L+1) x T fp64 matrices, log p."""

    augmented_label: list
    alpha: np.ndarray
    beta: np.ndarray
    log_prob: float


def ctc_lattice_batch(activations, flat_labels, label_lengths, input_lengths, blank: Optional[int] = None,
                      stream=None):
    """Batched lattice export on the GPU (ds2ctc_ctc_lattice). Returns
    (alpha, beta, log_prob) as fp64 CUDA tensors: alpha / beta flat over all
    utterances' row-major [2L_b+1][T_b] blocks, log_prob [B]."""
    import torch

    if not (activations.is_cuda and activations.dtype == torch.float32 and activations.is_contiguous()):
        raise ValueError("activations must be a contiguous float32 CUDA tensor [T, B, A]")
    T_max, B, A = activations.shape
    blank = A - 1 if blank is None else int(blank)
    dev = activations.device
    ll, il = _i32(label_lengths), _i32(input_lengths)
    cells, wsb = ctypes.c_size_t(), ctypes.c_size_t()
    _lib.check(_lib.lib().ds2ctc_lattice_get_sizes(_iptr(ll), _iptr(il), B, ctypes.byref(cells), ctypes.byref(wsb)),
               "ds2ctc_lattice_get_sizes")
    alpha = torch.empty(max(int(cells.value), 1), dtype=torch.float64, device=dev)
    beta = torch.empty_like(alpha)
    log_prob = torch.empty(max(B, 1), dtype=torch.float64, device=dev)
    ws = _default_ws.setdefault(dev.index, Workspace(dev))
    ws_ptr, ws_bytes = ws.get(int(wsb.value))
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    st = _lib.lib().ds2ctc_ctc_lattice(
        ctypes.c_void_p(activations.data_ptr()), _iptr(_i32(flat_labels)), _iptr(ll), _iptr(il), A, B, blank,
        ctypes.c_void_p(alpha.data_ptr()), ctypes.c_void_p(beta.data_ptr()), ctypes.c_void_p(log_prob.data_ptr()),
        ctypes.c_void_p(ws_ptr), ws_bytes, ctypes.c_void_p(stream.cuda_stream))
    _lib.check(st, "ds2ctc_ctc_lattice")
    return alpha[:int(cells.value)], beta[:int(cells.value)], log_prob[:B]


def ctc_lattice(frame_logits, label: Sequence[int], blank: int, device: int = 0) -> CtcLattice:
    """Drop-in for asr::ctc::ctc_lattice (ctc.cpp:145-169) on one utterance."""
    import torch

    x = np.ascontiguousarray(np.asarray(frame_logits, dtype=np.float32))
    T, A = x.shape
    lab = [int(c) for c in label]
    if T < 1:
        raise ValueError("ctc: need at least one frame")
    xt = torch.from_numpy(x.reshape(T, 1, A)).to(torch.device("cuda", device))
    alpha, beta, lp = ctc_lattice_batch(xt, lab, [len(lab)], [T], blank=blank)
    S = 2 * len(lab) + 1
    aug = [blank]
    for c in lab:
        aug += [c, blank]
    return CtcLattice(aug, alpha.cpu().numpy().reshape(S, T), beta.cpu().numpy().reshape(S, T), float(lp[0].item()))


def dump_lattice_tsv(lat: CtcLattice, out) -> None:
    """dump_lattice_tsv (ctc.cpp:372-383): for "alpha" then "beta", a header
    "# <name> (<rows> x <cols>)" and one line per augmented position -- its
    symbol, then the row's values tab-separated in C++ default stream format
    (6 significant digits, "%g")."""
    for name, m in (("alpha", lat.alpha), ("beta", lat.beta)):
        m = np.asarray(m)
        out.write(f"# {name} ({m.shape[0]} x {m.shape[1]})\n")
        for s in range(m.shape[0]):
            out.write(str(int(lat.augmented_label[s])) + "".join("\t" + format(float(v), "g") for v in m[s]) + "\n")


def fc_backward(dlogits, x, w, dw=None, db=None, dx=None, want_dx: bool = True, stream=None,
                workspace: Optional[Workspace] = None):
    """The output layer's backward pass on the CTC gradient, on the device
    (ds2ctc_fc_backward; FullyConnectedLayer::backward, nn.cpp:874-899):
    db += sum_rows dlogits, dw += dlogits^T x, dx = dlogits w.

    dlogits: float32 CUDA [T, B, A] (the compute_ctc_loss gradients), x: float32
    CUDA [T, B, H], w: float32 CUDA [A, H]. dw [A, H] / db [A] accumulate (zeros
    when not given). Returns (dw, db, dx or None); asynchronous on `stream`."""
    import torch

    for t in (dlogits, x, w):
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
            raise ValueError("dlogits, x, w must be contiguous float32 CUDA tensors")
    T, B, A = dlogits.shape
    H = x.shape[-1]
    if x.shape[:2] != (T, B) or tuple(w.shape) != (A, H):
        raise ValueError("shapes: dlogits [T,B,A], x [T,B,H], w [A,H]")
    dev = dlogits.device
    dw = torch.zeros((A, H), dtype=torch.float32, device=dev) if dw is None else dw
    db = torch.zeros(A, dtype=torch.float32, device=dev) if db is None else db
    if want_dx and dx is None:
        dx = torch.empty((T, B, H), dtype=torch.float32, device=dev)
    rows = T * B
    out = ctypes.c_size_t()
    _lib.check(_lib.lib().ds2ctc_fc_backward_workspace_size(rows, A, H, ctypes.byref(out)),
               "ds2ctc_fc_backward_workspace_size")
    if workspace is None:
        workspace = _default_ws.setdefault(("fc", dev.index), Workspace(dev))
    ws_ptr, ws_bytes = workspace.get(int(out.value))
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    st = _lib.lib().ds2ctc_fc_backward(
        ctypes.c_void_p(dlogits.data_ptr()), ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(w.data_ptr()),
        ctypes.c_void_p(dw.data_ptr()), ctypes.c_void_p(db.data_ptr()),
        ctypes.c_void_p(dx.data_ptr()) if want_dx else None, rows, A, H, ctypes.c_void_p(ws_ptr), ws_bytes,
        ctypes.c_void_p(stream.cuda_stream))
    _lib.check(st, "ds2ctc_fc_backward")
    return dw, db, (dx if want_dx else None)
