"""ctypes binding of libds2ctc.so (the C-ABI in include/ds2ctc.h).

This is the binding a Python caller of the reference's CTC would add; there
is no fallback: if the in-tree library is missing or cannot be loaded, every
call raises (the product never silently runs anything on the CPU).
"""
from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
# DS2CTC_LIB: debug experiments only (a variant build of the same sources, see build.build_variant)
LIB_PATH = os.environ.get("DS2CTC_LIB") or os.path.join(PKG, "libds2ctc.so")

STATUS = {
    0: "SUCCESS",
    1: "INVALID_VALUE",
    2: "EXECUTION_FAILED",
    3: "MEMOPS_FAILED",
    4: "UNSUPPORTED",
}

# Every symbol include/ds2ctc.h declares (tests check the .so exports them all).
EXPORTS = (
    "ds2ctc_status_string",
    "ds2ctc_version",
    "ds2ctc_get_workspace_size",
    "ds2ctc_compute_loss",
    "ds2ctc_compute_loss_checked",
    "ds2ctc_compute_loss_host",
    "ds2ctc_loss_sum",
    "ds2ctc_mailbox_alloc",
    "ds2ctc_mailbox_open",
    "ds2ctc_mailbox_close",
    "ds2ctc_loss_sum_allreduce",
    "ds2ctc_exchange_size",
    "ds2ctc_exchange_alloc",
    "ds2ctc_vec_allreduce",
    "ds2ctc_reduce_fault",
    "ds2ctc_fc_backward_workspace_size",
    "ds2ctc_fc_backward",
    "ds2ctc_viterbi_get_workspace_size",
    "ds2ctc_viterbi_align",
    "ds2ctc_lattice_get_sizes",
    "ds2ctc_ctc_lattice",
    "ds2ctc_viterbi_align_host",
    "ds2ctc_ctc_lattice_host",
    "ds2ctc_profile_enable",
    "ds2ctc_profile_read",
    "ds2ctc_debug_watchdog",
    "ds2ctc_sortagrad_order",
    "ds2ctc_rank_slice",
    "ds2ctc_shard_lpt",
)


class Ds2CtcError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: ds2ctc status {status} ({STATUS.get(status, '?')})")


_lock = threading.Lock()
_lib = None

_p = ctypes.c_void_p
_ip = ctypes.POINTER(ctypes.c_int)
_i64p = ctypes.POINTER(ctypes.c_int64)
_dp = ctypes.POINTER(ctypes.c_double)
_szp = ctypes.POINTER(ctypes.c_size_t)


class _missing:
    def __init__(self, name):
        self.name = name

    def __call__(self, *a):
        raise RuntimeError(f"{LIB_PATH} (DS2CTC_LIB variant) does not export {self.name}")


def lib():
    """Loads the in-tree libds2ctc.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1512_02595_b200.build` "
                                  "(there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            if os.environ.get("DS2CTC_LIB"):
                # a debug variant (e.g. an older build for an A/B) may predate some
                # entry points: give those a stub that fails loudly if called
                for name in EXPORTS:
                    try:
                        getattr(L, name)
                    except AttributeError:
                        setattr(L, name, _missing(name))
            L.ds2ctc_status_string.restype = ctypes.c_char_p
            L.ds2ctc_status_string.argtypes = [ctypes.c_int]
            L.ds2ctc_version.restype = ctypes.c_char_p
            L.ds2ctc_version.argtypes = []
            L.ds2ctc_get_workspace_size.restype = ctypes.c_int
            L.ds2ctc_get_workspace_size.argtypes = [_ip, _ip, ctypes.c_int, ctypes.c_int, _szp]
            L.ds2ctc_compute_loss.restype = ctypes.c_int
            L.ds2ctc_compute_loss.argtypes = [_p, _p, _ip, _ip, _ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _p,
                                              _p]
            L.ds2ctc_compute_loss_checked.restype = ctypes.c_int
            L.ds2ctc_compute_loss_checked.argtypes = [_p, _p, _ip, _ip, _ip, ctypes.c_int, ctypes.c_int,
                                                      ctypes.c_int, _p, _p, ctypes.c_size_t, _p]
            L.ds2ctc_compute_loss_host.restype = ctypes.c_int
            L.ds2ctc_compute_loss_host.argtypes = [_p, _p, _ip, _ip, _ip, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                                   _p, ctypes.c_int]
            L.ds2ctc_loss_sum.restype = ctypes.c_int
            L.ds2ctc_loss_sum.argtypes = [_p, ctypes.c_int, _p, _p]
            L.ds2ctc_mailbox_alloc.restype = ctypes.c_int
            L.ds2ctc_mailbox_alloc.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), _p]
            L.ds2ctc_mailbox_open.restype = ctypes.c_int
            L.ds2ctc_mailbox_open.argtypes = [_p, ctypes.POINTER(ctypes.c_void_p)]
            L.ds2ctc_mailbox_close.restype = ctypes.c_int
            L.ds2ctc_mailbox_close.argtypes = [_p, ctypes.c_int]
            L.ds2ctc_loss_sum_allreduce.restype = ctypes.c_int
            L.ds2ctc_loss_sum_allreduce.argtypes = [_p, ctypes.c_int, _p, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
                                                    ctypes.c_int, ctypes.c_ulonglong, _p]
            L.ds2ctc_fc_backward_workspace_size.restype = ctypes.c_int
            L.ds2ctc_fc_backward_workspace_size.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _szp]
            L.ds2ctc_fc_backward.restype = ctypes.c_int
            L.ds2ctc_fc_backward.argtypes = [_p, _p, _p, _p, _p, _p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p,
                                             ctypes.c_size_t, _p]
            L.ds2ctc_exchange_size.restype = ctypes.c_int
            L.ds2ctc_exchange_size.argtypes = [ctypes.c_size_t, _szp]
            L.ds2ctc_exchange_alloc.restype = ctypes.c_int
            L.ds2ctc_exchange_alloc.argtypes = [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p), _p]
            L.ds2ctc_vec_allreduce.restype = ctypes.c_int
            L.ds2ctc_vec_allreduce.argtypes = [_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
                                               ctypes.c_int, ctypes.c_ulonglong, _p]
            L.ds2ctc_reduce_fault.restype = ctypes.c_int
            L.ds2ctc_reduce_fault.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
            L.ds2ctc_viterbi_get_workspace_size.restype = ctypes.c_int
            L.ds2ctc_viterbi_get_workspace_size.argtypes = [_ip, _ip, ctypes.c_int, ctypes.c_int, _szp]
            L.ds2ctc_lattice_get_sizes.restype = ctypes.c_int
            L.ds2ctc_lattice_get_sizes.argtypes = [_ip, _ip, ctypes.c_int, _szp, _szp]
            L.ds2ctc_ctc_lattice.restype = ctypes.c_int
            L.ds2ctc_ctc_lattice.argtypes = [_p, _ip, _ip, _ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _p, _p,
                                             _p, ctypes.c_size_t, _p]
            L.ds2ctc_viterbi_align_host.restype = ctypes.c_int
            L.ds2ctc_viterbi_align_host.argtypes = [_p, _ip, _ip, _ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p,
                                                    _p, ctypes.c_int]
            L.ds2ctc_ctc_lattice_host.restype = ctypes.c_int
            L.ds2ctc_ctc_lattice_host.argtypes = [_p, _ip, _ip, _ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _p,
                                                  _p, ctypes.c_int]
            L.ds2ctc_viterbi_align.restype = ctypes.c_int
            L.ds2ctc_viterbi_align.argtypes = [_p, _ip, _ip, _ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, _p, _p,
                                               _p, ctypes.c_size_t, _p]
            L.ds2ctc_profile_enable.restype = ctypes.c_int
            L.ds2ctc_profile_enable.argtypes = [ctypes.c_int]
            L.ds2ctc_profile_read.restype = ctypes.c_int
            L.ds2ctc_profile_read.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
            L.ds2ctc_debug_watchdog.restype = ctypes.c_int
            L.ds2ctc_debug_watchdog.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
            L.ds2ctc_sortagrad_order.restype = ctypes.c_int
            L.ds2ctc_sortagrad_order.argtypes = [_ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                                 ctypes.c_int, _i64p]
            L.ds2ctc_rank_slice.restype = ctypes.c_int
            L.ds2ctc_rank_slice.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _ip, _ip]
            L.ds2ctc_shard_lpt.restype = ctypes.c_int
            L.ds2ctc_shard_lpt.argtypes = [_ip, _ip, ctypes.c_int, ctypes.c_int, ctypes.c_int, _ip, _dp]
            _lib = L
    return _lib


def watchdog():
    """(kind, block, warp, step) of the first bounded wait that gave up since the last call, or None."""
    out = (ctypes.c_ulonglong * 4)()
    check(lib().ds2ctc_debug_watchdog(out), "ds2ctc_debug_watchdog")
    return None if out[0] == 0 else tuple(int(v) for v in out)


def reduce_fault():
    """The step (seq) of the first fused all-reduce whose peer wait timed out since the last call, or None."""
    out = ctypes.c_ulonglong(0)
    check(lib().ds2ctc_reduce_fault(ctypes.byref(out)), "ds2ctc_reduce_fault")
    return None if out.value == 0 else int(out.value)


def check(status: int, where: str) -> None:
    if status != 0:
        raise Ds2CtcError(status, where)
