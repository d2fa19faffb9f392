"""C-ABI checks that need no GPU: the in-tree library loads, exports every
symbol include/ds2ctc.h declares, sizes workspaces, and rejects bad input
with the documented status codes before touching CUDA."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1512_02595_b200 import _lib, ctc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    with open(os.path.join(ROOT, "include", "ds2ctc.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(ds2ctc_[a-z_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    declared = header_functions()
    assert declared, "no declarations parsed"
    assert set(declared) == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), f"{name} not exported"


def test_version_and_status_strings():
    lib = _lib.lib()
    assert b"sm_100a" in lib.ds2ctc_version()
    assert lib.ds2ctc_status_string(0) == b"no error"
    assert lib.ds2ctc_status_string(1) == b"invalid value"


def test_workspace_size_monotone():
    a = ctc.workspace_size([40] * 16, [150] * 16, 29)
    b = ctc.workspace_size([150] * 64, [700] * 64, 29)
    c = ctc.workspace_size([60] * 64, [350] * 64, 6000)
    assert 0 < a < b
    # half-lattice store: per frame fp32 deltas (2L+1 -> mult. of 4) + per-warp offsets
    assert b >= 64 * (304 + 4) * 701 * 4
    # the split (large-alphabet) path also keeps compact occupancy rows and per-frame lse
    assert c >= 64 * (124 + 4) * 351 * 4 + 64 * 350 * 61 * 4 + 64 * 350 * 8
    assert ctc.workspace_size([], [], 29) == 0


def _call(acts_ptr=None, A=29, B=1, blank=28, labels=(1,), ll=(1,), il=(3,), costs_ptr=1, ws=256):
    lib = _lib.lib()
    P = ctypes.POINTER(ctypes.c_int)
    lab = np.asarray(labels if len(labels) else [0], dtype=np.int32)
    lla = np.asarray(ll if len(ll) else [0], dtype=np.int32)
    ila = np.asarray(il if len(il) else [0], dtype=np.int32)
    return lib.ds2ctc_compute_loss(acts_ptr, None, lab.ctypes.data_as(P), lla.ctypes.data_as(P),
                                   ila.ctypes.data_as(P), A, B, blank, costs_ptr, ws, None)


def test_invalid_values_rejected_without_gpu():
    assert _call(A=1, blank=0) == 1                      # alphabet must include blank + 1 symbol
    assert _call(blank=29) == 1                          # blank out of range
    assert _call(blank=-1) == 1
    assert _call(labels=(29,)) == 1                      # label out of range (reference UB; rejected)
    assert _call(labels=(-2,)) == 1
    assert _call(ll=(-1,)) == 1                          # negative lengths
    assert _call(il=(-3,)) == 1
    assert _call(B=-1) == 1
    assert _call(acts_ptr=1, costs_ptr=None) == 1        # costs required
    assert _call(acts_ptr=1, ws=None) == 1               # workspace required
    assert _call(acts_ptr=1, ws=257) == 1                # 256-byte alignment


def test_too_many_states_unsupported():
    L = 2048  # 2L+1 = 4097 > DS2CTC_MAX_STATES
    assert _call(labels=tuple([1] * L), ll=(L,), il=(5000,)) == 4
    out = ctypes.c_size_t()
    P = ctypes.POINTER(ctypes.c_int)
    ll = np.asarray([L], dtype=np.int32)
    il = np.asarray([5000], dtype=np.int32)
    assert _lib.lib().ds2ctc_get_workspace_size(ll.ctypes.data_as(P), il.ctypes.data_as(P), 29, 1,
                                                ctypes.byref(out)) == 4


def test_empty_minibatch_is_noop():
    # an empty data-parallel shard (trainer.cpp:141-155) must be a valid no-op
    assert _call(B=0, labels=(), ll=(), il=()) == 0


def test_checked_variant_rejects_small_workspace():
    lib = _lib.lib()
    P = ctypes.POINTER(ctypes.c_int)
    lab = np.asarray([1, 2], dtype=np.int32)
    ll = np.asarray([2], dtype=np.int32)
    il = np.asarray([10], dtype=np.int32)
    need = ctc.workspace_size(ll, il, 29)
    st = lib.ds2ctc_compute_loss_checked(1, None, lab.ctypes.data_as(P), ll.ctypes.data_as(P), il.ctypes.data_as(P),
                                         29, 1, 28, 1, 256, need - 1, None)
    assert st == 1


def test_missing_library_fails_loudly(monkeypatch):
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libds2ctc.so")
    with pytest.raises(ImportError):
        _lib.lib()


def test_alignment_and_lattice_entry_points_validate_without_gpu():
    lib = _lib.lib()
    P = ctypes.POINTER(ctypes.c_int)
    ll = np.array([2, 3], dtype=np.int32)
    il = np.array([5, 7], dtype=np.int32)
    out = ctypes.c_size_t()
    assert lib.ds2ctc_viterbi_get_workspace_size(ll.ctypes.data_as(P), il.ctypes.data_as(P), 6, 2,
                                                 ctypes.byref(out)) == 0
    assert out.value >= 5 * 5 + 7 * 7  # one backpointer byte per lattice cell
    cells, wsb = ctypes.c_size_t(), ctypes.c_size_t()
    assert lib.ds2ctc_lattice_get_sizes(ll.ctypes.data_as(P), il.ctypes.data_as(P), 2, ctypes.byref(cells),
                                        ctypes.byref(wsb)) == 0
    assert cells.value == 5 * 5 + 7 * 7
    bad = np.array([-1, 3], dtype=np.int32)
    assert lib.ds2ctc_viterbi_get_workspace_size(bad.ctypes.data_as(P), il.ctypes.data_as(P), 6, 2,
                                                 ctypes.byref(out)) == 1
    # label outside [0, A) and T = 0 for the lattice are rejected before any CUDA call
    lab = np.array([0, 9, 1, 2, 3], dtype=np.int32)
    assert lib.ds2ctc_viterbi_align(None, lab.ctypes.data_as(P), ll.ctypes.data_as(P), il.ctypes.data_as(P), 6, 2, 5,
                                    1, 1, 256, 1 << 20, None) == 1
    il0 = np.array([0, 7], dtype=np.int32)
    lab_ok = np.array([0, 1, 1, 2, 3], dtype=np.int32)
    assert lib.ds2ctc_ctc_lattice(None, lab_ok.ctypes.data_as(P), ll.ctypes.data_as(P), il0.ctypes.data_as(P), 6, 2,
                                  5, 1, 1, 1, 256, 1 << 20, None) == 1
    # an empty minibatch is a valid no-op (empty data-parallel shard)
    assert lib.ds2ctc_viterbi_align(None, None, None, None, 6, 0, 5, None, None, None, 0, None) == 0


def test_fc_backward_entry_points_validate_without_gpu():
    # the output-FC backward (nn.cpp:874-899) validates before touching the device
    import ctypes

    from paper_1512_02595_b200 import _lib

    L = _lib.lib()
    out = ctypes.c_size_t()
    # A % 4 != 0: the gradient rows are re-pitched (rows x 32 floats) + W^T (H x 32)
    assert L.ds2ctc_fc_backward_workspace_size(1000, 29, 256, ctypes.byref(out)) == 0
    assert out.value >= 4 * (1000 * 32 + 256 * 32)
    assert L.ds2ctc_fc_backward_workspace_size(1000, 6000, 256, ctypes.byref(out)) == 0
    assert out.value == 4 * 256 * 6000  # aligned gradient rows: W^T only
    assert L.ds2ctc_fc_backward_workspace_size(-1, 29, 256, ctypes.byref(out)) == 1
    p = ctypes.c_void_p(256)  # never dereferenced: every case below fails validation or is a no-op
    # rows == 0 is a no-op (an empty shard)
    assert L.ds2ctc_fc_backward(p, p, p, p, p, p, 0, 29, 256, None, 0, None) == 0
    # in_dim % 4 != 0 cannot be tiled by TMA: unsupported
    assert L.ds2ctc_fc_backward(p, p, p, p, p, p, 10, 29, 250, None, 0, None) == 4
    # misaligned buffers and a short workspace are invalid values
    assert L.ds2ctc_fc_backward(ctypes.c_void_p(258), p, p, p, p, p, 10, 29, 256, None, 0, None) == 1
    assert L.ds2ctc_fc_backward(p, p, p, p, p, p, 10, 29, 256, p, 16, None) == 1
    # a NULL gradient with any requested output
    assert L.ds2ctc_fc_backward(None, p, p, p, p, p, 10, 29, 256, p, 1 << 20, None) == 1


def test_dump_lattice_tsv_format():
    # dump_lattice_tsv (ctc.cpp:372-383) as test_ctc.cpp:277-284 checks it, on a
    # hand-made lattice (no GPU): headers, one line per augmented position,
    # the symbol then tab-separated values in C++ default stream format
    import io

    import numpy as np

    from paper_1512_02595_b200 import ctc

    a = np.array([[-1.0986122886681098, -2.1972245773362196, -np.inf],
                  [-1.0986122886681098, -1.504077396776274, -2.1972245773362196],
                  [-np.inf, -2.1972245773362196, 1e-05]])
    lat = ctc.CtcLattice([2, 0, 2], a, a * 2, -1.0)
    buf = io.StringIO()
    ctc.dump_lattice_tsv(lat, buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == "# alpha (3 x 3)" and lines[4] == "# beta (3 x 3)" and len(lines) == 8
    assert lines[1] == "2\t-1.09861\t-2.19722\t-inf"
    assert lines[3] == "2\t-inf\t-2.19722\t1e-05"
    assert lines[5].split("\t")[0] == "2" and lines[6].split("\t")[0] == "0"
