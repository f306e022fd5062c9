"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol declared
in include/dme.h (no compute calls: there is no GPU here), and the host-side logic that needs
no device (status strings, default options, argument validation paths) behaves."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "dme.h")).read()
    return sorted(set(re.findall(r"\b(dme_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported():
    import paper_1805_08990_b200 as dme
    lib = ctypes.CDLL(dme.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(dme.EXPORTED) == declared


def test_status_strings_and_defaults():
    import paper_1805_08990_b200 as dme
    lib = dme._lib
    for code, text in dme.STATUS.items():
        assert lib.dme_status_string(code).decode() == text
    o = dme._Options()
    lib.dme_default_options(ctypes.byref(o))
    assert o.trunc_tol == 1e-16 and o.quad_nodes == 14 and o.quad_subpanels == 1 and o.world_size == 1


def test_workspace_size_host_only():
    import numpy as np
    import paper_1805_08990_b200 as dme
    n = 100
    A = np.zeros((n, n))
    pr = dme._Problem(n=n, A=A.ctypes.data_as(dme._dp), p=0, C=None, m=0, B=None, R=None, S=None,
                      r0=0, L0=None, D0=None)
    o = dme._Options()
    dme._lib.dme_default_options(ctypes.byref(o))
    nb = ctypes.c_size_t(0)
    assert dme._lib.dme_workspace_size(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(nb)) == 0
    assert nb.value > 12 * n * n * 8
    pr.n = 0
    assert dme._lib.dme_workspace_size(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(nb)) == 1
    assert b"positive" in dme._lib.dme_last_error()


def test_init_rejects_bad_input_without_device():
    # host-side validation happens before any CUDA call (A and S, the n x n inputs, are checked for
    # finiteness on the device after the upload: see tests/test_gpu_edge.py::test_errors)
    import numpy as np
    import paper_1805_08990_b200 as dme
    n = 8
    A = np.eye(n)
    pr = dme._Problem(n=n, A=A.ctypes.data_as(dme._dp), p=0, C=None, m=0, B=None, R=None, S=None,
                      r0=0, L0=None, D0=None)
    o = dme._Options()
    dme._lib.dme_default_options(ctypes.byref(o))
    ctx = ctypes.c_void_p()
    o.h = -1.0
    assert dme._lib.dme_dle_init(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(ctx)) == 1
    o.h = 0.01
    C = np.full((1, n), np.nan)
    pr.p, pr.C = 1, C.ctypes.data_as(dme._dp)
    assert dme._lib.dme_dle_init(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(ctx)) == 1
    pr.p, pr.C = 0, None
    R = np.array([[-1.0]])
    B = np.ones((n, 1))
    pr.m, pr.B, pr.R = 1, B.ctypes.data_as(dme._dp), R.ctypes.data_as(dme._dp)
    assert dme._lib.dme_dre_init(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(ctx)) == 1
    assert b"positive definite" in dme._lib.dme_last_error()
    assert dme._lib.dme_dle_init(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(ctx)) == 1
    assert dme._lib.dme_split_step(None, 0, 0, 1) == 1


def _host_problem(n):
    import numpy as np
    import paper_1805_08990_b200 as dme
    A = -2.0 * np.eye(n)
    keep = [A]
    pr = dme._Problem(n=n, A=A.ctypes.data_as(dme._dp), p=0, C=None, m=0, B=None, R=None, S=None,
                      r0=0, L0=None, D0=None)
    o = dme._Options()
    dme._lib.dme_default_options(ctypes.byref(o))
    return pr, o, keep


def test_csr_s_validation_host_only():
    """The CSR form of S (T4 by sparse products) is validated on the host before any device work."""
    import numpy as np
    import paper_1805_08990_b200 as dme
    n = 6
    pr, o, keep = _host_problem(n)
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int32)
    vv = np.full(n, 0.5)
    keep += [rp, ci, vv]
    pr.S_nnz = n
    pr.S_rowptr = rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    pr.S_colind = ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    pr.S_values = vv.ctypes.data_as(dme._dp)
    nb = ctypes.c_size_t(0)
    assert dme._lib.dme_workspace_size(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(nb)) == 0
    assert nb.value > 0
    # (the init validates the host inputs before any device call: DME_ERR_INVALID here, no GPU)
    o.h = 0.01
    ctx = ctypes.c_void_p()
    ci[2] = n + 3                      # column index out of range
    assert dme._lib.dme_dle_init(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(ctx)) == 1
    assert b"CSR S" in dme._lib.dme_last_error()
    ci[2] = 2
    vv[1] = np.inf                     # non-finite value
    assert dme._lib.dme_dle_init(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(ctx)) == 1
    vv[1] = 0.5
    rp[3] = 1                          # decreasing row pointers
    assert dme._lib.dme_dle_init(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(ctx)) == 1


def test_virtual_world_plan_host_only():
    """options.virtual_world = G plans the G-shard staging blocks and digit images on one GPU;
    out-of-range values are rejected."""
    import paper_1805_08990_b200 as dme
    n = 200
    pr, o, keep = _host_problem(n)
    nb1, nbg = ctypes.c_size_t(0), ctypes.c_size_t(0)
    assert dme._lib.dme_workspace_size(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(nb1)) == 0
    o.virtual_world = 4
    assert dme._lib.dme_workspace_size(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(nbg)) == 0
    assert nbg.value > nb1.value       # + the 4 x n_loc x 224 staging blocks
    o.virtual_world = 65
    o.h = 0.01
    ctx = ctypes.c_void_p()
    assert dme._lib.dme_dle_init(ctypes.byref(pr), ctypes.byref(o), ctypes.byref(ctx)) == 1
    assert b"virtual_world" in dme._lib.dme_last_error()


def test_compression_option_values():
    import paper_1805_08990_b200 as dme
    o = dme._Options()
    dme._lib.dme_default_options(ctypes.byref(o))
    assert o.compression == 0 and o.virtual_world == 0      # refined compression, no virtual shards
