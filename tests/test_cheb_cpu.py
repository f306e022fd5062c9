"""Host logic of the sparse-A path (no GPU): the Chebyshev coefficients e^{-gamma} I_k(gamma) of
e^{gamma (x - 1)} on [-1, 1] that the library computes by Miller's backward recurrence
(dme_cheb_coeffs, csrc/cheb.cu), pinned against
  * scipy.special.ive (an independent Bessel implementation),
  * the closed forms of the expansion at x = 1, 0, -1 (T_k(1) = 1, T_k(0) = cos(k pi / 2),
    T_k(-1) = (-1)^k): 1, e^{-gamma}, e^{-2 gamma},
  * the degree rule: the tail beyond K is <= tol and the tail beyond K - 1 is not.
"""
import numpy as np
import pytest
import scipy.special as sp

import paper_1805_08990_b200 as dme

GAMMAS = [0.0, 1e-8, 0.3, 2.7, 25.0, 204.0, 408.0, 1500.0]


@pytest.mark.parametrize("gamma", GAMMAS)
def test_coeffs_vs_scipy_ive(gamma):
    c = dme.cheb_coeffs(gamma)
    ref = sp.ive(np.arange(c.size), gamma)
    big = ref > 1e-250
    assert np.all(np.abs(c[big] - ref[big]) <= 1e-12 * ref[big])


@pytest.mark.parametrize("gamma", GAMMAS)
def test_expansion_closed_forms(gamma):
    c = dme.cheb_coeffs(gamma)
    k = np.arange(c.size)
    w = np.where(k == 0, 1.0, 2.0) * c
    assert abs(w.sum() - 1.0) <= 1e-14                                     # x = 1
    assert abs((w * np.cos(k * np.pi / 2)).sum() - np.exp(-gamma)) <= 1e-14   # x = 0
    assert abs((w * (-1.0) ** k).sum() - np.exp(-2 * gamma)) <= 1e-14          # x = -1


@pytest.mark.parametrize("gamma", [0.3, 25.0, 204.0])
@pytest.mark.parametrize("tol", [1e-8, 2.0 ** -56])
def test_degree_rule(gamma, tol):
    c = dme.cheb_coeffs(gamma, tol)
    K = c.size - 1
    tail = lambda k0: 2 * sp.ive(np.arange(k0 + 1, k0 + 3000), gamma).sum()
    assert tail(K) <= tol * (1 + 1e-6)
    assert tail(K - 1) > tol * (1 - 1e-6)


def test_degree_growth_is_sublinear():
    # the reason for a Chebyshev (or Leja) polynomial on the heat spectrum: degree ~ sqrt(gamma)
    K = [dme.cheb_coeffs(g).size - 1 for g in (100.0, 400.0, 1600.0)]
    assert K[1] < 2.2 * K[0] and K[2] < 2.2 * K[1]  # (linear growth would be 4x)


def _workspace(A_dense=None, csr=None, n=None, **kw):
    """dme_workspace_size through the C ABI (host only: plans the buffers, no device)."""
    import ctypes
    from paper_1805_08990_b200 import _lib, _Options, _Problem, _ptr
    pr = _Problem(n=n)
    keep = []
    if A_dense is not None:
        a = np.ascontiguousarray(A_dense, dtype=np.float64)
        keep.append(a)
        pr.A = _ptr(a)
    if csr is not None:
        rp = np.ascontiguousarray(csr.indptr, dtype=np.int64)
        ci = np.ascontiguousarray(csr.indices, dtype=np.int32)
        vv = np.ascontiguousarray(csr.data, dtype=np.float64)
        keep += [rp, ci, vv]
        pr.A_nnz = vv.size
        pr.A_rowptr = rp.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        pr.A_colind = ci.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        pr.A_values = _ptr(vv)
    opt = _Options()
    _lib.dme_default_options(ctypes.byref(opt))
    opt.rank_cap = 64
    for key, val in kw.items():
        setattr(opt, key, val)
    nbytes = ctypes.c_size_t(0)
    code = _lib.dme_workspace_size(ctypes.byref(pr), ctypes.byref(opt), ctypes.byref(nbytes))
    return code, nbytes.value


def test_sparse_workspace_has_no_dense_matrices():
    """The sparse-A plan holds no n x n buffer (no E, no Padé scratch): at n = 10^4 it is a few
    hundred MB against ~8 GB for the dense path."""
    import scipy.sparse as sps
    from workloads import make_config
    prob = make_config(5)
    code_d, dense = _workspace(A_dense=prob.A, n=prob.n)
    code_s, sparse = _workspace(csr=sps.csr_matrix(prob.A), n=prob.n)
    assert code_d == 0 and code_s == 0
    assert dense > 8 * prob.n ** 2 * 8  # E_{h/2}, E_h, Padé scratch
    assert sparse < 0.05 * dense


def test_sparse_plan_errors():
    import scipy.sparse as sps
    from workloads import make_config
    prob = make_config(3, nx=8)  # nonsymmetric convection-diffusion: the Taylor route (accepted)
    assert _workspace(csr=sps.csr_matrix(prob.A), n=prob.n)[0] == 0
    # symmetric but not diagonally dominant (-L^2): the Chebyshev accuracy gate rejects it
    from workloads import heat2d_matrix
    L = heat2d_matrix(12)
    assert _workspace(csr=sps.csr_matrix(-(L @ L)), n=L.shape[0], h=2e-4)[0] == 3
    A = sps.csr_matrix(make_config(5, nx=8).A)
    bad = A.copy()
    bad.indices = bad.indices.copy()
    bad.indices[0] = -1
    assert _workspace(csr=bad, n=A.shape[0])[0] == 1
    bad = A.copy()
    bad.data = bad.data.copy()
    bad.data[5] = np.nan
    assert _workspace(csr=bad, n=A.shape[0])[0] == 1
