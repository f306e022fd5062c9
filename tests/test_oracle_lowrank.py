"""Pins for oracle.lowrank (P10 in DESIGN.md): SPEC.md compress/concat examples,
reconstruction bound, idempotence, rank monotonicity, and the QR-stacked parity metric
against a dense Frobenius norm."""
import numpy as np
import pytest

from oracle import lowrank


def test_concat_example():
    # a=(L=[1;0],D=[2]), b=(L=[0;1],D=[3]), w=0.5 -> diag(2, 1.5)
    L, D = lowrank.concat(np.array([[1.0], [0.0]]), np.array([[2.0]]),
                          np.array([[0.0], [1.0]]), np.array([[3.0]]), 0.5)
    assert np.allclose(lowrank.to_dense(L, D), np.diag([2.0, 1.5]))


def test_compress_duplicated_columns_rank1():
    # L = [v, v], D = I -> rank 1 reconstructing 2 v v^T
    v = np.arange(1.0, 7.0)[:, None]
    L, D = lowrank.column_compression(np.hstack([v, v]), np.eye(2), 1e-12)
    assert L.shape[1] == 1
    assert np.allclose(lowrank.to_dense(L, D), 2 * v @ v.T, rtol=1e-14, atol=1e-13)


def test_compress_small_eigenvalue_dropped():
    # L = I3, D = diag(1, 1e-20, 1), tol 1e-12 -> rank 2
    L, D = lowrank.column_compression(np.eye(3), np.diag([1.0, 1e-20, 1.0]), 1e-12)
    assert L.shape[1] == 2


@pytest.mark.parametrize("seed", range(5))
def test_compress_reconstruction_and_orthonormal(seed):
    rng = np.random.default_rng(seed)
    n, r = 50, 20
    G = rng.standard_normal((n, 8))
    L = np.hstack([G, G @ rng.standard_normal((8, r - 8))])   # numerical rank 8
    D = np.diag(rng.uniform(0.1, 2.0, r))
    P = lowrank.to_dense(L, D)
    L2, D2 = lowrank.column_compression(L, D, 1e-10)
    assert L2.shape[1] == 8
    assert np.allclose(L2.T @ L2, np.eye(8), atol=1e-13)
    assert np.allclose(D2, np.diag(np.diag(D2)))
    assert np.linalg.norm(lowrank.to_dense(L2, D2) - P) <= 1e-10 * np.linalg.norm(P)
    # idempotent
    L3, D3 = lowrank.column_compression(L2, D2, 1e-10)
    assert L3.shape[1] == L2.shape[1]


def test_compress_indefinite_signature_kept():
    rng = np.random.default_rng(7)
    L = rng.standard_normal((30, 6))
    D = np.diag([3.0, -2.0, 1.0, -0.5, 0.25, 2.0])
    L2, D2 = lowrank.column_compression(L, D, 1e-14)
    assert np.sum(np.diag(D2) < 0) == 2
    assert np.allclose(lowrank.to_dense(L2, D2), lowrank.to_dense(L, D), atol=1e-12)


def test_rank_monotone_and_cap():
    rng = np.random.default_rng(3)
    L = rng.standard_normal((40, 12)) * np.logspace(0, -11, 12)[None, :]
    ranks = [lowrank.column_compression(L, np.eye(12), t)[0].shape[1] for t in (1e-16, 1e-12, 1e-8, 1e-4)]
    assert ranks == sorted(ranks, reverse=True)
    assert lowrank.column_compression(L, np.eye(12), 1e-16, rank_cap=5)[0].shape[1] == 5
    # rank cap keeps the best rank-5 approximation: error = 6th eigenvalue
    L5, D5 = lowrank.column_compression(L, np.eye(12), 1e-16, rank_cap=5)
    P = L @ L.T
    ev = np.sort(np.linalg.eigvalsh(P))[::-1]
    assert np.isclose(np.linalg.norm(P - lowrank.to_dense(L5, D5), 2), ev[5], rtol=1e-6)


def test_rank0():
    L, D = lowrank.column_compression(np.zeros((5, 0)), np.zeros((0, 0)))
    assert L.shape == (5, 0)
    L, D = lowrank.column_compression(np.zeros((5, 2)), np.eye(2))
    assert L.shape == (5, 0)


@pytest.mark.parametrize("eps", [1e-4, 1e-8, 1e-12])
def test_rel_diff_matches_dense(eps):
    # the metric must resolve small relative differences exactly
    rng = np.random.default_rng(11)
    n = 60
    L1 = rng.standard_normal((n, 7))
    D1 = np.diag(rng.uniform(0.5, 1.5, 7))
    L2 = L1 + eps * rng.standard_normal((n, 7))
    d = lowrank.rel_diff(L2, D1, L1, D1)
    P1, P2 = lowrank.to_dense(L1, D1), lowrank.to_dense(L2, D1)
    ref = np.linalg.norm(P2 - P1) / np.linalg.norm(P1)
    assert abs(d - ref) <= 1e-3 * ref + 1e-15
