"""Pins for the objective, spectral initialisation
 and metrics."""
import itertools

import numpy as np
import pytest

from oracle import instance as inst
from oracle import metrics as mt
from oracle import nsrgs as ns


def _haar(rng, d):
    Q, R = np.linalg.qr(rng.standard_normal((d, d)))
    return Q * np.sign(np.diag(R))


# ---------------------------------------------------------------- objective
def test_objective_hand_example():
    # d = 1, n = 2, A_12 = A_21 = 1, X = (1; -1): 1/2*4 + 1/2*4 = 4
    A = np.array([[0.0, 1.0], [1.0, 0.0]])
    X = np.array([1.0, -1.0]).reshape(2, 1, 1)
    assert ns.objective(A, X) == 4.0
    assert ns.objective_expanded(A, X) == 4.0


def test_objective_expansion_and_invariance():
    n, d, sigma = 25, 3, 1.1
    Z = inst.ground_truth(9, n, d)
    A = inst.measurement_matrix(9, Z, sigma)
    rng = np.random.default_rng(0)
    X = Z + 0.1 * rng.standard_normal(Z.shape)           # off-manifold too
    f1, f2 = ns.objective(A, X), ns.objective_expanded(A, X)
    assert abs(f1 - f2) <= 1e-12 * f1
    Q = _haar(rng, d)
    assert abs(ns.objective(A, X @ Q) - f1) <= 1e-12 * f1
    A0 = inst.measurement_matrix(9, Z, 0.0, dtype=np.float64)
    assert ns.objective(A0, Z) < 1e-25


# ---------------------------------------------------------------- spectral init
def test_noiseless_spectrum_closed_form():
    # sigma = 0: A = ZZ^T - I has eigenvalues n-1 (mult d) and -1 (mult nd-d).
    n, d = 12, 3
    Z = inst.ground_truth(1, n, d)
    A = inst.measurement_matrix(1, Z, 0.0, dtype=np.float64)
    w = np.sort(np.linalg.eigvalsh(A))
    assert np.allclose(w[-d:], n - 1, atol=1e-12)
    assert np.allclose(w[:-d], -1.0, atol=1e-12)


@pytest.mark.parametrize("method", ["eigh", "subspace"])
def test_noiseless_exact_recovery(method):
    n, d = 50, 3
    Z = inst.ground_truth(2, n, d)
    A = inst.measurement_matrix(2, Z, 0.0, dtype=np.float64)
    Y0 = inst.initial_subspace(2, n, d)
    X0, _, _ = ns.spectral_init(A, d, method, Y0=Y0)
    assert mt.d_F(X0, Z) <= 1e-8
    assert mt.rel_err_dense(X0, Z) <= 1e-8
    assert mt.rel_err(X0, Z) <= 1e-7      # Gram form: sqrt of a cancelling sum, floor ~sqrt(eps)


def test_subspace_matches_eigh():
    n, d, sigma = 200, 3, 2.0
    Z = inst.ground_truth(3, n, d)
    A = inst.measurement_matrix(3, Z, sigma)
    _, Ya, _ = ns.spectral_init(A, d, "eigh")
    _, Yb, sweeps = ns.spectral_init(A, d, "subspace", Y0=inst.initial_subspace(3, n, d), tol=1e-13)
    assert sweeps < 500
    assert np.linalg.norm(Ya @ Ya.T - Yb @ Yb.T) < 1e-10


# ---------------------------------------------------------------- metrics
def test_dF_bruteforce_d1():
    rng = np.random.default_rng(0)
    for n in range(2, 9):
        for _ in range(10):
            X = rng.choice([-1.0, 1.0], n).reshape(n, 1, 1) * rng.uniform(0.5, 1.5, (n, 1, 1))
            Y = rng.choice([-1.0, 1.0], n).reshape(n, 1, 1)
            brute = min(np.linalg.norm(X.ravel() - q * Y.ravel()) for q in (-1.0, 1.0))
            assert abs(mt.d_F_nuclear(X, Y) - brute) < 1e-12
            if abs(float(Y.ravel() @ X.ravel())) > 1e-9:
                assert abs(mt.d_F(X, Y) - brute) < 1e-12


def test_dF_antipodal_degenerate():
    # x = (1;1), y = (1;-1) -> Y^T X = 0, both Q = +-1 give 2.
    X = np.array([1.0, 1.0]).reshape(2, 1, 1)
    Y = np.array([1.0, -1.0]).reshape(2, 1, 1)
    assert abs(mt.d_F_nuclear(X, Y) - 2.0) < 1e-15


def test_dF_grid_search_O2():
    rng = np.random.default_rng(1)
    th = np.arange(0.0, 2 * np.pi, 1e-3)
    rots = np.stack([np.stack([np.cos(th), -np.sin(th)], -1), np.stack([np.sin(th), np.cos(th)], -1)], -2)
    refl = rots @ np.diag([1.0, -1.0])
    grid = np.concatenate([rots, refl])
    for _ in range(20):
        n = rng.integers(2, 7)
        X = np.stack([_haar(rng, 2) for _ in range(n)]) + 0.2 * rng.standard_normal((n, 2, 2))
        Y = np.stack([_haar(rng, 2) for _ in range(n)])
        Xs, Ys = X.reshape(-1, 2), Y.reshape(-1, 2)
        vals = np.linalg.norm(Xs[None] - Ys[None] @ grid, axis=(1, 2))
        g = vals.min()
        a, b = mt.d_F(X, Y), mt.d_F_nuclear(X, Y)
        assert a <= g + 1e-12 and g - a < 1e-5
        assert abs(a - b) < 1e-10


def test_le_sigma_identity_and_relerr_forms():
    # d_F^2 = 2nd - 2||Y^T X||_* for orthogonal stacks
    rng = np.random.default_rng(5)
    n, d = 30, 3
    X = np.stack([_haar(rng, d) for _ in range(n)])
    Y = np.stack([_haar(rng, d) for _ in range(n)])
    nuc = np.sum(np.linalg.svd(Y.reshape(-1, d).T @ X.reshape(-1, d), compute_uv=False))
    assert abs(mt.d_F(X, Y) ** 2 - (2 * n * d - 2 * nuc)) < 1e-10 * n * d
    assert abs(mt.rel_err(X, Y) - mt.rel_err_dense(X, Y)) < 1e-12
    Q = _haar(rng, d)
    assert abs(mt.rel_err(X @ Q, Y) - mt.rel_err(X, Y)) < 1e-12
    assert mt.rel_err(Y @ Q, Y) < 1e-13
    r, dF, m = mt.alignment_error(X, Y)
    assert abs(m - dF ** 2 / n) < 1e-14 * max(1, m)


def test_dF_pseudometric():
    rng = np.random.default_rng(6)
    n, d = 8, 3
    S = [np.stack([_haar(rng, d) for _ in range(n)]) + 0.1 * rng.standard_normal((n, d, d)) for _ in range(3)]
    for a, b, c in itertools.permutations(range(3)):
        assert mt.d_F(S[a], S[c]) <= mt.d_F(S[a], S[b]) + mt.d_F(S[b], S[c]) + 1e-12
    assert abs(mt.d_F(S[0], S[1]) - mt.d_F(S[1], S[0])) < 1e-12
