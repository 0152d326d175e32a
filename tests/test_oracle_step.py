"""Pins for the NS-RGS step (§2.2, Algorithm 2 :232-251)."""
import numpy as np
import pytest

from oracle import instance as inst
from oracle import nsrgs as ns


def _haar(rng, d):
    Q, R = np.linalg.qr(rng.standard_normal((d, d)))
    return Q * np.sign(np.diag(R))


def _stack_haar(rng, n, d):
    return np.stack([_haar(rng, d) for _ in range(n)])


# ---------------------------------------------------------------- tangent projection
def test_tangent_projection_special_cases():
    rng = np.random.default_rng(0)
    d = 4
    G = rng.standard_normal((d, d))
    # X = I gives the skew part
    assert np.allclose(ns.tangent_project(np.eye(d), G), 0.5 * (G - G.T))
    X = _haar(rng, d)
    H = rng.standard_normal((d, d)); H = H - H.T
    S = rng.standard_normal((d, d)); S = S + S.T
    assert np.allclose(ns.tangent_project(X, X @ H), X @ H)      # tangent vectors fixed
    assert np.allclose(ns.tangent_project(X, X @ S), 0.0)        # normal space annihilated
    P = ns.tangent_project(X, G)
    assert np.allclose(ns.tangent_project(X, P), P)              # idempotent on-manifold
    assert np.allclose(X.T @ P, -(X.T @ P).T)                    # in T_X = {XH : H skew}


def test_tangent_projection_is_orthogonal_projection():
    rng = np.random.default_rng(1)
    d = 5
    X = _haar(rng, d)
    G = rng.standard_normal((d, d))
    R = G - ns.tangent_project(X, G)
    for _ in range(10):
        H = rng.standard_normal((d, d)); H = H - H.T
        assert abs(np.sum(R * (X @ H))) < 1e-12               # residual is normal to T_X


# ---------------------------------------------------------------- gradient vs objective
def test_gradient_matches_finite_difference_of_objective():
    # For X in O(d)^n and symmetric A with A_ii = 0, dF/dX_i = 2 sum_{j!=i}(X_i X_j^T X_j - A_ij X_j)
    # = 2 G_i (PAPER.md:200-202 uses X_j^T X_j = I).  Central differences of the literal F pin
    # the sign, indices and transposes of G.
    n, d, sigma = 6, 3, 0.8
    Z = inst.ground_truth(4, n, d)
    A = inst.measurement_matrix(4, Z, sigma, dtype=np.float64)
    rng = np.random.default_rng(2)
    X = _stack_haar(rng, n, d)
    G = ns.euclidean_gradient(A, X)
    h = 1e-6
    for i in (0, 3, 5):
        E = np.zeros_like(X)
        E[i] = rng.standard_normal((d, d))
        fd = (ns.objective(A, X + h * E) - ns.objective(A, X - h * E)) / (2 * h)
        assert abs(fd - 2.0 * np.sum(G[i] * E[i])) < 1e-6 * max(1.0, abs(fd))


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("n,d,K", [(2, 2, 1), (5, 3, 3), (8, 3, 5), (4, 5, 2)])
def test_step_matches_bruteforce_loops(n, d, K):
    rng = np.random.default_rng(10 * n + d)
    A = rng.standard_normal((n * d, n * d)); A = A + A.T        # nonzero A_ii: exclusion path
    X = _stack_haar(rng, n, d) + 0.01 * rng.standard_normal((n, d, d))
    mu = 1.0 / n
    Xv, _, _ = ns.step(A, X, mu, K)
    Xb = ns.step_bruteforce(A, X, mu, K)
    assert np.max(np.abs(Xv - Xb)) < 1e-13


# ---------------------------------------------------------------- invariances
def test_noiseless_truth_is_fixed_point():
    n, d = 30, 3
    Z = inst.ground_truth(1, n, d)
    A = inst.measurement_matrix(1, Z, 0.0, dtype=np.float64)
    Xn, F, G = ns.step(A, Z, 1.0 / n, 5)
    assert np.max(np.abs(G)) < 1e-12
    assert np.max(np.abs(Xn - Z)) < 1e-14


def test_global_rotation_equivariance():
    n, d, sigma, T = 40, 3, 0.5, 10
    Z = inst.ground_truth(5, n, d)
    A = inst.measurement_matrix(5, Z, sigma, dtype=np.float64)
    X0, _, _ = ns.spectral_init(A, d)
    Q = _haar(np.random.default_rng(3), d)
    XT = ns.run(A, X0, T, 1.0 / n, 3)
    XTQ = ns.run(A, X0 @ Q, T, 1.0 / n, 3)
    assert np.max(np.abs(XTQ - XT @ Q)) < 1e-12


def test_gauge_equivariance():
    # A'_ij = R_i^T A_ij R_j, X'_i = R_i^T X_i  =>  X'^{t+1}_i = R_i^T X^{t+1}_i
    n, d, sigma = 20, 4, 0.6
    Z = inst.ground_truth(6, n, d)
    A = inst.measurement_matrix(6, Z, sigma, dtype=np.float64)
    rng = np.random.default_rng(4)
    R = _stack_haar(rng, n, d)
    D = np.zeros((n * d, n * d))
    for i in range(n):
        D[i * d:(i + 1) * d, i * d:(i + 1) * d] = R[i]
    A2 = D.T @ A @ D
    X = _stack_haar(rng, n, d)
    X1, _, _ = ns.step(A, X, 1.0 / n, 4)
    X2, _, _ = ns.step(A2, np.transpose(R, (0, 2, 1)) @ X, 1.0 / n, 4)
    assert np.max(np.abs(X2 - np.transpose(R, (0, 2, 1)) @ X1)) < 1e-12


def test_ns_retraction_agrees_with_svd_retraction():
    # e_F^t = ||X^t - sgn(F^{t-1})||_F is tiny at K >= 3 (Remark :272-278).
    n, d, sigma = 100, 3, 0.5
    Z = inst.ground_truth(0, n, d)
    A = inst.measurement_matrix(0, Z, sigma)
    X0, _, _ = ns.spectral_init(A, d)
    Xa = ns.run(A, X0, 20, 1.0 / n, 3, "ns")
    Xb = ns.run(A, X0, 20, 1.0 / n, 3, "svd")
    assert np.linalg.norm(Xa - Xb) / np.linalg.norm(Xb) < 1e-10


def test_ns_region_and_descent():
    # ||I - F_i^T F_i||_2 < 1 every iteration (PAPER.md:449-468 le:error, Eq. eq:conclusion:sigma)
    # and F non-increasing at eta = 0.1/n.
    n, d, sigma = 60, 3, 2.0
    Z = inst.ground_truth(7, n, d)
    A = inst.measurement_matrix(7, Z, sigma)
    X, _, _ = ns.spectral_init(A, d)
    f_prev = ns.objective(A, X)
    I = np.eye(d)
    for _ in range(15):
        X, F, _ = ns.step(A, X, 0.1 / n, 5)
        assert max(np.linalg.norm(I - Fi.T @ Fi, 2) for Fi in F) < 1.0
        f = ns.objective(A, X)
        assert f <= f_prev * (1 + 1e-13)
        f_prev = f


def test_step_rows_equals_full_step():
    n, d, sigma = 30, 4, 0.9
    Z = inst.ground_truth(8, n, d)
    A = inst.measurement_matrix(8, Z, sigma)
    X = _stack_haar(np.random.default_rng(5), n, d)
    Xfull, _, _ = ns.step(A, X, 1.0 / n, 3)
    nodes = [0, 7, 29]
    R = inst.measurement_rows(8, Z, sigma, nodes)
    assert np.max(np.abs(ns.step_rows(R, X, nodes, 1.0 / n, 3) - Xfull[nodes])) < 1e-13


# ---------------------------------------------------------------- GPM (comparison method)
@pytest.mark.parametrize("n,d", [(3, 2), (6, 3), (5, 4)])
def test_gpm_matches_bruteforce(n, d):
    rng = np.random.default_rng(n + 10 * d)
    A = rng.standard_normal((n * d, n * d)); A = A + A.T
    X = _stack_haar(rng, n, d)
    assert np.max(np.abs(ns.gpm_step(A, X) - ns.gpm_step_bruteforce(A, X))) < 1e-12


def test_gpm_fixed_point_and_orthogonality():
    n, d = 25, 3
    Z = inst.ground_truth(2, n, d)
    A0 = inst.measurement_matrix(2, Z, 0.0, dtype=np.float64)
    assert np.max(np.abs(ns.gpm_step(A0, Z) - Z)) < 1e-13          # sgn((n-1) Z_i) = Z_i
    A = inst.measurement_matrix(2, Z, 1.5)
    Xn = ns.gpm_step(A, _stack_haar(np.random.default_rng(0), n, d))
    assert np.max(np.abs(np.einsum("nka,nkb->nab", Xn, Xn) - np.eye(d))) < 1e-13


def test_gpm_gauge_equivariance():
    n, d, sigma = 15, 3, 0.5
    Z = inst.ground_truth(6, n, d)
    A = inst.measurement_matrix(6, Z, sigma, dtype=np.float64)
    rng = np.random.default_rng(4)
    R = _stack_haar(rng, n, d)
    D = np.zeros((n * d, n * d))
    for i in range(n):
        D[i * d:(i + 1) * d, i * d:(i + 1) * d] = R[i]
    X = _stack_haar(rng, n, d)
    Rt = np.transpose(R, (0, 2, 1))
    assert np.max(np.abs(ns.gpm_step(D.T @ A @ D, Rt @ X) - Rt @ ns.gpm_step(A, X))) < 1e-12


def test_solve_protocol_stops_on_relative_decrease():
    n, d, sigma = 80, 3, 0.5
    Z = inst.ground_truth(3, n, d)
    A = inst.measurement_matrix(3, Z, sigma)
    X0, _, _ = ns.spectral_init(A, d)
    X, it, tr = ns.solve_protocol(A, X0, 1.0 / n, 1, "ns_rgs", max_iter=100, tol=1e-8)
    assert it < 100 and len(tr) == it + 1
    assert (tr[-2] - tr[-1]) / tr[-1] < 1e-8
    assert all((tr[k] - tr[k + 1]) / tr[k + 1] >= 1e-8 for k in range(it - 1))
    X1 = ns.run(A, X0, it, 1.0 / n, 1)
    assert np.max(np.abs(X1 - X)) < 1e-14
