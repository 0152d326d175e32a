"""Oracle for NS-RGS (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Every function follows PAPER.md in the paper's order and notation, in fp64.
Block stacks X, Z, Y, F, G are arrays of shape (n, d, d) (block i = X[i]);
``stack(X)`` gives the nd x d matrix of PAPER.md:128 (§1.4).
"""
from __future__ import annotations

import numpy as np


# ----------------------------------------------------------------------------- helpers
def stack(X: np.ndarray) -> np.ndarray:
    """(n, d, d) blocks -> nd x d matrix (X_1; ...; X_n)."""
    n, d, _ = X.shape
    return X.reshape(n * d, d)


def unstack(M: np.ndarray, d: int) -> np.ndarray:
    return M.reshape(-1, d, d)


# ----------------------------------------------------------------------------- §2.1
def sgn(A: np.ndarray) -> np.ndarray:
    """Matrix sign sgn(A) = U V^T from the SVD A = U S V^T (§2.1).
    Works blockwise on (..., d, d) arrays ("sgn(Phi) = (sgn(A_1); ...)", :141)."""
    U, _, Vt = np.linalg.svd(A)
    return U @ Vt


def newton_schulz(A: np.ndarray, Ts: int) -> np.ndarray:
    """Algorithm 1: S_0 = A; S_{t+1} = 1/2 S_t (3 I_d - S_t^T S_t),
    t = 0..Ts-1.  No pre-scaling (Alg. 1 "Set S_0 = A").  Blockwise on (..., d, d)."""
    S = np.array(A, dtype=np.float64, copy=True)
    d = S.shape[-1]
    I = np.eye(d)
    for _ in range(Ts):
        S = 0.5 * S @ (3.0 * I - np.swapaxes(S, -1, -2) @ S)
    return S


def tangent_project(X: np.ndarray, G: np.ndarray) -> np.ndarray:
    """P_{T_X}(G) = (G - X G^T X) / 2 (§2.2), applied literally even when
    X is off the manifold ("pseudo projection")."""
    return 0.5 * (G - X @ np.swapaxes(G, -1, -2) @ X)


# ----------------------------------------------------------------------------- §2.2 Alg. 2
def euclidean_gradient(A: np.ndarray, X: np.ndarray) -> np.ndarray:
    """G_i = sum_{j != i} (X_i - A_ij X_j)  (PAPER.md:243, Alg. 2 first line; :200-202).

    The sum over j != i is written as (n-1) X_i - (sum_j A_ij X_j - A_ii X_i); the
    matmul A @ stack(X) is the library step.  A_ii is excluded literally even if
    nonzero (it is zero for every instance of PAPER.md:229)."""
    n, d, _ = X.shape
    AX = unstack(A @ stack(X), d)                       # sum_j A_ij X_j
    Aii = np.stack([A[i * d:(i + 1) * d, i * d:(i + 1) * d] for i in range(n)])
    return (n - 1) * X - (AX - Aii @ X)


def step(A: np.ndarray, X: np.ndarray, mu: float, Ts: int, retraction: str = "ns"):
    """One iteration t -> t+1 of Algorithm 2, all i from X^t (Jacobi):

        G_i^t = sum_{j != i} (X_i^t - A_ij X_j^t)
        F_i^t = X_i^t - mu P_{T_{X_i^t}}(G_i^t)
        X_i^{t+1} = S(F_i^t)      (S = Algorithm 1 with Ts steps)

    ``retraction="svd"`` uses the exact retraction X~^{t+1} = sgn(F^t).
    Returns (X^{t+1}, F^t, G^t)."""
    G = euclidean_gradient(A, X)
    F = X - mu * tangent_project(X, G)
    if retraction == "ns":
        Xn = newton_schulz(F, Ts)
    elif retraction == "svd":
        Xn = sgn(F)
    else:
        raise ValueError(retraction)
    return Xn, F, G


def step_rows(A_rows: np.ndarray, X: np.ndarray, nodes, mu: float, Ts: int) -> np.ndarray:
    """Algorithm 2's update for the listed nodes only, given just their block
    rows of A (shape (len(nodes)*d, nd)): the same arithmetic as ``step`` restricted to rows
    i in `nodes` (Jacobi, reads X^t only).  Used for sampled parity at sizes where the dense A
    does not fit the host, and for the bounded-sample CPU baseline."""
    n, d, _ = X.shape
    Xs = stack(X)
    out = []
    for k, i in enumerate(nodes):
        Ai = A_rows[k * d:(k + 1) * d]
        Aii = Ai[:, i * d:(i + 1) * d]
        G = (n - 1) * X[i] - (Ai @ Xs - Aii @ X[i])          # sum_{j != i}(X_i - A_ij X_j)
        F = X[i] - mu * tangent_project(X[i], G)
        out.append(newton_schulz(F, Ts))
    return np.stack(out)


def step_bruteforce(A, X, mu, Ts):
    """Algorithm 2's inner loop written with explicit Python loops over i, j and matrix
    entries (no numpy matmul).  The oracle's own oracle for n <= 8."""
    n, d, _ = X.shape
    Xl = X.tolist()
    Al = np.asarray(A).tolist()

    def mm(P, Q):
        return [[sum(P[a][k] * Q[k][b] for k in range(d)) for b in range(d)] for a in range(d)]

    def tr(P):
        return [[P[b][a] for b in range(d)] for a in range(d)]

    out = []
    for i in range(n):
        Gi = [[0.0] * d for _ in range(d)]
        for j in range(n):
            if j == i:
                continue
            Aij = [[Al[i * d + a][j * d + b] for b in range(d)] for a in range(d)]
            AX = mm(Aij, Xl[j])
            for a in range(d):
                for b in range(d):
                    Gi[a][b] += Xl[i][a][b] - AX[a][b]
        XGX = mm(mm(Xl[i], tr(Gi)), Xl[i])
        F = [[Xl[i][a][b] - mu * 0.5 * (Gi[a][b] - XGX[a][b]) for b in range(d)] for a in range(d)]
        S = F
        for _ in range(Ts):
            StS = mm(tr(S), S)
            M = [[(3.0 if a == b else 0.0) - StS[a][b] for b in range(d)] for a in range(d)]
            SM = mm(S, M)
            S = [[0.5 * SM[a][b] for b in range(d)] for a in range(d)]
        out.append(S)
    return np.array(out)


def run(A: np.ndarray, X0: np.ndarray, T: int, mu: float, Ts: int, retraction: str = "ns",
        trace_objective: bool = False):
    """Riemannian gradient updates of Algorithm 2 for t = 0..T-1.
    Returns X^T and (optionally) [F(X^0), ..., F(X^{T-1})]."""
    X = np.array(X0, dtype=np.float64, copy=True)
    trace = []
    for _ in range(T):
        if trace_objective:
            trace.append(objective(A, X))
        X, _, _ = step(A, X, mu, Ts, retraction)
    return (X, trace) if trace_objective else X


# ----------------------------------------------------------------------------- GPM (comparison method)
def gpm_step(A: np.ndarray, X: np.ndarray) -> np.ndarray:
    """Generalized power method, the paper's comparison system (§4.1, cited from
    Ling 2022): X_i^{t+1} = sgn(sum_{j != i} A_ij X_j^t) blockwise (definition as in SPEC.md:245-253;
    DESIGN.md reading R17).  Jacobi, exact SVD sign."""
    n, d, _ = X.shape
    AX = unstack(A @ stack(X), d)
    Aii = np.stack([A[i * d:(i + 1) * d, i * d:(i + 1) * d] for i in range(n)])
    return sgn(AX - Aii @ X)


def gpm_step_bruteforce(A, X):
    """gpm_step with explicit Python loops for the block sums (the SVD sign is the library step)."""
    n, d, _ = X.shape
    out = []
    for i in range(n):
        S = [[0.0] * d for _ in range(d)]
        for j in range(n):
            if j == i:
                continue
            for a in range(d):
                for b in range(d):
                    S[a][b] += sum(A[i * d + a, j * d + k] * X[j][k][b] for k in range(d))
        out.append(sgn(np.array(S)))
    return np.array(out)


def solve_protocol(A: np.ndarray, X0: np.ndarray, mu: float, Ts: int, algorithm: str = "ns_rgs",
                   max_iter: int = 100, tol: float = 1e-8):
    """The paper's experimental protocol (§4.1): iterate from X^0 until
    R^t = (F(X^t) - F(X^{t+1})) / F(X^{t+1}) < tol or MaxIter iterations.  Returns
    (X_final, iterations, [F(X^0), F(X^1), ...])."""
    X = np.array(X0, dtype=np.float64, copy=True)
    f = objective_expanded(A, X)
    trace = [f]
    it = 0
    while it < max_iter:
        Xn = step(A, X, mu, Ts)[0] if algorithm == "ns_rgs" else gpm_step(A, X)
        fn = objective_expanded(A, Xn)
        it += 1
        X = Xn
        trace.append(fn)
        R = (f - fn) / fn
        f = fn
        if R < tol:
            break
    return X, it, trace


# ----------------------------------------------------------------------------- spectral init
def spectral_init(A: np.ndarray, d: int, method: str = "eigh", Y0=None, tol: float = 1e-13,
                  max_sweeps: int = 500):
    """Spectral initialization of Algorithm 2: Y = top d
    eigenvectors of A with Y^T Y = I_d, X^0 = sgn(Y) blockwise.

    "Top" = largest algebraic eigenvalues (reading R7).  method="eigh": dense
    symmetric eigendecomposition (library step).  method="subspace": block power
    iteration Y <- A Y with Cholesky-QR orthonormalisation, stopped when the subspace
    change ||Y_new - Y_old (Y_old^T Y_new)||_F < tol (finds the largest-|lambda| subspace,
    equal to the algebraic one under the gap condition of reading R7).
    Returns (X0, Y, sweeps_used)."""
    N = A.shape[0]
    if method == "eigh":
        w, V = np.linalg.eigh(A)
        Y = V[:, np.argsort(w)[::-1][:d]]
        sweeps = 0
    elif method == "subspace":
        Y = np.array(Y0, dtype=np.float64, copy=True)
        Y = _chol_qr(Y)
        sweeps = 0
        while sweeps < max_sweeps:
            W = A @ Y
            Yn = _chol_qr(W)
            sweeps += 1
            change = np.linalg.norm(Yn - Y @ (Y.T @ Yn))
            Y = Yn
            if change < tol:
                break
    else:
        raise ValueError(method)
    X0 = sgn(unstack(Y, d))
    return X0, Y, sweeps


def _chol_qr(W):
    L = np.linalg.cholesky(W.T @ W)
    return np.linalg.solve(L, W.T).T       # W L^{-T}


# ----------------------------------------------------------------------------- objective
def objective(A: np.ndarray, X: np.ndarray) -> float:
    """F(X) = sum_{i != j} 1/2 ||X_i X_j^T - A_ij||_F^2 (PAPER.md:70-72 Eq. def:f;
    :192-194), summed literally over ordered pairs i != j, block row by block row."""
    n, d, _ = X.shape
    total = 0.0
    for i in range(n):
        R = np.einsum("ak,jbk->jab", X[i], X)            # X_i X_j^T for all j
        Ai = A[i * d:(i + 1) * d, :].reshape(d, n, d).transpose(1, 0, 2)
        D = R - Ai
        D[i] = 0.0                                       # exclude j = i
        total += 0.5 * float(np.sum(D * D))
    return total


def objective_expanded(A: np.ndarray, X: np.ndarray) -> float:
    """Algebraic expansion of F used by the device path (ours; pinned equal to
    ``objective``):  F = 1/2(||X^T X||^2 - sum_i ||X_i^T X_i||^2) - <X, A X> + 1/2 ||A||^2,
    valid when A_ii = 0."""
    Xs = stack(X)
    XtX = Xs.T @ Xs
    own = sum(float(np.sum((Xi.T @ Xi) ** 2)) for Xi in X)
    return 0.5 * (float(np.sum(XtX ** 2)) - own) - float(np.sum(Xs * (A @ Xs))) + 0.5 * float(np.sum(A * A))
