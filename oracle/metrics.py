"""Oracle recovery metrics (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py)."""
from __future__ import annotations

import numpy as np

from .nsrgs import sgn, stack


def d_F(X: np.ndarray, Y: np.ndarray) -> float:
    """Distance up to a global rotation d_F(X, Y) = min_{Q in O(d)} ||X - Y Q||_F
    (§1.4).  Evaluated with the minimiser Q* = sgn(Y^T X)
    (PAPER.md:633 proof of le:sigma, "Q* = sgn(Y^T X) ... achieves this minimum")."""
    Xs, Ys = stack(X), stack(Y)
    Q = sgn(Ys.T @ Xs)
    return float(np.linalg.norm(Xs - Ys @ Q))


def d_F_nuclear(X: np.ndarray, Y: np.ndarray) -> float:
    """Nuclear-norm form d_F^2 = ||X||_F^2 + ||Y||_F^2 - 2 ||Y^T X||_*  (PAPER.md:633-637,
    proof of le:sigma, where ||X||^2 = ||Y||^2 = nd for orthogonal stacks; the general
    form is reading R13).  Needs no tie-break when Y^T X is singular."""
    Xs, Ys = stack(X), stack(Y)
    nuc = float(np.sum(np.linalg.svd(Ys.T @ Xs, compute_uv=False)))
    v = float(np.sum(Xs * Xs) + np.sum(Ys * Ys) - 2.0 * nuc)
    return float(np.sqrt(max(v, 0.0)))


def rel_err(X: np.ndarray, Z: np.ndarray) -> float:
    """Rel.Err. = ||Z Z^T - X X^T||_F / ||Z Z^T||_F (§4.1), via the d x d
    Gram identity ||ZZ^T - XX^T||^2 = ||Z^T Z||^2 + ||X^T X||^2 - 2 ||Z^T X||^2."""
    Xs, Zs = stack(X), stack(Z)
    zz = float(np.sum((Zs.T @ Zs) ** 2))
    xx = float(np.sum((Xs.T @ Xs) ** 2))
    zx = float(np.sum((Zs.T @ Xs) ** 2))
    return float(np.sqrt(max(zz + xx - 2.0 * zx, 0.0)) / np.sqrt(zz))


def rel_err_dense(X: np.ndarray, Z: np.ndarray) -> float:
    """Rel.Err. by its definition with the nd x nd matrices materialised (small n only)."""
    Xs, Zs = stack(X), stack(Z)
    return float(np.linalg.norm(Zs @ Zs.T - Xs @ Xs.T) / np.linalg.norm(Zs @ Zs.T))


def mse(Xhat: np.ndarray, X: np.ndarray) -> float:
    """MSE = (1/n) d_F(X^, X)^2 (§4.2)."""
    return d_F_nuclear(Xhat, X) ** 2 / Xhat.shape[0]


def alignment_error(X: np.ndarray, Z: np.ndarray):
    """(Rel.Err., d_F, MSE) of estimate X against ground truth Z — the triple returned by
    nsrgs_alignment_error (reading R12).  d_F is measured from X to the truth Z, i.e.
    d_F(X, Z) = min_Q ||X - Z Q||_F; MSE = d_F^2 / n."""
    dF = d_F_nuclear(X, Z)
    return rel_err(X, Z), dF, dF * dF / X.shape[0]
