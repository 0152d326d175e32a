"""Statistical pin: the oracle reproduces PAPER.md Table 1 (p = 1 row) with the paper's own
protocol (§4.1): spectral init, mu = 1/(np), one Newton-Schulz step,
stop at R^t < 1e-8 or MaxIter = 100.  One seed (the paper averages 10 trials; at
n = 500, d = 25 the trial-to-trial spread of Rel.Err. is far below the 5% band)."""
import os

import numpy as np
import pytest

from oracle import instance as inst
from oracle import metrics as mt
from oracle import nsrgs as ns

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _table1():
    with open(os.path.join(GOLD, "table1_relerr.txt")) as f:
        return [tuple(float(t) for t in l.split()) for l in f if l.strip() and not l.startswith("#")]


@pytest.fixture(scope="module")
def table1_instance():
    n, d, seed = 500, 25, 0
    Z = inst.ground_truth(seed, n, d)
    A1 = inst.measurement_matrix(seed, Z, 1.0, dtype=np.float64)     # Z Z^T + 1 * W (off-diagonal)
    Zs = Z.reshape(n * d, d)
    A0 = Zs @ Zs.T
    for i in range(n):
        A0[i * d:(i + 1) * d, i * d:(i + 1) * d] = 0.0
    return n, d, seed, Z, A0, A1 - A0


def _mask_matrix(seed, n, d, p):
    M = np.zeros((n, n), dtype=bool)
    for i in range(n - 1):
        js = np.arange(i + 1, n)
        M[i, js] = inst.observed(seed, i, js, p)
    M = M | M.T
    return np.kron(M, np.ones((d, d), dtype=bool))


@pytest.mark.parametrize("p", [1.0, 0.8, 0.5])
def test_table1_relerr(table1_instance, p):
    """Table 1 row p for NS-RGS and GPM, mu = 1/(np)."""
    n, d, seed, Z, A0, W = table1_instance
    M = _mask_matrix(seed, n, d, p) if p < 1.0 else None
    cells = [c for c in _table1() if c[2] == p]
    assert len(cells) == 3
    for (n_, d_, p_, sigma, rel_paper) in cells:
        assert (int(n_), int(d_)) == (n, d)
        A = A0 + sigma * W
        if M is not None:
            A = np.where(M, A, 0.0)                                   # A_ij = 0 off the edge set
        X0, _, _ = ns.spectral_init(A, d, "subspace", Y0=inst.initial_subspace(seed, n, d), tol=1e-10)
        rels = {}
        for alg in ("ns_rgs", "gpm"):                               # Table 1 rows NS-RGS and GPM
            X, it, _ = ns.solve_protocol(A, X0, 1.0 / (n * p), 1, alg)   # mu = 1/(np), T_s = 1
            rels[alg] = mt.rel_err(X, Z)
            assert abs(rels[alg] - rel_paper) <= 0.05 * rel_paper, (alg, p, sigma, rels[alg], rel_paper)
        # NS-RGS and GPM agree (identical printed values)
        assert abs(rels["ns_rgs"] - rels["gpm"]) <= 1e-4
        # first-order closed form Rel.Err ~ sigma sqrt((d-1)/(np)) (ours) within 3%
        assert abs(rels["ns_rgs"] - sigma * np.sqrt((d - 1) / (n * p))) <= 0.03 * rels["ns_rgs"]


def test_mask_is_symmetric_bernoulli():
    n, p = 2000, 0.3
    i, j = np.triu_indices(n, 1)
    m = inst.observed(5, i, j, p)
    frac = m.mean()
    assert abs(frac - p) < 5 * np.sqrt(p * (1 - p) / m.size)
    # measurement_matrix applies the same mask to both triangles, rows agree with the matrix
    Z = inst.ground_truth(1, 40, 3)
    A = inst.measurement_matrix(1, Z, 0.5, p=0.4)
    assert np.array_equal(A, A.T)
    R = inst.measurement_rows(1, Z, 0.5, [0, 17, 39], p=0.4)
    for k, nd in enumerate([0, 17, 39]):
        assert np.array_equal(R[k * 3:(k + 1) * 3], A[nd * 3:(nd + 1) * 3])
    blocks = A.reshape(40, 3, 40, 3).transpose(0, 2, 1, 3)
    zero = np.all(blocks == 0, axis=(2, 3))
    iu = np.triu_indices(40, 1)
    assert np.array_equal(~zero[iu], inst.observed(1, iu[0], iu[1], 0.4))
