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


def test_table1_p1_relerr(table1_instance):
    n, d, seed, Z, A0, W = table1_instance
    for (n_, d_, p, sigma, rel_paper) in _table1():
        assert (int(n_), int(d_), p) == (n, d, 1.0)
        A = A0 + sigma * W
        X0, _, _ = ns.spectral_init(A, d, "subspace", Y0=inst.initial_subspace(seed, n, d), tol=1e-10)
        rels = {}
        for alg in ("ns_rgs", "gpm"):                               # Table 1 rows NS-RGS and GPM
            X, it, _ = ns.solve_protocol(A, X0, 1.0 / (n * p), 1, alg)   # mu = 1/(np), T_s = 1
            rels[alg] = mt.rel_err(X, Z)
            assert abs(rels[alg] - rel_paper) <= 0.05 * rel_paper, (alg, sigma, rels[alg], rel_paper)
        # NS-RGS and GPM agree (identical printed values)
        assert abs(rels["ns_rgs"] - rels["gpm"]) <= 1e-4
        # first-order closed form Rel.Err ~ sigma sqrt((d-1)/(np)) (ours) within 2%
        assert abs(rels["ns_rgs"] - sigma * np.sqrt((d - 1) / n)) <= 0.02 * rels["ns_rgs"]
