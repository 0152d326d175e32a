"""Resolution of the R^t < 1e-8 stopping rule with fp32 iterates (reading R21).

For Table 1 cells (n = 500, d = 25, T_s = 1, mu = 1/(np)), run the fp64 oracle protocol from the
fp32-rounded spectral X^0 twice: with fp64 iterates, and with every iterate rounded to fp32
(arithmetic otherwise fp64).  Prints both R^t sequences: their difference is the band within
which an fp32 implementation cannot reproduce the fp64 decision.  Oracle-only (CPU).
"""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import instance as inst  # noqa: E402
from oracle import nsrgs as ons  # noqa: E402

n, d = 500, 25
Z = inst.ground_truth(0, n, d)
Y0 = inst.initial_subspace(0, n, d)
for p, sigma in [(0.8, 0.2), (1.0, 0.2), (0.5, 0.2)]:
    A = inst.measurement_matrix(0, Z, sigma, p=p).astype(np.float64)
    X0, _, _ = ons.spectral_init(A, d, "subspace", Y0=Y0, tol=1e-10)
    X0 = X0.astype(np.float32).astype(np.float64)
    _, _, tr = ons.solve_protocol(A, X0, 1 / (n * p), 1, "ns_rgs", max_iter=6, tol=0)
    tr = np.array(tr)
    X, F = X0.copy(), [ons.objective_expanded(A, X0)]
    for _ in range(6):
        X = ons.step(A, X, 1 / (n * p), 1)[0].astype(np.float32).astype(np.float64)
        F.append(ons.objective_expanded(A, X))
    F = np.array(F)
    print(p, sigma, "R fp64 iterates", (tr[:-1] - tr[1:]) / tr[1:])
    print("          R fp32 iterates", (F[:-1] - F[1:]) / F[1:])
