"""Bias of the fused fp32 objective (one-sided error of <X, A X>) of the wide-pass variants and
tcgen05 drain periods vs the fp64 oracle (test infrastructure: imports oracle/).  n 1100, d 16."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2604_07372_b200 import nsrgs
from oracle import instance as inst
from oracle import nsrgs as ons
from tests.gpu_helpers import oracle_iterate_near, rel_fro
n, d, sigma, K = 1100, 16, 0.2, 2
Z = inst.ground_truth(4, n, d); A = inst.measurement_matrix(4, Z, sigma)
X = oracle_iterate_near(Z, 0.1, 2).astype(np.float32)
Xo, _, _ = ons.step(A, X.astype(np.float64), 1.0 / n, K); fo = ons.objective(A, X.astype(np.float64))
xax = float(np.sum(X.astype(np.float64).reshape(-1, d) * (A @ X.astype(np.float64).reshape(-1, d))))
for mma, dr in (("0", "1"), ("1", "1"), ("2", "1"), ("2", "2"), ("2", "4")):
    os.environ["NSRGS_WIDE_MMA"] = mma; os.environ["NSRGS_WIDE_DRAIN"] = dr
    s = nsrgs.Solver(n, d); s.generate(4, sigma, want_Z=False); s.set_X(X); f = s.step(1.0 / n, K)
    print(f"mma={mma} drain={dr}: step rel {rel_fro(s.get_X(), Xo):.2e}  F err {f - fo:+.3f} rel F {abs(f - fo) / fo:.2e}  rel <X,AX> {abs(f - fo) / xax:.2e}", flush=True)
    s.close()
print("F", fo, "<X,AX>", xax)
