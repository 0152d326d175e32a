"""Measured one-step error at full sizes (sampled nodes vs the fp64 oracle) and the fixed-point
residual of X^T after spectral init + T iterations: ||step_rows(X^T)_i - X^T_i|| on sampled nodes."""
import sys

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import instance as inst  # noqa: E402
from oracle import nsrgs as ons  # noqa: E402
from paper_2604_07372_b200 import nsrgs  # noqa: E402

FULL = {"mid": (6000, 3, 1.0, 5), "c3": (20000, 5, 0.3 * np.sqrt(20000) / 5, 5),
        "c4": (12000, 10, 0.2 * np.sqrt(12000) / 10, 6), "c5": (40000, 5, 0.3 * np.sqrt(40000) / 5, 5)}


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


for cfg in sys.argv[1:] or FULL:
    n, d, sigma, K = FULL[cfg]
    s = nsrgs.Solver(n, d)
    Z = s.generate(0, sigma).astype(np.float64)
    rng = np.random.default_rng(3)
    X = ons.sgn(Z + 0.05 * rng.standard_normal(Z.shape)).astype(np.float32)
    s.set_X(X)
    s.step(1.0 / n, K)
    Xg = s.get_X()
    nodes = np.unique(np.r_[0, n - 1, np.random.default_rng(1).integers(0, n, 62)])
    R = inst.measurement_rows(0, Z, sigma, nodes)
    Xo = ons.step_rows(R, X.astype(np.float64), nodes, 1.0 / n, K)
    blk = np.linalg.norm(Xg[nodes] - Xo, axis=(1, 2)) / np.sqrt(d)
    # fp32 rounding of X alone
    r32 = rel(Xo.astype(np.float32), Xo)
    s.init_spectral(0, 100, 1e-5)
    s.run(100, 1.0 / n, K, trace=False)
    XT = s.get_X().astype(np.float64)
    Xf = ons.step_rows(R, XT, nodes, 1.0 / n, K)
    fblk = np.linalg.norm(Xf - XT[nodes], axis=(1, 2)) / np.sqrt(d)
    print(f"{cfg}: one-step rel {rel(Xg[nodes], Xo):.3e} max-block {blk.max():.3e} (fp32 rounding of X alone "
          f"{r32:.3e}); fixed-point residual rel {rel(XT[nodes], Xf):.3e} max-block {fblk.max():.3e}", flush=True)
    s.close()
