"""One multi-iteration NS-RGS launch on a small config (no init launches): target for ncu."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2604_07372_b200 import nsrgs

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 200
n, d, sigma, K = {"c1": (100, 3, 0.5, 3), "c2": (2000, 3, 0.5, 5)}[cfg]
s = nsrgs.Solver(n, d)
s.generate(0, sigma, want_Z=False)
rng = np.random.default_rng(0)
X0 = np.stack([np.linalg.qr(rng.standard_normal((d, d)))[0] for _ in range(n)]).reshape(n * d, d)
s.set_X(X0)
tr = s.run(T, 1.0 / n, K, trace=True)
print(cfg, "trace tail", tr[-2:])
