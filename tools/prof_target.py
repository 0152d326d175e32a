"""Minimal ncu target: one config, a random orthogonal X, 4 single-iteration NS-RGS launches
(nsrgs_step: one panel launch each).  ncu -k regex:panel_kernel -s 3 -c 1 captures the 4th.
`python tools/prof_target.py c3 sym`: the same with the symmetric pass (-k regex:sym_block);
`w25` (n 4000, d 25) exercises the wide pass (-k regex:wide_kernel)."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2604_07372_b200 import nsrgs
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
sym = "sym" in sys.argv[2:]   # symmetric half-storage pass (sym_block_kernel + sym_final_kernel)
n, d, c, K = {"c2": (2000, 3, None, 5), "c3": (20000, 5, 0.3, 5), "c4": (12000, 10, 0.2, 6),
              "w25": (4000, 25, 0.2, 1), "w500": (500, 25, 0.2, 1), "w16": (8000, 16, 0.2, 1)}[cfg]   # w25: wide pass (-k regex:wide_kernel)
s = nsrgs.Solver(n, d)
s.generate(0, 0.5 if c is None else c * np.sqrt(n) / d, want_Z=False)
rng = np.random.default_rng(0)
if sym:
    s.set_symmetric(True)
s.set_X(np.linalg.qr(rng.standard_normal((n, d, d)))[0].astype(np.float32))
for _ in range(4):
    f = s.step(1.0 / n, K)
print(cfg, "F", f, "stats", s.stats())
