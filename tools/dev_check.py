"""Developer check: time the panel pass on a BASELINE config (no oracle).  [--sym] [--gpm]"""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2604_07372_b200 import nsrgs

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
sym = "--sym" in sys.argv
n, d, c = {"c2": (2000, 3, None), "c3": (20000, 5, 0.3), "c4": (12000, 10, 0.2), "c5": (40000, 5, 0.3)}[cfg]
sigma = 0.5 if c is None else c * np.sqrt(n) / d
K = {"c2": 5, "c3": 5, "c4": 6, "c5": 5}[cfg]
s = nsrgs.Solver(n, d)
t = time.time(); Z = s.generate(0, sigma); torch.cuda.synchronize(); print("generate s", time.time() - t, flush=True)
if sym:
    s.set_symmetric(True)
t = time.time(); sw = s.init_spectral(0, 100, 1e-5, allow_unconverged=True); print("init sweeps", sw, "s", time.time() - t, flush=True)
s.reset_stats(True)
tr = s.run(20, 1.0 / n, K)
st = s.stats()
N = n * d
ms = st["panel_ms_total"] / st["panel_launches"]
print(cfg, "sym" if sym else "dense", "trace", tr[:2], tr[-2:], "rel_err", s.alignment_error(Z)[0])
print("stats", st)
print(f"{cfg} {'sym' if sym else 'dense'} pass ms {ms:.3f}  A-bytes GB/s {st['a_bytes_per_pass'] / ms / 1e6:.1f}  "
      f"dense-equivalent GB/s {4 * N * N / ms / 1e6:.1f}")
