"""Spectral init + a few iterations at a given size, for an ncu launch list of the init kernels."""
import sys
sys.path.insert(0, ".")
from paper_2604_07372_b200 import nsrgs
n, d, sg = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (500, 25, 0.1)
s = nsrgs.Solver(n, d)
s.generate(0, sg, want_Z=False)
s.init_spectral(0, 200, 1e-6, allow_unconverged=True)
s.init_spectral(0, 200, 1e-6, allow_unconverged=True)
s.run(3, 1.0 / n, 1)
