"""Per-sweep subspace change of the spectral init (NSRGS_DEBUG_INIT=1 prints it from the library).
Usage: python tools/init_trace.py [n d sigma]; NSRGS_INIT_CHEB=0 for plain subspace iteration."""
import sys; sys.path.insert(0,'.')
import os
os.environ["NSRGS_DEBUG_INIT"]="1"
import numpy as np
from paper_2604_07372_b200 import nsrgs
n, d, sg = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (2000, 3, 8.0)
s=nsrgs.Solver(n,d); s.generate(3, sg, want_Z=False)
print("sweeps", s.init_spectral(3, 100, 1e-6, allow_unconverged=True), flush=True)
