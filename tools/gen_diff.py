"""Generator parity diagnostics: worst |A_gpu - A_oracle| in fp32 ulps for a wide-d instance."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from oracle import instance as inst
from paper_2604_07372_b200 import nsrgs

for (n, d, sigma, seed) in [(130, 14, 0.2, 4), (130, 14, 0.2, 5), (60, 12, 0.5, 4), (100, 16, 0.2, 4)]:
    s = nsrgs.Solver(n, d)
    Zg = s.generate(seed, sigma)
    Z = inst.ground_truth(seed, n, d)
    A = inst.measurement_matrix(seed, Z, sigma)
    Ag = s.copy_A_rows(0, n * d).astype(np.float64)
    sp = np.spacing(np.abs(A).astype(np.float32)).astype(np.float64)
    r = np.abs(Ag - A) / sp
    k = np.unravel_index(np.argmax(r), r.shape)
    print(n, d, sigma, seed, "max ulps", r.max(), "count>1", int((r > 1).sum()), "at", k, "A", A[k], "Ag", Ag[k],
          "Zdiff", float(np.max(np.abs(Zg - Z))), flush=True)
    s.close()
