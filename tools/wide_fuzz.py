"""Shape fuzz of the tcgen05 wide pass against the CUDA-core pass (NSRGS_WIDE_MMA=0): random small
and ragged (n, d), step / objective / GPM / subspace product via init.  Usage: python tools/wide_fuzz.py [cases]"""
import os, sys
sys.path.insert(0, '.')
import numpy as np
from paper_2604_07372_b200 import nsrgs
rng = np.random.default_rng(7)
cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
ds = [11, 12, 13, 14, 15, 16, 20, 24, 25, 32]
worst = 0.0
for c in range(cases):
    d = int(rng.choice(ds)); n = int(rng.choice([1, 2, 3, 5, 9, 10, 11, 17, 33, 64, 100, 129, 257, 400]))
    if n * d < 16: n = 3
    sigma = float(rng.choice([0.0, 0.1, 0.5])); K = int(rng.integers(0, 4))
    X = np.linalg.qr(rng.standard_normal((n, d, d)))[0].astype(np.float32)
    out = {}
    for v in ("0", "2"):
        os.environ["NSRGS_WIDE_MMA"] = v
        s = nsrgs.Solver(n, d); s.generate(c, sigma, want_Z=False)
        s.set_X(X); f = s.step(1.0 / max(n, 2), K); X1 = s.get_X()
        s.set_X(X); s.gpm_run(1); X2 = s.get_X()
        s.set_X(X); fo = s.objective()
        out[v] = (f, X1, X2, fo); s.close()
    e1 = np.linalg.norm(out["2"][1] - out["0"][1]) / np.linalg.norm(out["0"][1])
    e2 = np.linalg.norm(out["2"][2] - out["0"][2]) / np.linalg.norm(out["0"][2])
    ef = abs(out["2"][0] - out["0"][0]) / max(abs(out["0"][0]), 1e-30)
    eo = abs(out["2"][3] - out["0"][3]) / max(abs(out["0"][3]), 1e-30)
    worst = max(worst, e1, e2)
    flag = "" if (e1 < 2e-6 and e2 < 2e-6 and ef < 1e-5 and eo < 1e-5) else "   <-- CHECK"
    print(f"n={n:4d} d={d:2d} sigma={sigma} K={K}: step {e1:.1e} gpm {e2:.1e} F {ef:.1e} obj {eo:.1e}{flag}", flush=True)
print("worst iterate difference", worst)
