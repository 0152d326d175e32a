"""Block-sparse (p < 1) pass timing: n, d, p from argv (default the c3 size at p = 0.5).
Prints pass ms (CUDA events around each pass, library stream) and GB/s of the stored bytes."""
import json, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2604_07372_b200 import nsrgs
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
T = int(sys.argv[4]) if len(sys.argv) > 4 else 20
storage = sys.argv[5] if len(sys.argv) > 5 else "bsr"   # "dense": the same instance, dense storage
K = 5
sigma = 0.3 * np.sqrt(n) / d
s = nsrgs.Solver(n, d)
s.generate(0, sigma, want_Z=False, p=p, storage=storage)
rng = np.random.default_rng(0)
s.set_X(np.linalg.qr(rng.standard_normal((n, d, d)))[0].astype(np.float32))
s.run(3, 1.0 / (n * p), K, trace=False)
s.reset_stats(timing=True)
s.run(T, 1.0 / (n * p), K, trace=True)
st = s.stats()
ms = st["panel_ms_total"] / st["panel_launches"]
out = {"storage": storage, "n": n, "d": d, "p": p, "nnzb": st["bsr_nnzb"], "bytes_per_pass": st["a_bytes_per_pass"],
       "pass_ms": ms, "gbs": st["a_bytes_per_pass"] / ms / 1e6,
       "dense_equiv_gbs": 4.0 * (n * d) ** 2 / ms / 1e6}
print(json.dumps(out))
