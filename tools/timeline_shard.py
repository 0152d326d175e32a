"""Phase timestamps of ONE pass of a P-way shard (rank 0, NSRGS_EMULATE_RANKS=1, one launch)."""
import os, sys
os.environ["NSRGS_EMULATE_RANKS"] = "1"
sys.path.insert(0, ".")
import numpy as np
from paper_2604_07372_b200 import nsrgs

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n, d, c, K = {"c3": (20000, 5, 0.3, 5), "c4": (12000, 10, 0.2, 6)}[cfg]
s = nsrgs.Solver(n, d, rank=0, world=world)
s.generate(0, c * np.sqrt(n) / d, want_Z=False)
rng = np.random.default_rng(0)
s.set_X(np.linalg.qr(rng.standard_normal((n, d, d)))[0].astype(np.float32))
s.run(3, 1.0 / n, K, trace=False)
s.debug_timestamps(1)
s.run(1, 1.0 / n, K, trace=False)
x = s.debug_timestamps(0).astype(np.int64)[0]
t0 = x[:, 0].min()
us = lambda v: (v - t0) / 1e3
print(f"{cfg} P={world} rank 0, grid {x.shape[0]}, stats {s.stats()['panels']} panels")
for name, k in [("producer start", 0), ("first stage", 2), ("stream done (last seg)", 5), ("combine done", 6),
                ("work done", 3), ("cta reduce done", 4)]:
    v = x[:, k]
    v = v[v > 0]
    if len(v):
        q = np.percentile(us(v), [0, 10, 50, 90, 100])
        print(f"{name:24s} min/p10/med/p90/max " + " ".join(f"{a:8.1f}" for a in q))
sm = x[:, 11]
done = us(x[:, 5])
order = np.argsort(sm)
print("smid -> stream done (us), sorted by smid:")
for i in range(0, len(order), 8):
    print(" ".join(f"{sm[j]:3d}:{done[j]:7.1f}" for j in order[i:i + 8]))
