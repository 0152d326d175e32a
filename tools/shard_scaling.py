"""Per-rank pass time of a P-way row-sharded config, measured rank by rank on ONE GPU with
NSRGS_EMULATE_RANKS=1 (no collectives): projects the kernel side of strong scaling (the NCCL
all-gather of X, 2-5 MB per iteration, is not included)."""
import os, sys, json
os.environ["NSRGS_EMULATE_RANKS"] = "1"
sys.path.insert(0, ".")
import numpy as np
from paper_2604_07372_b200 import nsrgs
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n, d, c, K = {"c3": (20000, 5, 0.3, 5), "c4": (12000, 10, 0.2, 6), "c5": (40000, 5, 0.3, 5)}[cfg]
sigma = c * np.sqrt(n) / d
Z = None
X = None
out = {"cfg": cfg}
worlds = [int(w) for w in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["1", "2", "4", "8"])]
for world in worlds:
    times = []
    for r in sorted({0, world - 1}):
        s = nsrgs.Solver(n, d, rank=r, world=world)
        s.generate(0, sigma, want_Z=False)
        if X is None:
            rng = np.random.default_rng(0)
            q, _ = np.linalg.qr(rng.standard_normal((n, d, d)))
            X = q.astype(np.float32)
        s.set_X(X)
        s.run(2, 1.0 / n, K, trace=False)
        s.reset_stats(True)
        s.run(10, 1.0 / n, K, trace=False)
        st = s.stats()
        times.append(st["panel_ms_total"] / st["panel_launches"])
        s.close()
    out[f"P{world}"] = {"rank_pass_ms": [round(t, 4) for t in times]}
t1 = out.get("P1", {}).get("rank_pass_ms", [None])[0]
for world in worlds:
    if t1 and world > 1:
        tw = max(out[f"P{world}"]["rank_pass_ms"])
        out[f"P{world}"]["kernel_scaling_eff"] = round(t1 / (world * tw), 4)
print(json.dumps(out))
