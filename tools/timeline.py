"""Per-CTA phase timeline of the dense panel kernel (debug timestamps) for a small config."""
import sys
sys.path.insert(0, ".")
import numpy as np
from paper_2604_07372_b200 import nsrgs

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n, d, sigma, K = {"c1": (100, 3, 0.5, 3), "c2": (2000, 3, 0.5, 5), "c3": (20000, 5, 8.485, 5)}[cfg]
T = 12
s = nsrgs.Solver(n, d)
s.generate(0, sigma, want_Z=False)
s.init_spectral(0, 30, 1e-5, allow_unconverged=True)
s.run(T, 1.0 / n, K, trace=False)
s.debug_timestamps(T)
s.run(T, 1.0 / n, K, trace=True)
ts = s.debug_timestamps(0).astype(np.int64)      # [T][grid][8]
t0 = ts[0, :, 0].min()
ts = ts - t0
print(f"{cfg}: grid {ts.shape[1]}, us relative to launch start")
prev_end = 0
for it in range(T):
    x = ts[it]
    ready = x[:, 1] if it > 0 else x[:, 0]
    row = {
        "x_ready med/max": (np.median(ready) / 1e3, ready.max() / 1e3),
        "first stage med/max": (np.median(x[:, 2]) / 1e3, x[:, 2].max() / 1e3),
        "work done med/max": (np.median(x[:, 3]) / 1e3, x[:, 3].max() / 1e3),
        "stream done med/max": (np.median(x[:, 5]) / 1e3, x[:, 5].max() / 1e3),
        "epi cost med/max": (np.median((x[:, 3] - x[:, 6])[x[:, 6] > 0]) / 1e3, (x[:, 3] - x[:, 6])[x[:, 6] > 0].max() / 1e3),
        "reduce done max": (x[:, 4].max() / 1e3,),
    }
    print(f"it {it:2d} " + "  ".join(f"{k} " + "/".join(f"{v:7.1f}" for v in vals) for k, vals in row.items()))
iters = [ts[it, :, 4].max() for it in range(T)]
print("per-iteration (us):", np.round(np.diff(np.array(iters)) / 1e3, 1))
if "--raw" in sys.argv:
    it = T - 2
    x = ts[it]
    base = x[:, 1].min()
    print("cta: x_ready first_stage stream_done warpsum stored+fenced arrived combine_done work_done reduce_done (us from x_ready)")
    order = np.argsort(x[:, 3])[::-1][:10] if x.shape[0] > 16 else range(x.shape[0])
    for b in order:
        print(b, " ".join(f"{(x[b, k] - base) / 1e3:6.1f}" if x[b, k] > 0 else "     -" for k in (1, 2, 5, 7, 8, 9, 6, 3, 4)))
