"""Where the wide pass spends its time at small n: objective-only pass vs K = 0 / 1 / 3 steps.
Usage: python tools/wide_parts.py [n d]"""
import sys, time
sys.path.insert(0, '.')
import numpy as np
from paper_2604_07372_b200 import nsrgs
n, d = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (500, 25)
s = nsrgs.Solver(n, d); s.generate(0, 0.1, want_Z=False)
rng = np.random.default_rng(0)
X = np.linalg.qr(rng.standard_normal((n, d, d)))[0].astype(np.float32)
def timed(fn, reps=20):
    s.set_X(X); fn(); s.reset_stats(True)
    for _ in range(reps):
        s.set_X(X); fn()
    st = s.stats(); return st['panel_ms_total'] / st['panel_launches'] * 1e3
print(f"n={n} d={d} grid={s.stats()['grid']}")
print(f"objective-only pass {timed(lambda: s.objective()):8.1f} us")
for K in (0, 1, 3):
    print(f"step K={K}            {timed(lambda: s.step(1.0 / n, K)):8.1f} us")
print(f"gpm                 {timed(lambda: s.gpm_run(1)):8.1f} us")
