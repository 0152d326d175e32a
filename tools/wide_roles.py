"""Per-role wait / busy cycles of the tcgen05 wide pass (wide_tc.cu debug counters, one launch).
Usage: python tools/wide_roles.py n d [K [warm-up iterations]]"""
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2604_07372_b200 import nsrgs
n, d = int(sys.argv[1]), int(sys.argv[2]); K = int(sys.argv[3]) if len(sys.argv) > 3 else 1
s = nsrgs.Solver(n, d); s.generate(0, 0.1, want_Z=False)
rng = np.random.default_rng(0)
X = np.linalg.qr(rng.standard_normal((n, d, d)))[0].astype(np.float32)
s.set_X(X); s.step(1.0 / n, K)
s.reset_stats(True)
for _ in range(5):
    s.set_X(X); s.step(1.0 / n, K)
st = s.stats(); us = st['panel_ms_total'] / st['panel_launches'] * 1e3
if len(sys.argv) > 4:   # sustained: the counters of a launch at power-capped clocks
    s.run(int(sys.argv[4]), 1.0 / n, K)
s.set_X(X); s.debug_timestamps(1); s.step(1.0 / n, K); ts = s.debug_timestamps(0)[0].astype(np.float64)
names = ["producer total", "producer wait empty", "split wait full", "split wait xfree", "split total",
         "mma wait full+split", "mma wait acc/seg free", "mma total", "drain wait acc_full", "drain stream total",
         "drain seg epilogue/slot", "shared epilogue", "final reduce"]
N = n * d
print(f"n={n} d={d} K={K} grid={st['grid']} pass {us:.1f} us  {4 * N * N / us / 1e3:.0f} GB/s")
for i, nm in enumerate(names):
    c = ts[:, i]
    print(f"  {nm:26s} mean {c.mean() / 1e3:9.1f} kcyc   min {c.min() / 1e3:9.1f}   max {c.max() / 1e3:9.1f}")
