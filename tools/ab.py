"""A/B timing in one process: dense vs symmetric pass on the same instance, alternating."""
import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2604_07372_b200 import nsrgs

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
n, d, c, K = {"c2": (2000, 3, None, 5), "c3": (20000, 5, 0.3, 5), "c4": (12000, 10, 0.2, 6)}[cfg]
sigma = 0.5 if c is None else c * np.sqrt(n) / d
s = nsrgs.Solver(n, d)
s.generate(0, sigma, want_Z=False)
s.init_spectral(0, 30, 1e-5, allow_unconverged=True)
modes = [False, True] if d <= 6 else [False]
res = {m: [] for m in modes}
clk = {m: [] for m in modes}
try:
    import pynvml
    pynvml.nvmlInit()
    hnd = pynvml.nvmlDeviceGetHandleByIndex(0)
    getclk = lambda: pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM)
    getpw = lambda: pynvml.nvmlDeviceGetPowerUsage(hnd) / 1000.0
except Exception:
    getclk = lambda: -1
    getpw = lambda: -1
for rep in range(4):
    for m in modes:
        s.set_symmetric(m)
        s.run(3, 1.0 / n, K, trace=False)
        s.reset_stats(True)
        s.run(5, 1.0 / n, K, trace=False)
        c0, p0 = getclk(), getpw()
        s.run(5, 1.0 / n, K, trace=False)
        clk[m].append((c0, round(p0)))
        st = s.stats()
        res[m].append(st["panel_ms_total"] / st["panel_launches"])
for m in modes:
    v = res[m]
    print(f"{cfg} {'sym' if m else 'dense'}: ms/pass min {min(v):.3f} med {np.median(v):.3f}  all {[round(x, 3) for x in v]}  (sm MHz, W) {clk[m]}")
