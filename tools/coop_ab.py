"""Whole run(T) wall time on the device: cooperative multi-iteration launch vs per-iteration launches."""
import os, sys, subprocess, json
import numpy as np
if len(sys.argv) > 2 and sys.argv[2] == "child":
    sys.path.insert(0, ".")
    import torch
    from paper_2604_07372_b200 import nsrgs
    cfg = sys.argv[1]
    n, d, c, K = {"c1": (100, 3, None, 3), "c2": (2000, 3, None, 5), "m1": (1500, 3, None, 5), "m2": (3000, 3, None, 5), "m3": (2000, 5, None, 5), "c3": (20000, 5, 0.3, 5), "c4": (12000, 10, 0.2, 6)}[cfg]
    sigma = 0.5 if c is None else c * np.sqrt(n) / d
    s = nsrgs.Solver(n, d)
    s.generate(0, sigma, want_Z=False)
    s.init_spectral(0, 30, 1e-5, allow_unconverged=True)
    T = 100
    s.run(T, 1.0 / n, K)
    st = torch.cuda.current_stream()
    res = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st); tr = s.run(T, 1.0 / n, K); e1.record(st); torch.cuda.synchronize()
        res.append(e0.elapsed_time(e1) / T)
    print(json.dumps({"cfg": cfg, "us_per_iter": [round(1000 * r, 2) for r in res], "F_last": tr[-1]}))
else:
    for cfg in sys.argv[1].split(","):
        for coop in ("0", "1"):
            env = dict(os.environ, NSRGS_NO_COOP="0" if coop == "1" else "1")
            out = subprocess.run([sys.executable, __file__, cfg, "child"], env=env, capture_output=True, text=True)
            print("coop" if coop == "1" else "plain", out.stdout.strip(), out.stderr.strip()[-300:])
