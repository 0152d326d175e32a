"""A/B of two builds (directories with a built paper_2604_07372_b200 package), interleaved in one
session: per-iteration time of run(T) (device events) with the SM clock sampled alongside.
usage: python tools/ab_tree.py OLD_DIR NEW_DIR c3,c4 [rounds] [plain]"""
import json, os, subprocess, sys

CHILD = r'''
import sys, json, threading, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2604_07372_b200 import nsrgs
import pynvml
cfg, T = sys.argv[1], int(sys.argv[2])
n, d, c, K = {"c1": (100, 3, None, 3), "c2": (2000, 3, None, 5), "c3": (20000, 5, 0.3, 5), "c4": (12000, 10, 0.2, 6),
              "m2": (3000, 3, None, 5)}[cfg]
sigma = 0.5 if c is None else c * np.sqrt(n) / d
s = nsrgs.Solver(n, d)
s.generate(0, sigma, want_Z=False)
rng = np.random.default_rng(0)
s.set_X(np.linalg.qr(rng.standard_normal((n, d, d)))[0].astype(np.float32))
s.run(3, 1.0 / n, K, trace=False)
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
clk, stop = [], [False]
def samp():
    while not stop[0]:
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)); time.sleep(0.01)
th = threading.Thread(target=samp); th.start()
st = torch.cuda.current_stream(); res = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); s.run(T, 1.0 / n, K); e1.record(st); torch.cuda.synchronize()
    res.append(1000 * e0.elapsed_time(e1) / T)
stop[0] = True; th.join()
print(json.dumps({"us": round(float(np.median(res)), 2), "sm_mhz": int(np.median(clk)) if clk else None}))
'''

if __name__ == "__main__":
    old, new, cfgs = sys.argv[1], sys.argv[2], sys.argv[3].split(",")
    rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    env = dict(os.environ)
    if len(sys.argv) > 5 and sys.argv[5] == "plain":
        env["NSRGS_NO_COOP"] = "1"
    for cfg in cfgs:
        T = {"c1": 200, "c2": 200, "m2": 100}.get(cfg, 30)
        out = {"old": [], "new": []}
        for r in range(rounds):
            for name, path in (("old", old), ("new", new)):
                p = subprocess.run([sys.executable, "-c", CHILD, cfg, str(T)], cwd=path, env=env, capture_output=True, text=True)
                line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-300:]
                out[name].append(line)
        print(cfg, json.dumps(out))
