"""Per-iteration run(T) time of the current build under NSRGS_UNITS settings (tail_panels,unit_div,unit_min)."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(__file__))
from ab_tree import CHILD  # noqa: E402  (child program text)
cfgs = sys.argv[1].split(",")
settings = sys.argv[2:]
for cfg in cfgs:
    T = {"c1": 200, "c2": 200, "m2": 100}.get(cfg, 30)
    for rnd in range(2):
        for st in settings:
            env = dict(os.environ, NSRGS_UNITS=st)
            p = subprocess.run([sys.executable, "-c", CHILD, cfg, str(T)], env=env, capture_output=True, text=True)
            print(cfg, st, p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-200:], flush=True)
