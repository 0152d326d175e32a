"""Per-step error of the wide-pass variants vs the fp64 oracle across n (test infrastructure:
imports oracle/).  Usage: python tools/wide_err.py"""
import os, sys, subprocess
sys.path.insert(0, '.')
if len(sys.argv) > 1:
    import numpy as np
    from paper_2604_07372_b200 import nsrgs
    from oracle import instance as inst
    from oracle import nsrgs as ons
    from tests.gpu_helpers import oracle_iterate_near
    n, d = int(sys.argv[1]), int(sys.argv[2])
    s = nsrgs.Solver(n, d); s.generate(4, 0.3, want_Z=False)
    Z = inst.ground_truth(4, n, d); A = inst.measurement_matrix(4, Z, 0.3)
    X = oracle_iterate_near(Z, 0.1, 2).astype(np.float32)
    s.set_X(X); f = s.step(1.0 / n, 1)
    Xo, _, _ = ons.step(A, X.astype(np.float64), 1.0 / n, 1)
    e = np.linalg.norm(s.get_X() - Xo) / np.linalg.norm(Xo)
    fo = ons.objective(A, X.astype(np.float64))
    print(f"variant={os.environ.get('NSRGS_WIDE_MMA','0')} n={n} d={d} step rel {e:.2e} obj rel {abs(f-fo)/fo:.2e}", flush=True)
    sys.exit(0)
for n, d in [(100, 25), (300, 25), (700, 25), (1500, 25), (700, 16), (1500, 12)]:
    for v in ("1", "2"):
        subprocess.run([sys.executable, __file__, str(n), str(d)], env={**os.environ, "NSRGS_WIDE_MMA": v}, timeout=300)
