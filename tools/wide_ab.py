"""A/B of the wide-pass variants (NSRGS_WIDE_MMA = 0 broadcast, 1 3xTF32) on one box:
mean panel pass over 20 iterations after spectral init.  Usage: python tools/wide_ab.py"""
import os, subprocess, sys
if len(sys.argv) > 1:
    sys.path.insert(0, '.')
    from paper_2604_07372_b200 import nsrgs
    n, d = int(sys.argv[1]), int(sys.argv[2])
    s = nsrgs.Solver(n, d); s.generate(0, 0.1)
    s.init_spectral(0, 200, 1e-6, allow_unconverged=True)
    s.run(5, 1.0 / n, 1)
    s.reset_stats(True)
    s.run(20, 1.0 / n, 1)
    st = s.stats(); ms = st['panel_ms_total'] / st['panel_launches']; N = n * d
    print(f"variant={os.environ.get('NSRGS_WIDE_MMA', '0')} d={d} n={n} pass {ms*1e3:.1f} us  {4*N*N/ms/1e6:.0f} GB/s", flush=True)
    sys.exit(0)
for n, d in [(500, 25), (2000, 25), (4000, 25), (7000, 25), (1000, 16), (8000, 16)]:
    for v in ("1", "2"):
        subprocess.run([sys.executable, __file__, str(n), str(d)], env={**os.environ, "NSRGS_WIDE_MMA": v}, timeout=300)
