import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2604_07372_b200 import nsrgs
for d, n in [(25, 500), (25, 4000), (16, 4000)]:
    s = nsrgs.Solver(n, d); s.generate(0, 0.1)
    sw = s.init_spectral(0, 200, 1e-6, allow_unconverged=True)
    s.reset_stats(True)
    s.run(10, 1.0 / n, 1)
    st = s.stats(); ms = st['panel_ms_total'] / st['panel_launches']; N = n * d
    print(f"d={d} n={n} sweeps={sw} grid={st['grid']} stages={st['stages']} pass ms {ms:.4f}  GB/s {4*N*N/ms/1e6:.0f}")
