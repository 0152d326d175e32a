import sys; sys.path.insert(0,'.')
from paper_2604_07372_b200 import nsrgs
for d,n in [(25,500),(5,20000),(3,2000)]:
    s=nsrgs.Solver(n,d); s.generate(0,0.1 if d==25 else 1.0)
    print(d, n, 'sweeps', s.init_spectral(0,200,1e-6,allow_unconverged=True))
