"""B200-native NS-RGS (arxiv 2604.07372): the data-parallel hot path behind a C-ABI.

    from paper_2604_07372_b200 import nsrgs
    s = nsrgs.Solver(n, d)            # one context per GPU
    Z = s.generate(seed, sigma)       # synthetic instance on the device
    s.init_spectral(seed)             # spectral init
    trace = s.run(T, 1.0 / n, K)      # Algorithm 2
    rel, dF, mse = s.alignment_error(Z)

The compute path is libnsrgs.so (CUDA, sm_100a); see include/nsrgs.h.
"""
