"""NS-RGS oracle — plain, slow, fp64 CPU reference.  TEST INFRASTRUCTURE ONLY.

This package defines what the B200 path must compute.  It follows PAPER.md
(arxiv 2604.07372, "NS-RGS: Newton-Schulz Based Riemannian Gradient Method for
Orthogonal Group Synchronization") step by step, in the paper's order and
notation, with NumPy float64 arithmetic.  Library primitives (matmul, svd, qr,
eigh) serve as single steps; there is no blocking, fusion or reordering beyond
what the paper's definitions state.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything from here.
The product path (``paper_2604_07372_b200`` + ``libnsrgs.so``) never imports,
links or executes this package, and this package never imports the product.
The two share no code: the oracle re-implements the counter-based instance
generator (Philox4x32-10 + Box-Muller, see ``instance.py``) independently of
the CUDA generator.

Modules
-------
instance  Philox4x32-10 counter RNG, Box-Muller normals, ground truth Z and
          measurement matrix A = ZZ^T + sigma W (§1.1,
          :225-230 Eq. def:measurements).
nsrgs     Algorithm 1 (Newton-Schulz), tangent projection
          (PAPER.md:213), Algorithm 2 (NS-RGS), spectral
          initialisation, the SVD-retraction variant,
          objective F, brute-force loop versions.
metrics   d_F, Rel.Err., MSE
          (PAPER.md:369-372).

Parity status: every function here is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against something other than itself (closed forms,
paper-printed values, brute force, invariants).  See DESIGN.md §"Oracle pins".
"""
