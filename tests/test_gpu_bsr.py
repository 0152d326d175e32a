"""GPU parity of the block-sparse (BSR) storage path — SURVEY §8(f) row 2, incomplete
observations (§4.1; step size mu = 1/(np), :324).

* generator: every stored block is bitwise the dense generator's block, the edge set is the
  oracle's (exact decision) and values are within 1 fp32 ulp of the oracle's;
* one NS-RGS step / GPM step / objective from a shared iterate: relative Frobenius <= 1e-6
  against the fp64 oracle (fp32 arithmetic, same bar as the dense pass);
* spectral init + T iterations end to end modulo the global rotation <= 1e-4, alignment
  error within 1e-3 relative (north-star bars);
* sharded ranks (emulated one after another on one GPU), a caller-attached BSR matrix with
  ragged, unpadded rows (including empty ones), the Table 1 p < 1 cells, the bytes per pass,
  and sampled parity at the bench size (n = 20000, d = 5, p = 0.5).
"""
import numpy as np
import pytest

from oracle import instance as inst
from oracle import metrics as mt
from oracle import nsrgs as ons
from tests.gpu_helpers import oracle_iterate_near, rel_fro, rel_mod_rotation

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsrgs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_07372_b200 import nsrgs as mod

    return mod


def expand(rowptr, col, vals, n, d):
    """Dense rows of a BSR shard (host, fp64)."""
    nl = len(rowptr) - 1
    A = np.zeros((nl * d, n * d))
    for il in range(nl):
        for b in range(rowptr[il], rowptr[il + 1]):
            j = col[b]
            A[il * d:(il + 1) * d, j * d:(j + 1) * d] += vals[b]
    return A


@pytest.mark.parametrize("n,d,p", [(300, 3, 0.5), (200, 5, 0.8), (120, 10, 0.3), (64, 25, 0.5), (100, 5, 1.0),
                                   (33, 7, 0.6), (40, 2, 0.05)])
def test_bsr_generator(nsrgs, n, d, p):
    sigma, seed = 0.6, 13
    sd = nsrgs.Solver(n, d)
    sd.generate(seed, sigma, want_Z=False, p=p)
    Ad = sd.copy_A_rows(0, n * d).astype(np.float64)
    fro_d = sd.stats()["a_fro2"]
    sd.close()
    s = nsrgs.Solver(n, d)
    Zg = s.generate(seed, sigma, p=p, storage="bsr")
    rowptr, col, vals = s.get_A_bsr()
    st = s.stats()
    assert st["bsr"] == 1 and st["bsr_nnzb"] == len(col)
    # structure: rows padded to multiples of 4, observed columns ascending, padding = own node, zeros
    assert rowptr[0] == 0 and np.all(np.diff(rowptr) % 4 == 0)
    Z = inst.ground_truth(seed, n, d)
    for i in range(n):
        c = col[rowptr[i]:rowptr[i + 1]]
        v = vals[rowptr[i]:rowptr[i + 1]]
        obs = np.flatnonzero(inst.observed(seed, np.minimum(i, np.arange(n)), np.maximum(i, np.arange(n)), p)
                             | (p >= 1.0))
        obs = obs[obs != i]
        m = len(obs)
        assert np.array_equal(c[:m], obs)                        # the oracle's edge set, ascending
        pad = obs[-1] if m else i                                # padding keeps the row sorted
        assert np.all(c[m:] == pad) and np.all(v[m:] == 0.0) and len(c) - m < 4
    A = expand(rowptr, col, vals, n, d)
    assert np.array_equal(A, Ad)                                 # bitwise the dense generator
    Ao = inst.measurement_matrix(seed, Z, sigma, p=p)
    ulp = np.spacing(np.abs(Ao).astype(np.float32)).astype(np.float64)
    assert np.all(np.abs(A - Ao) <= ulp)
    assert abs(st["a_fro2"] - fro_d) <= 1e-12 * fro_d
    assert np.max(np.abs(Zg.astype(np.float64) - Z)) <= 2e-7
    s.close()


@pytest.mark.parametrize("n,d,sigma,p,K", [(300, 3, 0.5, 0.5, 3), (160, 5, 0.4, 0.8, 5), (90, 10, 0.3, 0.3, 6),
                                           (70, 6, 0.5, 1.0, 4), (45, 9, 0.2, 0.7, 2), (40, 25, 0.1, 0.5, 1),
                                           (30, 12, 0.3, 0.6, 3)])
def test_bsr_step_gpm_objective(nsrgs, n, d, sigma, p, K):
    s = nsrgs.Solver(n, d)
    s.generate(5, sigma, want_Z=False, p=p, storage="bsr")
    Z = inst.ground_truth(5, n, d)
    A = inst.measurement_matrix(5, Z, sigma, p=p)
    X = oracle_iterate_near(Z, 0.2, 3).astype(np.float32)
    Xd = X.astype(np.float64)
    eta = 1.0 / (n * p)
    s.set_X(X)
    f = s.step(eta, K)
    Xo, _, _ = ons.step(A, Xd, eta, K)
    assert rel_fro(s.get_X(), Xo) <= 1e-6
    fo = ons.objective(A, Xd)
    assert abs(f - fo) <= 2e-6 * abs(fo)
    s.set_X(X)
    assert abs(s.objective() - fo) <= 2e-6 * abs(fo)
    s.set_X(X)
    s.gpm_run(1)
    assert rel_fro(s.get_X(), ons.gpm_step(A, Xd)) <= 1e-6
    s.close()


@pytest.mark.parametrize("n,d,p,ring", [(3000, 5, 0.9, "1"), (2000, 3, 0.8, "1"), (1000, 2, 1.0, "1"),
                                         (700, 6, 0.75, "1"), (500, 4, 1.0, "1"), (3000, 5, 0.5, "8"),
                                         (900, 4, 0.35, "8"), (2000, 3, 0.5, "8"), (600, 6, 0.1, "8"),
                                         (800, 5, 0.6, "4")])
def test_bsr_slab_pass_equals_gather_pass(nsrgs, monkeypatch, n, d, p, ring):
    """The slab pass (sorted rows: column-group X slabs shared by the CTA's rows) and the
    per-block gather pass multiply the same blocks in the same per-lane order: identical X^{t+1};
    the objective partials differ only by the fp64 CTA grouping."""
    sigma, K = 0.4, 3
    X = oracle_iterate_near(inst.ground_truth(12, n, d), 0.2, 4).astype(np.float32)
    out = []
    for slab in (ring, "0"):   # "1": the default choice (the 4-slot ring at p >= 0.75), "4"/"8": forced ring
        monkeypatch.setenv("NSRGS_BSR_SLAB", slab)
        s = nsrgs.Solver(n, d)
        s.generate(12, sigma, want_Z=False, p=p, storage="bsr")
        assert s.stats()["bsr_slab"] == (slab != "0")
        s.set_X(X)
        f = s.step(1.0 / (n * p), K)
        out.append((s.get_X(), f))
        s.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert abs(out[0][1] - out[1][1]) <= 1e-12 * abs(out[1][1])
    if n <= 1000:
        A = inst.measurement_matrix(12, inst.ground_truth(12, n, d), sigma, p=p)
        Xo, _, _ = ons.step(A, X.astype(np.float64), 1.0 / (n * p), K)
        assert rel_fro(out[0][0], Xo) <= 1e-6


@pytest.mark.parametrize("n,d,p", [(3000, 5, 0.5), (2000, 3, 0.2), (800, 2, 0.6), (700, 6, 0.3), (500, 4, 0.05)])
def test_bsr_gather4_pass_equals_lsu_gather(nsrgs, monkeypatch, n, d, p):
    """X records by TMA tile::gather4 vs the LSU gather: same blocks, same per-lane order ->
    identical X^{t+1}; against the oracle for the small cases."""
    sigma, K = 0.4, 3
    X = oracle_iterate_near(inst.ground_truth(13, n, d), 0.2, 4).astype(np.float32)
    out = []
    monkeypatch.setenv("NSRGS_BSR_SLAB", "0")   # the per-block gather family
    for g4 in ("1", "0"):
        monkeypatch.setenv("NSRGS_BSR_G4", g4)
        s = nsrgs.Solver(n, d)
        s.generate(13, sigma, want_Z=False, p=p, storage="bsr")
        assert s.stats()["bsr_g4"] == (g4 == "1")
        s.set_X(X)
        f = s.step(1.0 / (n * p), K)
        out.append((s.get_X(), f))
        s.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert abs(out[0][1] - out[1][1]) <= 1e-12 * abs(out[1][1])
    if n <= 1000:
        A = inst.measurement_matrix(13, inst.ground_truth(13, n, d), sigma, p=p)
        Xo, _, _ = ons.step(A, X.astype(np.float64), 1.0 / (n * p), K)
        assert rel_fro(out[0][0], Xo) <= 1e-6


def test_bsr_matches_dense_pass(nsrgs):
    """Same instance in both storages: T iterations agree to fp32 summation-order noise."""
    n, d, sigma, p, K, T = 500, 5, 0.6, 0.5, 5, 20
    X = oracle_iterate_near(inst.ground_truth(9, n, d), 0.3, 1).astype(np.float32)
    out = []
    for storage in ("dense", "bsr"):
        s = nsrgs.Solver(n, d)
        s.generate(9, sigma, want_Z=False, p=p, storage=storage)
        s.set_X(X)
        tr = s.run(T, 1.0 / (n * p), K)
        out.append((s.get_X(), tr, s.stats()["a_bytes_per_pass"]))
        s.close()
    assert rel_fro(out[1][0], out[0][0]) <= 1e-5
    assert np.all(np.abs(out[1][1] - out[0][1]) <= 1e-6 * np.abs(out[0][1]))
    # bytes per pass ~ p of the dense shard (values + 4-byte column index + row pointers)
    ratio = out[1][2] / out[0][2]
    assert abs(ratio - p * (1 + 4 / (4 * d * d))) <= 0.03


def test_bsr_end_to_end(nsrgs):
    n, d, sigma, p, K, T = 400, 3, 0.3, 0.5, 3, 40
    Z = inst.ground_truth(2, n, d)
    A = inst.measurement_matrix(2, Z, sigma, p=p)
    X0, _, _ = ons.spectral_init(A, d)
    Xo = ons.run(A, X0, T, 1.0 / (n * p), K)
    s = nsrgs.Solver(n, d)
    Zg = s.generate(2, sigma, p=p, storage="bsr")
    s.init_spectral(2, 300, 1e-6)
    s.run(T, 1.0 / (n * p), K, trace=False)
    assert rel_mod_rotation(s.get_X(), Xo) <= 1e-4
    rel = s.alignment_error(Zg)[0]
    assert abs(rel - mt.rel_err(Xo, Z)) <= 1e-3 * rel
    s.close()


@pytest.mark.parametrize("n,d,world", [(200, 5, 2), (96, 3, 4), (64, 12, 2)])
def test_bsr_sharded_rank_by_rank(nsrgs, monkeypatch, n, d, world):
    """Each rank generates only its node rows' blocks; the assembled step equals the single-GPU
    step and the oracle (ranks run one after another: NSRGS_EMULATE_RANKS, no collectives)."""
    monkeypatch.setenv("NSRGS_EMULATE_RANKS", "1")
    sigma, p, K = 0.5, 0.6, 3
    Z = inst.ground_truth(8, n, d)
    X = oracle_iterate_near(Z, 0.2, 2).astype(np.float32)
    eta = 1.0 / (n * p)
    full = nsrgs.Solver(n, d)
    full.generate(8, sigma, want_Z=False, p=p, storage="bsr")
    full.set_X(X)
    full.step(eta, K)
    Xref = full.get_X()
    rp_full, col_full, vals_full = full.get_A_bsr()
    full.close()
    nl = n // world
    Xsh = np.empty_like(X)
    for r in range(world):
        s = nsrgs.Solver(n, d, rank=r, world=world)
        s.generate(8, sigma, want_Z=False, p=p, storage="bsr")
        rp, col, vals = s.get_A_bsr()
        lo, hi = rp_full[r * nl], rp_full[(r + 1) * nl]
        assert np.array_equal(rp, rp_full[r * nl:(r + 1) * nl + 1] - lo)
        assert np.array_equal(col, col_full[lo:hi]) and np.array_equal(vals, vals_full[lo:hi])
        s.set_X(X)
        s.step(eta, K)
        Xsh[r * nl:(r + 1) * nl] = s.get_X()[r * nl:(r + 1) * nl]
        s.close()
    assert rel_fro(Xsh, Xref) <= 1e-6
    A = inst.measurement_matrix(8, Z, sigma, p=p)
    Xo, _, _ = ons.step(A, X.astype(np.float64), eta, K)
    assert rel_fro(Xsh, Xo) <= 1e-6


def test_bsr_attach_ragged(nsrgs):
    """A caller-owned BSR matrix: rows of arbitrary length (not padded, some empty), columns in
    any order; the pass must match the oracle on the dense expansion."""
    import torch

    n, d, K = 150, 4, 3
    rng = np.random.default_rng(4)
    Z = inst.ground_truth(3, n, d)
    A = inst.measurement_matrix(3, Z, 0.5, p=0.4)
    A[:4 * d] = 0.0                                  # nodes 0..3: no observations at all (rows and
    A[:, :4 * d] = 0.0                               # columns, keeping A symmetric)
    rowptr, cols, vals = [0], [], []
    for i in range(n):
        js = [j for j in range(n) if np.any(A[i * d:(i + 1) * d, j * d:(j + 1) * d] != 0.0)]
        rng.shuffle(js)
        for j in js:
            cols.append(j)
            vals.append(A[i * d:(i + 1) * d, j * d:(j + 1) * d])
        rowptr.append(len(cols))
    dev = torch.device("cuda", 0)
    t_rp = torch.tensor(rowptr, dtype=torch.int64, device=dev)
    t_col = torch.tensor(cols, dtype=torch.int32, device=dev)
    t_val = torch.tensor(np.array(vals), dtype=torch.float32, device=dev).contiguous()
    s = nsrgs.Solver(n, d)
    s.attach_A_bsr(t_rp, t_col, t_val)
    assert abs(s.stats()["a_fro2"] - np.sum(A * A)) <= 1e-9 * np.sum(A * A)
    X = oracle_iterate_near(Z, 0.2, 6).astype(np.float32)
    s.set_X(X)
    f = s.step(1.0 / (n * 0.4), K)
    Xo, _, _ = ons.step(A, X.astype(np.float64), 1.0 / (n * 0.4), K)
    assert rel_fro(s.get_X(), Xo) <= 1e-6
    assert abs(f - ons.objective(A, X.astype(np.float64))) <= 2e-6 * f
    # leaving block-sparse storage: a dense generate switches back
    s.generate(3, 0.5, want_Z=False)
    assert s.stats()["bsr"] == 0
    s.close()


def _table1_rows():
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "table1_relerr.txt")
    return [tuple(float(t) for t in l.split()) for l in open(path) if l.strip() and not l.startswith("#")]


def test_table1_p_lt_1_bsr(nsrgs):
    """PAPER.md Table 1 p = 0.8 and p = 0.5 cells (:351-359) through the block-sparse path
    (d = 25 wide BSR kernel), the paper's protocol: spectral init, T_s = 1, mu = 1/(np),
    stop at R^t < 1e-8 / MaxIter 100.  Printed Rel.Err. within 5 % (10-trial means)."""
    n, d = 500, 25
    for (_, _, p, sigma, rel_paper) in _table1_rows():
        if p >= 1.0:
            continue
        s = nsrgs.Solver(n, d)
        Zg = s.generate(0, sigma, p=p, storage="bsr")
        s.init_spectral(0, 200, 1e-6)
        it, tr = s.solve("ns_rgs", max_iter=100, eta=1.0 / (n * p), K=1, stop_tol=1e-8)
        assert it <= 100 and np.all(np.isfinite(tr))
        rel = s.alignment_error(Zg)[0]
        assert abs(rel - rel_paper) <= 0.05 * rel_paper, (p, sigma, rel, rel_paper)
        s.close()


def test_bsr_bench_size_sampled(nsrgs):
    """n = 20000, d = 5, p = 0.5 (the bench's block-sparse line): one step, sampled nodes
    (first, last, ragged interior) against the oracle on independently regenerated rows."""
    n, d, p, K = 20000, 5, 0.5, 5
    sigma = 0.3 * np.sqrt(n) / d
    s = nsrgs.Solver(n, d)
    s.generate(0, sigma, want_Z=False, p=p, storage="bsr")
    Z = inst.ground_truth(0, n, d)
    X = oracle_iterate_near(Z, 0.1, 9).astype(np.float32)
    s.set_X(X)
    s.step(1.0 / (n * p), K)
    Xg = s.get_X()
    nodes = np.array([0, 1, 7, 8191, 12345, n - 2, n - 1])
    R = inst.measurement_rows(0, Z, sigma, nodes, p=p)
    Xo = ons.step_rows(R, X.astype(np.float64), nodes, 1.0 / (n * p), K)
    assert rel_fro(Xg[nodes], Xo) <= 1e-6
    s.close()


def test_bsr_c4_size_sampled(nsrgs):
    """n = 12000, d = 10, p = 0.5 (two lanes per block, 16-block chunks): one step, sampled nodes
    against the oracle on independently regenerated rows."""
    n, d, p, K = 12000, 10, 0.5, 6
    sigma = 0.2 * np.sqrt(n) / d
    s = nsrgs.Solver(n, d)
    s.generate(1, sigma, want_Z=False, p=p, storage="bsr")
    Z = inst.ground_truth(1, n, d)
    X = oracle_iterate_near(Z, 0.1, 2).astype(np.float32)
    s.set_X(X)
    s.step(1.0 / (n * p), K)
    Xg = s.get_X()
    nodes = np.array([0, 5, 4097, 9999, n - 1])
    R = inst.measurement_rows(1, Z, sigma, nodes, p=p)
    Xo = ons.step_rows(R, X.astype(np.float64), nodes, 1.0 / (n * p), K)
    assert rel_fro(Xg[nodes], Xo) <= 1e-6
    s.close()


@pytest.mark.parametrize("n,d,p", [(2, 3, 1.0), (3, 5, 1.0), (4, 2, 0.5), (2, 25, 1.0)])
def test_bsr_tiny_instances(nsrgs, n, d, p):
    """Degenerate sizes: a row has 0-3 observed blocks plus padding; step and objective match the
    oracle (and an unobserved pair gives an all-zero row)."""
    s = nsrgs.Solver(n, d)
    s.generate(21, 0.3, want_Z=False, p=p, storage="bsr")
    Z = inst.ground_truth(21, n, d)
    A = inst.measurement_matrix(21, Z, 0.3, p=p)
    X = oracle_iterate_near(Z, 0.2, 1).astype(np.float32)
    s.set_X(X)
    f = s.step(1.0 / (n * p), 3)
    Xo, _, _ = ons.step(A, X.astype(np.float64), 1.0 / (n * p), 3)
    assert rel_fro(s.get_X(), Xo) <= 1e-6
    fo = ons.objective(A, X.astype(np.float64))
    assert abs(f - fo) <= 2e-6 * abs(fo) + 1e-9
    s.close()


def test_bsr_error_paths(nsrgs):
    """Block-sparse C-ABI contracts: F32 only, p in (0, 1], dense-only calls refuse while it is
    active, get_A_bsr refuses a dense A, and a dense generate switches back."""
    s = nsrgs.Solver(50, 3, nsrgs.F64)
    with pytest.raises(nsrgs.NSRGSError) as e:
        s.generate(1, 0.5, want_Z=False, p=0.5, storage="bsr")
    assert e.value.name == "INVALID_ARG"
    s.close()
    s = nsrgs.Solver(50, 3)
    for p in (0.0, 1.5, -0.1):
        with pytest.raises(nsrgs.NSRGSError) as e:
            s.generate(1, 0.5, want_Z=False, p=p, storage="bsr")
        assert e.value.name == "INVALID_ARG"
    s.generate(1, 0.5, want_Z=False)
    with pytest.raises(nsrgs.NSRGSError) as e:
        s.get_A_bsr()
    assert e.value.name == "STATE"
    s.generate(1, 0.5, want_Z=False, p=0.5, storage="bsr")
    for call in (lambda: s.copy_A_rows(0, 3), lambda: s.set_symmetric(True)):
        with pytest.raises(nsrgs.NSRGSError) as e:
            call()
        assert e.value.name == "STATE"
    assert s.stats()["bsr"] == 1
    s.generate(1, 0.5, want_Z=False)
    assert s.stats()["bsr"] == 0 and s.copy_A_rows(0, 3).shape == (3, 150)
    s.close()
