"""P > 1 against the fp64 oracle: sharded ranks with REAL collectives on one GPU.

Each rank is an emulated context (NSRGS_EMULATE_RANKS=1: its own row shard of A generated from
the per-(i,j) counters, its own X buffers, its own stream) joined into an in-process rank group
(nsrgs_debug_group): the all-reduces of fp64 partials (||A||_F^2, the init's Gram matrices and
subspace change, the objective partials) and the X all-gather of every iteration exchange real
data between the ranks, with host barriers between the phases, so no kernel ever waits for
another rank's kernel on the shared GPU.  Every library call is issued for all ranks at once,
one host thread per rank (tests/gpu_helpers.group_map).  This is the multi-GPU program of
SURVEY §8(e) (row-block sharding by node, Jacobi update, collectives after each pass) run
rank for rank; results are compared with the fp64 oracle (oracle/), not with the library's own
single-GPU output.

Sizes satisfy (n / P) d sizeof(dtype) % 16 == 0 (TMA row segments of each rank slice).
"""
import numpy as np
import pytest

from oracle import instance as inst
from oracle import metrics as mt
from oracle import nsrgs as ons

from tests.gpu_helpers import group_map, max_block_err, rel_fro, rel_mod_rotation

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nsrgs():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_07372_b200 import nsrgs as mod

    return mod


def _group(nsrgs, n, d, world, dtype=None):
    import torch

    dt = nsrgs.F32 if dtype is None else dtype
    ranks = [nsrgs.Solver(n, d, dtype=dt, rank=r, world=world, stream=torch.cuda.Stream()) for r in range(world)]
    nsrgs.link_group(ranks)
    return ranks


def _close(ranks):
    for s in ranks:
        s.close()


def _same_on_all_ranks(vals):
    for v in vals[1:]:
        assert np.array_equal(np.asarray(v), np.asarray(vals[0]))
    return vals[0]


@pytest.mark.parametrize("n,d,world,dtype", [(1920, 3, 2, "f32"), (1920, 3, 8, "f32"), (1280, 5, 4, "f32"),
                                             (1280, 5, 8, "f32"), (640, 10, 8, "f32"), (320, 16, 4, "f32"),
                                             (400, 4, 4, "f64")])
def test_group_pipeline_matches_oracle(nsrgs, monkeypatch, n, d, world, dtype):
    """generate -> init_spectral -> run(T) -> objective / objective_fp64 -> alignment_error ->
    GPM -> solve, all sharded over `world` ranks, against the oracle on the same instance."""
    monkeypatch.setenv("NSRGS_EMULATE_RANKS", "1")
    seed, sigma, K, T = 11, 0.3 * np.sqrt(n) / d, 5, 30
    f64 = dtype == "f64"
    ranks = _group(nsrgs, n, d, world, nsrgs.F64 if f64 else nsrgs.F32)
    Zs = group_map(ranks, lambda s: s.generate(seed, sigma))
    Zg = _same_on_all_ranks(Zs)
    Z = inst.ground_truth(seed, n, d)
    A = inst.measurement_matrix(seed, Z, sigma, dtype=np.float64 if f64 else np.float32).astype(np.float64)
    # ||A||_F^2: every rank's shard sum, all-reduced
    fro = [s.stats()["a_fro2"] for s in ranks]
    assert all(f == fro[0] for f in fro)
    assert abs(fro[0] - np.sum(A * A)) <= 1e-12 * np.sum(A * A)

    # spectral init: Gram all-reduce + Y all-gather every sweep; X^0 modulo the global rotation
    sw = group_map(ranks, lambda s: s.init_spectral(seed, 400, 1e-12 if f64 else 1e-6))
    assert len(set(sw)) == 1
    X0g = _same_on_all_ranks(group_map(ranks, lambda s: s.get_X()))
    X0o, _, _ = ons.spectral_init(A, d, "subspace", Y0=inst.initial_subspace(seed, n, d), tol=1e-12)
    assert rel_mod_rotation(X0g, X0o) <= (1e-9 if f64 else 1e-4)

    # T iterations from the oracle's X^0 (strict parity, no rotation freedom)
    X0 = X0o.astype(ranks[0].np_dtype)
    group_map(ranks, lambda s: s.set_X(X0))
    trs = group_map(ranks, lambda s: s.run(T, 1.0 / n, K, trace=True))
    tr = _same_on_all_ranks(trs)
    XT = _same_on_all_ranks(group_map(ranks, lambda s: s.get_X()))
    Xo, Fo = X0.astype(np.float64), []
    for _ in range(T):
        Fo.append(ons.objective_expanded(A, Xo))
        Xo, _, _ = ons.step(A, Xo, 1.0 / n, K)
    tol_x = 1e-11 if f64 else 1e-5
    assert rel_fro(XT, Xo) <= tol_x                                  # north star: 1e-4 after T
    assert max_block_err(XT, Xo) <= (1e-10 if f64 else 1e-4)
    assert np.max(np.abs(tr - np.array(Fo)) / np.abs(Fo)) <= (1e-10 if f64 else 2e-6)

    # objective of the current iterate (one extra pass, partials all-reduced)
    XTd = XT.astype(np.float64)
    Fx = ons.objective_expanded(A, XTd)
    F = _same_on_all_ranks(group_map(ranks, lambda s: s.objective()))
    assert abs(F - Fx) <= (1e-10 if f64 else 2e-6) * abs(Fx)
    if not f64:
        F64 = _same_on_all_ranks(group_map(ranks, lambda s: s.objective_fp64()))
        assert abs(F64 - Fx) <= 1e-12 * abs(Fx)

    # alignment metrics (replicated X, no collective) on every rank
    met = _same_on_all_ranks(group_map(ranks, lambda s: np.array(s.alignment_error(Zg))))
    mo = np.array(mt.alignment_error(XTd, Z))
    assert np.all(np.abs(met - mo) <= 1e-6 * mo)

    # GPM on the same sharded pass: X_i <- sgn(B_i)
    group_map(ranks, lambda s: s.gpm_run(3, trace=False))
    Xg = _same_on_all_ranks(group_map(ranks, lambda s: s.get_X()))
    Xgo = XTd
    for _ in range(3):
        Xgo = ons.gpm_step(A, Xgo)
    assert rel_fro(Xg, Xgo) <= (1e-11 if f64 else 1e-5)

    # paper protocol (R^t < 1e-8 stop, T_s = 1) from the oracle's X^0: the oracle's stopping iteration
    group_map(ranks, lambda s: s.set_X(X0))
    res = group_map(ranks, lambda s: s.solve("ns_rgs", max_iter=100, K=1, stop_tol=1e-8))
    its = [r[0] for r in res]
    assert len(set(its)) == 1
    Xso, it_o, _ = ons.solve_protocol(A, X0.astype(np.float64), 1.0 / n, 1, "ns_rgs", max_iter=100, tol=1e-8)
    assert its[0] == it_o, (its[0], it_o)
    Xs = _same_on_all_ranks(group_map(ranks, lambda s: s.get_X()))
    assert rel_fro(Xs, Xso) <= (1e-11 if f64 else 1e-5)
    _close(ranks)


@pytest.mark.parametrize("n,d,world,p", [(1280, 5, 4, 0.5), (960, 3, 2, 0.3)])
def test_group_block_sparse_matches_oracle(nsrgs, monkeypatch, n, d, world, p):
    """p < 1 on block-sparse shards: the per-rank BSR generator (observed
    pairs from the per-(i,j) counters), the sharded gather pass and its collectives."""
    monkeypatch.setenv("NSRGS_EMULATE_RANKS", "1")
    seed, sigma, K, T = 5, 1.0, 5, 20
    ranks = _group(nsrgs, n, d, world)
    group_map(ranks, lambda s: s.generate(seed, sigma, want_Z=False, p=p, storage="bsr"))
    assert all(s.stats()["bsr"] == 1 for s in ranks)
    Z = inst.ground_truth(seed, n, d)
    A = inst.measurement_matrix(seed, Z, sigma, p=p).astype(np.float64)
    fro = ranks[0].stats()["a_fro2"]
    assert abs(fro - np.sum(A * A)) <= 1e-12 * np.sum(A * A)
    X0o, _, _ = ons.spectral_init(A, d, "subspace", Y0=inst.initial_subspace(seed, n, d), tol=1e-12)
    group_map(ranks, lambda s: s.init_spectral(seed, 400, 1e-6))
    X0g = _same_on_all_ranks(group_map(ranks, lambda s: s.get_X()))
    assert rel_mod_rotation(X0g, X0o) <= 1e-4
    X0 = X0o.astype(np.float32)
    group_map(ranks, lambda s: s.set_X(X0))
    mu = 1.0 / (n * p)
    tr = _same_on_all_ranks(group_map(ranks, lambda s: s.run(T, mu, K, trace=True)))
    XT = _same_on_all_ranks(group_map(ranks, lambda s: s.get_X()))
    Xo = ons.run(A, X0.astype(np.float64), T, mu, K)
    assert rel_fro(XT, Xo) <= 1e-5 and max_block_err(XT, Xo) <= 1e-4
    assert abs(tr[0] - ons.objective_expanded(A, X0.astype(np.float64))) <= 2e-6 * abs(tr[0])
    _close(ranks)


def test_group_equals_single_gpu_schedule(nsrgs, monkeypatch):
    """The sharded run differs from the single-GPU run only by fp32 summation order (the rank
    slices of the column sweep), so the two agree to the step bar after T iterations."""
    n, d, world, K, T = 1280, 5, 4, 5, 10
    monkeypatch.setenv("NSRGS_NO_COOP", "1")
    full = nsrgs.Solver(n, d)
    full.generate(2, 1.5, want_Z=False)
    Z = inst.ground_truth(2, n, d)
    X = ons.sgn(Z + 0.05 * np.random.default_rng(1).standard_normal(Z.shape)).astype(np.float32)
    full.set_X(X)
    tr1 = full.run(T, 1.0 / n, K)
    X1 = full.get_X()
    full.close()
    monkeypatch.setenv("NSRGS_EMULATE_RANKS", "1")
    ranks = _group(nsrgs, n, d, world)
    group_map(ranks, lambda s: s.generate(2, 1.5, want_Z=False))
    group_map(ranks, lambda s: s.set_X(X))
    trP = _same_on_all_ranks(group_map(ranks, lambda s: s.run(T, 1.0 / n, K)))
    XP = _same_on_all_ranks(group_map(ranks, lambda s: s.get_X()))
    assert rel_fro(XP, X1) <= 1e-6
    assert np.max(np.abs(trP - tr1) / np.abs(tr1)) <= 1e-6
    _close(ranks)


def test_group_rejects_mismatched_ranks(nsrgs, monkeypatch):
    monkeypatch.setenv("NSRGS_EMULATE_RANKS", "1")
    a = nsrgs.Solver(64, 2, rank=0, world=2)
    b = nsrgs.Solver(64, 3, rank=1, world=2)
    with pytest.raises(nsrgs.NSRGSError) as e:
        nsrgs.link_group([a, b])
    assert e.value.name == "INVALID_ARG"
    c = nsrgs.Solver(64, 2, rank=1, world=2)
    nsrgs.link_peers([a, c])                      # P2P-linked ranks cannot join a host-barrier group
    with pytest.raises(nsrgs.NSRGSError):
        nsrgs.link_group([a, c])
    for s in (a, b, c):
        s.close()
