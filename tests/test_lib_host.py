"""Host-side checks of libnsrgs.so (no GPU): the library loads, exports every entry point
include/nsrgs.h declares, and its pure-host sharding plan / tile layout are right — including
a world_size-2 gloo emulation of the sharded iteration (row-block shards, per-rank X slices
exchanged with all_gather) against the single-process oracle."""
import ctypes as ct
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_07372_b200", "libnsrgs.so")


@pytest.fixture(scope="module")
def nsrgs():
    if not os.path.exists(LIB):
        from paper_2604_07372_b200.build import build

        build()
    from paper_2604_07372_b200 import nsrgs as mod

    return mod


def _header_functions():
    src = open(os.path.join(ROOT, "include", "nsrgs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(nsrgs_\w+)\s*\(", src)))


def test_exports_every_declared_symbol(nsrgs):
    names = _header_functions()
    assert len(names) >= 18
    lib = ct.CDLL(LIB)
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(nsrgs.EXPORTED)
    assert nsrgs.version() == 1


def _tile_index(c, k, d, rows_local, tpr):
    # the layout formula as written in include/nsrgs.h (nsrgs_plan comment)
    g, cl = divmod(c, rows_local)
    if d > 10:
        return (g * tpr * 32 + cl) * d + k
    j, o = divmod(cl, 128)
    b = (g * tpr + j) * d * 128
    if d % 2 == 1 and k == d - 1:
        return b + (d - 1) * 128 + o
    return b + (k - k % 2) * 128 + 2 * o + k % 2


@pytest.mark.parametrize("n,d,world", [(2, 2, 1), (100, 3, 1), (100, 3, 4), (43, 5, 1), (20000, 5, 8),
                                       (12000, 10, 8), (40000, 5, 4), (7, 9, 7), (500, 25, 4)])
def test_plan_partitions_rows(nsrgs, n, d, world):
    rows = []
    for r in range(world):
        p = nsrgs.plan(n, d, world, r)
        assert p["n_local"] * world == n and p["node0"] == r * p["n_local"]
        assert p["rows_local"] == p["n_local"] * d and p["row0"] == p["node0"] * d
        ct = 32 if d > 10 else 128
        assert p["col_tile"] == ct and p["tiles_per_rank"] == -(-p["rows_local"] // ct)
        assert p["x_slice_elems"] * world == p["x_elems"]
        assert p["x_slice_elems"] == p["tiles_per_rank"] * d * ct
        rows.append((p["row0"], p["row0"] + p["rows_local"]))
    assert rows[0][0] == 0 and rows[-1][1] == n * d
    assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))


@pytest.mark.parametrize("kw", [dict(n=1, d=3), dict(n=10, d=1), dict(n=10, d=17), dict(n=10, d=33), dict(n=10, d=3, world=3),
                                dict(n=10, d=3, world=2, rank=2)])
def test_plan_rejects(nsrgs, kw):
    with pytest.raises(nsrgs.NSRGSError):
        nsrgs.plan(kw["n"], kw["d"], kw.get("world", 1), kw.get("rank", 0))


@pytest.mark.parametrize("n,d,world", [(10, 3, 2), (43, 5, 1), (300, 7, 3), (64, 2, 4), (40, 25, 2), (30, 12, 1)])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_pack_layout(nsrgs, n, d, world, dt):
    N = n * d
    X = np.random.default_rng(0).standard_normal((N, d)).astype(dt)
    t = nsrgs.pack_host(X, n, d, world)
    p = nsrgs.plan(n, d, world, 0)
    ref = np.zeros(p["x_elems"], dtype=dt)
    for c in range(N):
        for k in range(d):
            ref[_tile_index(c, k, d, p["rows_local"], p["tiles_per_rank"])] = X[c, k]
    assert np.array_equal(t, ref)                        # padding entries are zero
    assert np.array_equal(nsrgs.unpack_host(t, n, d, world), X)


# ---------------------------------------------------------------------------- gloo world 2
def _sharded_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import instance as inst
        from oracle import nsrgs as ons
        from paper_2604_07372_b200 import nsrgs

        n, d, sigma, K, T = 24, 3, 0.6, 4, 6
        p = nsrgs.plan(n, d, world, rank)
        Z = inst.ground_truth(1, n, d)
        nodes = np.arange(p["node0"], p["node0"] + p["n_local"])
        A_rows = inst.measurement_rows(1, Z, sigma, nodes)               # this rank's shard only
        X, _, _ = ons.spectral_init(inst.measurement_matrix(1, Z, sigma), d)
        for _ in range(T):
            # own nodes from the own row shard (Algorithm 2 is Jacobi: reads X^t only)
            Xs = X.reshape(n * d, d)
            out = []
            for k, i in enumerate(nodes):
                Ai = A_rows[k * d:(k + 1) * d]
                G = (n - 1) * X[i] - Ai @ Xs
                out.append(ons.newton_schulz(X[i] - (1.0 / n) * ons.tangent_project(X[i], G), K))
            Xnew = X.copy()
            Xnew[nodes] = np.stack(out)
            # device layout: own slice = contiguous x_slice_elems of the tiled buffer
            tiled = nsrgs.pack_host(Xnew.reshape(n * d, d), n, d, world)
            sl = p["x_slice_elems"]
            mine = torch.from_numpy(tiled[rank * sl:(rank + 1) * sl].copy())
            parts = [torch.empty_like(mine) for _ in range(world)]
            dist.all_gather(parts, mine)                                   # = ncclAllGather in place
            full = torch.cat(parts).numpy()
            X = nsrgs.unpack_host(full, n, d, world).reshape(n, d, d)
        q.put((rank, X))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_iteration_matches_single_process(nsrgs):
    import multiprocessing as mp
    import socket

    from oracle import instance as inst
    from oracle import nsrgs as ons

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    n, d, sigma, K, T = 24, 3, 0.6, 4, 6
    Z = inst.ground_truth(1, n, d)
    A = inst.measurement_matrix(1, Z, sigma)
    X0, _, _ = ons.spectral_init(A, d)
    Xref = ons.run(A, X0, T, 1.0 / n, K)
    for r in range(2):
        assert np.max(np.abs(res[r] - Xref)) < 1e-12
