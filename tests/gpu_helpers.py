"""Helpers shared by the -m gpu parity tests: oracle-side per-node step (sampled parity) and
rotation-aligned comparison.  Everything here calls only oracle/ (NumPy fp64)."""
import numpy as np

from oracle import nsrgs as ons


def rel_fro(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - np.asarray(b, np.float64)) / np.linalg.norm(b))


def rel_mod_rotation(X, Xref):
    """min_Q ||X - Xref Q||_F / ||Xref||_F (Q* = sgn(Xref^T X))."""
    d = X.shape[-1]
    Xs, Rs = np.asarray(X, np.float64).reshape(-1, d), np.asarray(Xref, np.float64).reshape(-1, d)
    Q = ons.sgn(Rs.T @ Xs)
    return float(np.linalg.norm(Xs - Rs @ Q) / np.linalg.norm(Rs))


def oracle_node_step(A_rows, X, nodes, mu, Ts):
    return ons.step_rows(A_rows, X, nodes, mu, Ts)


def oracle_iterate_near(Z, noise, seed):
    """An oracle-side iterate X = sgn(Z_i + noise * N(0,1)) (blockwise), fp64."""
    rng = np.random.default_rng(seed)
    return ons.sgn(Z + noise * rng.standard_normal(Z.shape))


def max_block_err(X, Xref):
    """max_i ||X_i - Xref_i||_F / ||Xref_i||_F over the n d x d blocks (a per-block bound: a
    single bad block cannot hide inside a global relative norm)."""
    d = X.shape[-1]
    a = np.asarray(X, np.float64).reshape(-1, d, d)
    b = np.asarray(Xref, np.float64).reshape(-1, d, d)
    return float(np.max(np.linalg.norm(a - b, axis=(1, 2)) / np.linalg.norm(b, axis=(1, 2))))


def group_map(solvers, fn):
    """Run fn(solver) for every rank of an in-process rank group, one host thread per rank (every
    library call is collective; ctypes releases the GIL).  Returns the per-rank results in rank
    order; re-raises the first rank's exception."""
    import threading

    out, err = [None] * len(solvers), [None] * len(solvers)

    def body(r):
        try:
            out[r] = fn(solvers[r])
        except BaseException as e:  # noqa: BLE001 - re-raised below
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(len(solvers))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return out
