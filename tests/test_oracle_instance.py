"""Pins for oracle/instance.py (the instance definition)."""
import os

import numpy as np
import pytest
from scipy import stats

from oracle import instance as inst

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _kat():
    rows = []
    with open(os.path.join(GOLD, "philox4x32_10_kat.txt")) as f:
        for line in f:
            if line.strip() and not line.startswith("#"):
                rows.append([int(t, 16) for t in line.split()])
    return rows


@pytest.mark.parametrize("row", _kat())
def test_philox_known_answers(row):
    c0, c1, c2, c3, k0, k1 = row[:6]
    out = inst.philox4x32_10(c0, c1, c2, c3, k0, k1)
    assert [int(x) for x in out] == row[6:]


def test_uniform_open_interval_and_box_muller_moments():
    z = inst.block_normals(7, np.arange(4000), 3, inst.TAG_W, 50).ravel()   # 2e5 normals
    assert np.all(np.isfinite(z))
    assert abs(z.mean()) < 5.0 / np.sqrt(z.size)
    assert abs(z.var() - 1.0) < 5.0 * np.sqrt(2.0 / z.size)
    assert stats.kstest(z, "norm").pvalue > 1e-4
    # pairs from one call are independent-looking (no correlation between cos/sin halves)
    zz = inst.block_normals(9, np.arange(50000), 0, inst.TAG_W, 2)
    assert abs(np.corrcoef(zz[:, 0], zz[:, 1])[0, 1]) < 5.0 / np.sqrt(zz.shape[0])


def test_counter_streams_differ_by_every_field():
    a = inst.block_normals(1, 3, 4, inst.TAG_W, 9)
    for args in [(2, 3, 4, inst.TAG_W), (1, 4, 4, inst.TAG_W), (1, 3, 5, inst.TAG_W), (1, 3, 4, inst.TAG_Z)]:
        b = inst.block_normals(args[0], args[1], args[2], args[3], 9)
        assert not np.allclose(a, b)
    # high word of the seed enters key1
    assert not np.allclose(inst.block_normals(1, 0, 0, 1, 4), inst.block_normals(1 + (1 << 32), 0, 0, 1, 4))


@pytest.mark.parametrize("d", [2, 3, 5, 10])
def test_ground_truth_is_unique_qr_factor(d):
    n = 40
    Z = inst.ground_truth(3, n, d)
    G = inst.block_normals(3, np.arange(n), 0, inst.TAG_Z, d * d).reshape(n, d, d)
    for i in range(n):
        assert np.linalg.norm(Z[i].T @ Z[i] - np.eye(d)) < 1e-13
        R = Z[i].T @ G[i]                                   # G = Z R
        assert np.allclose(np.tril(R, -1), 0.0, atol=1e-12)
        assert np.all(np.diag(R) > 0)


def test_haar_first_moments():
    # Haar on O(d): E[Z] = 0, E[Z_ab^2] = 1/d, det = +-1 with probability 1/2 each.
    n, d = 4000, 3
    Z = inst.ground_truth(11, n, d)
    assert np.abs(Z.mean(axis=0)).max() < 5 * np.sqrt(1.0 / d / n)
    assert np.abs((Z ** 2).mean(axis=0) - 1.0 / d).max() < 0.02
    frac_pos = np.mean(np.linalg.det(Z) > 0)
    assert abs(frac_pos - 0.5) < 5 * np.sqrt(0.25 / n)


def test_measurement_matrix_structure():
    n, d, sigma, seed = 12, 3, 0.7, 5
    Z = inst.ground_truth(seed, n, d)
    A = inst.measurement_matrix(seed, Z, sigma)
    assert np.array_equal(A, A.T)                                      # bitwise symmetric
    for i in range(n):
        assert not A[i * d:(i + 1) * d, i * d:(i + 1) * d].any()        # A_ii = 0
    assert np.array_equal(A.astype(np.float32).astype(np.float64), A)  # fp32 values
    # A_ij - Z_i Z_j^T = sigma W_ij with W_ij from counter (i, j) for i < j and W_ji = W_ij^T
    for i in range(n):
        for j in range(n):
            if i == j:
                continue
            W = inst.noise_block(seed, min(i, j), max(i, j), d)
            W = W if i < j else W.T
            blk = A[i * d:(i + 1) * d, j * d:(j + 1) * d]
            exact = Z[i] @ Z[j].T + sigma * W
            assert np.allclose(blk, exact, rtol=0, atol=4e-7 * np.abs(exact).max())


def test_sigma_zero_is_rank_d_signal():
    n, d = 9, 4
    Z = inst.ground_truth(2, n, d)
    A = inst.measurement_matrix(2, Z, 0.0, dtype=np.float64)
    Zs = Z.reshape(n * d, d)
    assert np.allclose(A, Zs @ Zs.T - np.eye(n * d), atol=1e-14)   # A = ZZ^T - I


def test_measurement_rows_regenerates_same_values():
    n, d, sigma, seed = 15, 5, 1.3, 8
    Z = inst.ground_truth(seed, n, d)
    A = inst.measurement_matrix(seed, Z, sigma)
    nodes = [0, 7, 14]
    R = inst.measurement_rows(seed, Z, sigma, nodes)
    for k, i in enumerate(nodes):
        assert np.array_equal(R[k * d:(k + 1) * d], A[i * d:(i + 1) * d])


def test_noise_statistics():
    n, d, seed = 60, 5, 4
    Z = inst.ground_truth(seed, n, d)
    A0 = inst.measurement_matrix(seed, Z, 0.0, dtype=np.float64)
    A1 = inst.measurement_matrix(seed, Z, 1.0, dtype=np.float64)
    Wm = A1 - A0
    iu = np.triu_indices(n * d, k=d)
    w = np.concatenate([Wm[i * d:(i + 1) * d, (i + 1) * d:].ravel() for i in range(n - 1)])
    assert stats.kstest(w, "norm").pvalue > 1e-4
    assert iu is not None
