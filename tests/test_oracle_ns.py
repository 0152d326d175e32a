"""Pins for the Newton-Schulz retraction (PAPER.md:148-151 Eq. eq:newton-schulz,
:172-182 Algorithm 1, :164-168 Lemma le:ns:bound)."""
import os

import numpy as np
import pytest

from oracle import nsrgs as ns

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _haar(rng, d):
    Q, R = np.linalg.qr(rng.standard_normal((d, d)))
    return Q * np.sign(np.diag(R))


def test_worked_example_golden():
    with open(os.path.join(GOLD, "ns_scalar_example.txt")) as f:
        rows = [l.split() for l in f if l.strip() and not l.startswith("#")]
    for r in rows:
        a, b, Ts, oa, ob = float(r[0]), float(r[1]), int(r[2]), float(r[3]), float(r[4])
        S = ns.newton_schulz(np.diag([a, b]), Ts)
        assert np.allclose(S, np.diag([oa, ob]), atol=1e-15)


@pytest.mark.parametrize("d", [2, 3, 5, 10, 25])
def test_fixed_point_on_orthogonal(d):
    rng = np.random.default_rng(d)
    Q = _haar(rng, d)
    assert np.linalg.norm(ns.newton_schulz(Q, 7) - Q) < 1e-13


@pytest.mark.parametrize("d", [2, 3, 5, 10])
@pytest.mark.parametrize("K", [1, 3, 6])
def test_singular_value_recursion_closed_form(d, K):
    # For A = U diag(s) V^T every NS step maps s -> s(3 - s^2)/2 with U, V fixed.
    rng = np.random.default_rng(100 * d + K)
    for _ in range(20):
        U, V = _haar(rng, d), _haar(rng, d)
        s = rng.uniform(0.2, 1.6, d)
        sK = s.copy()
        for _ in range(K):
            sK = sK * (3 - sK ** 2) / 2
        A = U @ np.diag(s) @ V.T
        assert np.allclose(ns.newton_schulz(A, K), U @ np.diag(sK) @ V.T, atol=1e-13)


@pytest.mark.parametrize("d", [2, 3, 5, 25])
def test_lemma_ns_bound_chain(d):
    # ||S_t - sgn A||_2 <= ||I - S_t^T S_t||_2 <= ||I - A^T A||_2^(2^t), t = 1, 2, 3,
    # on 1000 random inputs with ||I - A^T A||_2 <= 0.9.
    rng = np.random.default_rng(d)
    I = np.eye(d)
    n_inputs = 1000 if d <= 5 else 200
    for _ in range(n_inputs):
        U, V = _haar(rng, d), _haar(rng, d)
        s = np.sqrt(rng.uniform(0.1, 1.9, d))
        A = U @ np.diag(s) @ V.T
        e0 = np.linalg.norm(I - A.T @ A, 2)
        assert e0 <= 0.9 + 1e-12
        sA = ns.sgn(A)
        for t in (1, 2, 3):
            St = ns.newton_schulz(A, t)
            lhs = np.linalg.norm(St - sA, 2)
            mid = np.linalg.norm(I - St.T @ St, 2)
            assert lhs <= mid + 1e-12
            assert mid <= e0 ** (2 ** t) + 1e-12


@pytest.mark.parametrize("d", [2, 3, 5])
def test_converges_to_svd_polar(d):
    rng = np.random.default_rng(7 + d)
    for _ in range(50):
        A = _haar(rng, d) @ np.diag(rng.uniform(0.5, 1.5, d)) @ _haar(rng, d)
        assert np.linalg.norm(ns.newton_schulz(A, 30) - ns.sgn(A)) < 1e-14


def test_sgn_examples():
    # I -> I, cQ -> Q, diag(2, -3) -> diag(1, -1)
    assert np.allclose(ns.sgn(np.eye(3)), np.eye(3))
    Q = _haar(np.random.default_rng(1), 4)
    assert np.allclose(ns.sgn(3.7 * Q), Q, atol=1e-14)
    assert np.allclose(ns.sgn(np.diag([2.0, -3.0])), np.diag([1.0, -1.0]))


def test_batched_equals_per_block():
    rng = np.random.default_rng(3)
    F = rng.standard_normal((6, 3, 3)) * 0.1 + np.eye(3)
    out = ns.newton_schulz(F, 4)
    for i in range(6):
        assert np.allclose(out[i], ns.newton_schulz(F[i], 4), rtol=0, atol=1e-15)
