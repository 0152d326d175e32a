"""Oracle instance generator (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Definition of the synthetic workload of PAPER.md §1.1 / §2.2:

    A_ij = Z_i Z_j^T + sigma W_ij,  i != j;   W_ji = W_ij^T,  W_ii = 0
    (PAPER.md:59-66 §1.1; :225-230 Eq. def:measurements, "W_ii = 0 ... W_ij
    ... independent standard Gaussian entries for 1 <= i < j <= n").

Readings (DESIGN.md "Readings" R8, R9): the paper does not fix the RNG, the
normal sampler nor the Haar sampler; BASELINE.json's configs fix "QR of N(0,1)
d x d with sign fix" for Z_i.  We fix:

* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11 "Parallel random numbers:
  as easy as 1, 2, 3"), key = (seed & 0xffffffff, seed >> 32), counter
  (c0, c1, c2, c3) = (i, j, q, tag); tag 1 = Z, 2 = W, 3 = Y0, 4 = mask.
* One Philox call -> two fp64 uniforms u = (m + 1) * 2^-53 in (0, 1], with
  m = (x0 >> 5) * 2^26 + (x1 >> 6) (resp. x2, x3) -> two Box-Muller normals
  r cos(2 pi u2), r sin(2 pi u2) with r = sqrt(-2 ln u1).  Call q yields the
  normals 2q, 2q+1 of a block, filled row-major.
* Z_i = Q of the QR factorisation of the d x d Gaussian block (tag 1, counter
  (i, 0, q, 1)) with the sign fix diag(R) > 0 (unique).
* W_ij for i < j from counter (i, j, q, 2); A_ij rounded to fp32
  (round-to-nearest) from the fp64 value; A_ji = A_ij^T from the SAME values;
  A_ii = 0.  ``dtype=np.float64`` keeps the fp64 values (config c1 "fp64").

The CUDA generator implements the same definition independently
(paper_2604_07372_b200/csrc/aux.cu, common.cuh); the two share no code.
* p < 1: pair {i < j} observed iff u < p, u the first uniform of
  counter (i, j, 0, 4); unobserved A_ij = A_ji = 0.
"""
from __future__ import annotations

import numpy as np

TAG_Z = 1
TAG_W = 2
TAG_Y0 = 3
TAG_MASK = 4

# Philox4x32 constants (Salmon et al., SC'11, §"Philox").
_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint64(0x9E3779B9)
_W1 = np.uint64(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Philox4x32 with 10 rounds on uint32 arrays (broadcast).  Returns 4 uint32 arrays.

    Round: (hi0, lo0) = mulhilo(M0, c0); (hi1, lo1) = mulhilo(M1, c2);
    c <- (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0); key bumped by (W0, W1)
    between rounds.
    """
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) & _MASK32 for c in (c0, c1, c2, c3))
    k0 = np.asarray(k0, dtype=np.uint64) & _MASK32
    k1 = np.asarray(k1, dtype=np.uint64) & _MASK32
    for r in range(10):
        if r > 0:
            k0 = (k0 + _W0) & _MASK32
            k1 = (k1 + _W1) & _MASK32
        p0 = _M0 * c0
        p1 = _M1 * c2
        hi0, lo0 = p0 >> _S32, p0 & _MASK32
        hi1, lo1 = p1 >> _S32, p1 & _MASK32
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return tuple(c.astype(np.uint32) for c in (c0, c1, c2, c3))


def _uniform53(hi, lo):
    m = (hi.astype(np.uint64) >> np.uint64(5)) * np.uint64(1 << 26) + (lo.astype(np.uint64) >> np.uint64(6))
    return (m.astype(np.float64) + 1.0) * 2.0 ** -53


def block_normals(seed: int, c0, c1, tag: int, count: int) -> np.ndarray:
    """`count` standard normals for each counter prefix (c0[k], c1[k]); shape (K, count)."""
    c0 = np.atleast_1d(np.asarray(c0, dtype=np.uint64))
    c1 = np.atleast_1d(np.asarray(c1, dtype=np.uint64))
    c0, c1 = np.broadcast_arrays(c0, c1)
    ncalls = (count + 1) // 2
    q = np.arange(ncalls, dtype=np.uint64)
    C0 = c0[:, None]
    C1 = c1[:, None]
    Q = q[None, :]
    x0, x1, x2, x3 = philox4x32_10(C0, C1, Q, np.uint64(tag), seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    u1 = _uniform53(x0, x1)
    u2 = _uniform53(x2, x3)
    r = np.sqrt(-2.0 * np.log(u1))
    th = 2.0 * np.pi * u2
    z = np.empty(c0.shape + (2 * ncalls,), dtype=np.float64)
    z[:, 0::2] = r * np.cos(th)
    z[:, 1::2] = r * np.sin(th)
    return z[:, :count]


def observed(seed: int, i, j, p: float) -> np.ndarray:
    """Observation mask of PAPER.md:300-310 (§4.1): the unordered pair {i, j} (i < j) is in the
    edge set with probability p (reading R18: unordered pairs, symmetric mask).  Drawn as
    u < p with u the first uniform of Philox counter (i, j, 0, TAG_MASK)."""
    i = np.atleast_1d(np.asarray(i, dtype=np.uint64))
    j = np.atleast_1d(np.asarray(j, dtype=np.uint64))
    i, j = np.broadcast_arrays(i, j)
    x0, x1, _, _ = philox4x32_10(i, j, np.uint64(0), np.uint64(TAG_MASK), seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF)
    return _uniform53(x0, x1) < p


def ground_truth(seed: int, n: int, d: int) -> np.ndarray:
    """Z in O(d)^{(x)n}, shape (n, d, d): Q of QR(G_i) with diag(R) > 0 (BASELINE configs)."""
    G = block_normals(seed, np.arange(n), 0, TAG_Z, d * d).reshape(n, d, d)
    Z = np.empty_like(G)
    for i in range(n):
        Q, R = np.linalg.qr(G[i])
        Z[i] = Q * np.sign(np.diag(R))[None, :]
    return Z


def noise_block(seed: int, i: int, j: int, d: int) -> np.ndarray:
    """W_ij for i < j (d x d, row-major from counter (i, j, q, TAG_W))."""
    assert i < j
    return block_normals(seed, i, j, TAG_W, d * d).reshape(d, d)


def measurement_rows(seed: int, Z: np.ndarray, sigma: float, nodes, dtype=np.float32, p: float = 1.0) -> np.ndarray:
    """Block rows of A for the given node indices: shape (len(nodes)*d, n*d), float64 array
    holding `dtype`-rounded values.  Independent regeneration used for sampled parity.
    p < 1: unobserved blocks are 0."""
    n, d, _ = Z.shape
    nodes = np.asarray(nodes, dtype=np.int64)
    out = np.zeros((len(nodes) * d, n * d), dtype=np.float64)
    for k, i in enumerate(nodes):
        js = np.arange(n)
        lo = np.minimum(i, js)
        hi = np.maximum(i, js)
        W = block_normals(seed, lo, hi, TAG_W, d * d).reshape(n, d, d)
        # W_ij for i > j is W_ji^T ("W_ij = W_ji^T").
        Wt = np.where((js > i)[:, None, None], W, np.transpose(W, (0, 2, 1)))
        blocks = np.einsum("ak,jbk->jab", Z[i], Z) + sigma * Wt  # (n, d, d): Z_i Z_j^T + sigma W_ij
        blocks = blocks.astype(dtype).astype(np.float64)
        if p < 1.0:
            blocks[~observed(seed, lo, hi, p)] = 0.0
        blocks[i] = 0.0  # A_ii = 0 ("W_ii = 0", self-loops excluded)
        out[k * d:(k + 1) * d, :] = blocks.transpose(1, 0, 2).reshape(d, n * d)
    return out


def measurement_matrix(seed: int, Z: np.ndarray, sigma: float, dtype=np.float32, p: float = 1.0) -> np.ndarray:
    """Dense A (nd x nd), values rounded to `dtype`, returned as float64.

    Built from the upper blocks i < j; the lower blocks are the transposes of the
    SAME rounded values, so A is bitwise symmetric ("symmetric").
    p < 1: each unordered pair is observed with probability p, else A_ij = A_ji = 0
    (§4.1)."""
    n, d, _ = Z.shape
    A = np.zeros((n * d, n * d), dtype=np.float64)
    for i in range(n - 1):
        js = np.arange(i + 1, n)
        W = block_normals(seed, i, js, TAG_W, d * d).reshape(len(js), d, d)
        blocks = np.einsum("ak,jbk->jab", Z[i], Z[js]) + sigma * W
        blocks = blocks.astype(dtype).astype(np.float64)
        if p < 1.0:
            blocks[~observed(seed, i, js, p)] = 0.0
        row = blocks.transpose(1, 0, 2).reshape(d, len(js) * d)
        A[i * d:(i + 1) * d, (i + 1) * d:] = row
        A[(i + 1) * d:, i * d:(i + 1) * d] = row.T
    return A


def initial_subspace(seed: int, n: int, d: int) -> np.ndarray:
    """Y0 (nd x d) Gaussian: row r from counter (r, 0, q, TAG_Y0)."""
    return block_normals(seed, np.arange(n * d), 0, TAG_Y0, d)


def config_sigma(name: str, n: int, d: int) -> float:
    """sigma of BASELINE.json configs c3-c5: sigma = c * sqrt(n) / d."""
    c = {"c3": 0.3, "c4": 0.2, "c5": 0.3}[name]
    return c * np.sqrt(n) / d
