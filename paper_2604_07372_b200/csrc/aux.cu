// aux.cu — the non-streaming kernels of the NS-RGS path: instance generator (a0), subspace
// orthonormalisation (a1), init polar by scaled Newton-Schulz (a2), layout pack/unpack,
// deterministic fp64 reductions, objective finalisation (a8) and recovery metrics (a9).
// All are O(n d^2) or one-time; the O(N^2) work is in panel.cu.
#include "common.cuh"
#include "kernels.h"

namespace nsrgs {

namespace {
constexpr int kRedThreads = 256;
constexpr int kChebRows = 64;   // rows per CTA of the Chebyshev combine (smem: 2 x 64 x 32 elements)

template <typename T> __device__ __forceinline__ double block_sum(double v, double *sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
  __syncthreads();
  return t;   // valid in thread 0
}
}  // namespace

// ----------------------------------------------------------------------------------------
// a0: ground truth Z_i = Q of QR(G_i), diag(R) > 0, G_i row-major normals of (i, 0, q, 1).
// Modified Gram-Schmidt on the columns in fp64 yields the same unique factor as a
// Householder QR with the sign fix (up to rounding).
template <int D>
__global__ void gen_Z_kernel(int64_t n, uint64_t seed, double *Z64) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double G[D][D];
#pragma unroll
  for (int q = 0; q < (D * D + 1) / 2; ++q) {
    double z0, z1;
    normal_pair(seed, (uint32_t)i, 0u, (uint32_t)q, 1u, z0, z1);
    const int e0 = 2 * q, e1 = 2 * q + 1;
    G[e0 / D][e0 % D] = z0;
    if (e1 < D * D) G[e1 / D][e1 % D] = z1;
  }
#pragma unroll
  for (int j = 0; j < D; ++j) {
#pragma unroll
    for (int k = 0; k < j; ++k) {
      double r = 0.0;
#pragma unroll
      for (int a = 0; a < D; ++a) r += G[a][k] * G[a][j];
#pragma unroll
      for (int a = 0; a < D; ++a) G[a][j] -= r * G[a][k];
    }
    double nr = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) nr += G[a][j] * G[a][j];
    nr = 1.0 / sqrt(nr);
#pragma unroll
    for (int a = 0; a < D; ++a) G[a][j] *= nr;
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) Z64[(i * D + a) * D + b] = G[a][b];
}

template <typename T>
__global__ void cast_kernel(const double *src, T *dst, int64_t count) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) dst[i] = (T)src[i];
}

// A shard rows of local nodes [node0, node0 + n_local): thread = (local node il, node j).
// A_ij = round(Z_i Z_j^T + sigma W_ij), W_ij from counter (min, max) transposed for i > j,
// A_ii = 0.  ||A_shard||_F^2 partial per block (of the rounded values).
template <typename T, int D>
__global__ void gen_A_kernel(int64_t n, int64_t node0, int64_t n_local, uint64_t seed, double sigma, double p_obs,
                             const double *Z64, T *A, int64_t lda, double *part) {
  __shared__ double Zi[D * D];
  __shared__ double sh[32];
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double ss = 0.0;
  for (int64_t il = blockIdx.y; il < n_local; il += gridDim.y) {
    const int64_t i = node0 + il;
    __syncthreads();
    for (int e = threadIdx.x; e < D * D; e += blockDim.x) Zi[e] = Z64[i * D * D + e];
    __syncthreads();
    if (j >= n) continue;
    T *Ab = A + (il * D) * lda + j * D;
    if (j == i) {
#pragma unroll
      for (int a = 0; a < D; ++a)
#pragma unroll
        for (int b = 0; b < D; ++b) Ab[a * lda + b] = T(0);
      continue;
    }
    const double *Zj = Z64 + j * D * D;
    const uint32_t lo = (uint32_t)min(i, j), hi = (uint32_t)max(i, j);
    const bool tr = i > j;
    if (p_obs < 1.0) {   // incomplete observations: pair {lo, hi} in the edge set?
      const U4 v = philox4x32_10(lo, hi, 0u, 4u, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
      if (!(uniform53(v.x, v.y) < p_obs)) {
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int b = 0; b < D; ++b) Ab[a * lda + b] = T(0);
        continue;
      }
    }
#pragma unroll
    for (int q = 0; q < (D * D + 1) / 2; ++q) {
      double w[2];
      normal_pair(seed, lo, hi, (uint32_t)q, 2u, w[0], w[1]);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = 2 * q + h;
        if (e < D * D) {
          const int a = tr ? e % D : e / D, b = tr ? e / D : e % D;   // position in A_ij
          double v = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k) v += Zi[a * D + k] * Zj[b * D + k];
          v += sigma * w[h];
          const T tv = (T)v;
          Ab[a * lda + b] = tv;
          ss += (double)tv * (double)tv;
        }
      }
    }
  }
  const double t = block_sum<T>(ss, sh);
  if (threadIdx.x == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
}

// Y0 rows r in [0, N): d normals from (r, 0, q, 3), into the tile layout.
template <typename T, int D>
__global__ void gen_Y0_kernel(int64_t N, uint64_t seed, T *Y, int64_t rows_local, int64_t tpr) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
#pragma unroll
  for (int q = 0; q < (D + 1) / 2; ++q) {
    double z0, z1;
    normal_pair(seed, (uint32_t)r, 0u, (uint32_t)q, 3u, z0, z1);
    Y[tile_index(r, 2 * q, D, rows_local, tpr)] = (T)z0;
    if (2 * q + 1 < D) Y[tile_index(r, 2 * q + 1, D, rows_local, tpr)] = (T)z1;
  }
}

template <typename T>
__global__ void sumsq_kernel(const T *A, int64_t rows, int64_t cols, int64_t lda, double *part) {
  __shared__ double sh[32];
  double ss = 0.0;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y)
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (int64_t)gridDim.x * blockDim.x) {
      const double v = (double)A[r * lda + c];
      ss += v * v;
    }
  const double t = block_sum<T>(ss, sh);
  if (threadIdx.x == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
}

// out[i] = sum_b part[b * width + i] in a fixed order (deterministic).  width == 1: 1024
// threads take strided slices, then a fixed-shape tree; width > 1: one thread per column.
__global__ void reduce_kernel(const double *part, int nblocks, int width, double *out) {
  if (width == 1) {
    __shared__ double sh[1024];
    double v = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x) v += part[b];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if ((int)threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = sh[0];
    return;
  }
  // width > 1: one CTA per column i, threads over the slots in a fixed partition, fixed-order tree
  __shared__ double sh2[256];
  const int i = blockIdx.x;
  double v = 0.0;
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x) v += part[(int64_t)b * width + i];
  sh2[threadIdx.x] = v;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) sh2[threadIdx.x] += sh2[threadIdx.x + st];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[i] = sh2[0];
}

template <typename T>
__global__ void pack_kernel(int d, int64_t N, T *stack, T *tiled, int64_t rows_local, int64_t tpr, int unpack) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= N * d) return;
  const int64_t c = idx / d;
  const int k = (int)(idx - c * d);
  const int64_t t = tile_index(c, k, d, rows_local, tpr);
  if (unpack) stack[idx] = tiled[t]; else tiled[t] = stack[idx];
}

// ----------------------------------------------------------------------------------------
// a1: Cholesky-QR of the sweep.  res = [W^T W (DD) | Y^T W (DD) | ...] (fp64, global sums).
// L L^T = W^T W, M = L^{-T} (upper triangular, Y_new = W M), CM = (Y^T W) M = Y^T Y_new.
// MC = [M (DD) | CM (DD)].
template <int D>
__global__ void chol_kernel(const double *res, double *MC, int *err) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double L[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) L[a][b] = 0.0;
  bool ok = true;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double s = res[j * D + j];
#pragma unroll
    for (int k = 0; k < j; ++k) s -= L[j][k] * L[j][k];
    if (!(s > 0.0)) { ok = false; s = 1.0; }
    L[j][j] = sqrt(s);
#pragma unroll
    for (int i = j + 1; i < D; ++i) {
      double t = res[i * D + j];
#pragma unroll
      for (int k = 0; k < j; ++k) t -= L[i][k] * L[j][k];
      L[i][j] = t / L[j][j];
    }
  }
  // Linv = L^{-1} (lower), M = Linv^T
  double Li[D][D];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) Li[a][b] = 0.0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    Li[c][c] = 1.0 / L[c][c];
#pragma unroll
    for (int i = c + 1; i < D; ++i) {
      double t = 0.0;
#pragma unroll
      for (int k = c; k < i; ++k) t += L[i][k] * Li[k][c];
      Li[i][c] = -t / L[i][i];
    }
  }
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) MC[a * D + b] = Li[b][a];
  const double *Cm = res + D * D;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double t = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) t += Cm[a * D + k] * Li[b][k];
      MC[D * D + a * D + b] = t;
    }
  if (!ok) atomicOr(err, kErrSingular);
}

// Y_new[r] = W[r] M (in place in W), and the subspace-change residual
// ||Y_new - Y_old (Y_old^T Y_new)||_F^2 = sum_r ||Y_new[r] - Y_old[r] CM||^2 (partial per block).
template <typename T, int D>
__global__ void scale_kernel(int64_t row0, int64_t rows, const double *MC, T *W, const T *Yold, int64_t rows_local,
                             int64_t tpr, double *part) {
  __shared__ double sMC[2 * D * D];
  __shared__ double sh[32];
  for (int e = threadIdx.x; e < 2 * D * D; e += blockDim.x) sMC[e] = MC[e];
  __syncthreads();
  const int64_t rl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double ss = 0.0;
  if (rl < rows) {
    const int64_t r = row0 + rl;
    double w[D], y[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
      w[k] = (double)W[tile_index(r, k, D, rows_local, tpr)];
      y[k] = (double)Yold[tile_index(r, k, D, rows_local, tpr)];
    }
#pragma unroll
    for (int b = 0; b < D; ++b) {
      double v = 0.0, pr = 0.0;
#pragma unroll
      for (int k = 0; k < D; ++k) {
        v += w[k] * sMC[k * D + b];
        pr += y[k] * sMC[D * D + k * D + b];
      }
      const T tv = (T)v;
      W[tile_index(r, b, D, rows_local, tpr)] = tv;
      const double dlt = (double)tv - pr;
      ss += dlt * dlt;
    }
  }
  const double t = block_sum<T>(ss, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// ----------------------------------------------------------------------------------------
// a1, Chebyshev-filtered subspace step (runtime d, O(N d^2)): Y_new = alpha W - beta Y_prev
// (in place in W; beta = 0 on the first filtered step), with the fp64 Gram partials
// [Y_new^T Y_new | Y_cur^T Y_new] per block (width 2 d^2) for the Cholesky-QR that follows.
template <typename T>
__global__ void cheb_combine_kernel(int d, int64_t row0, int64_t rows, double alpha, double beta, T *W,
                                    const T *Yprev, const T *Ycur, int64_t rows_local, int64_t tpr, double *part) {
  // CTA = kChebRows rows: phase 1 forms this CTA's rows of Y_new (thread = row) and stages Y_new,
  // Y_cur in smem; phase 2 forms the CTA's Gram partials entry-parallel (fixed row order)
  __shared__ T sy[kChebRows * kMaxD], sc[kChebRows * kMaxD];
  const int DD = d * d;
  const int64_t rbase = (int64_t)blockIdx.x * kChebRows;
  const int nr = (int)min((int64_t)kChebRows, rows - rbase);
  const int t = threadIdx.x;
  if (t < nr) {
    const int64_t r = row0 + rbase + t;
    for (int k = 0; k < d; ++k) {
      const int64_t ix = tile_index(r, k, d, rows_local, tpr);
      double v = alpha * (double)W[ix];
      if (beta != 0.0) v -= beta * (double)Yprev[ix];
      const T tv = (T)v;
      W[ix] = tv;
      sy[t * d + k] = tv;
      sc[t * d + k] = Ycur[ix];
    }
  }
  __syncthreads();
  for (int e = t; e < 2 * DD; e += blockDim.x) {
    const int a = (e % DD) / d, b = (e % DD) % d;
    const T *left = e < DD ? sy : sc;
    double acc = 0.0;
    for (int r = 0; r < nr; ++r) acc += (double)left[r * d + a] * (double)sy[r * d + b];
    part[(int64_t)blockIdx.x * 2 * DD + e] = acc;
  }
}

// Y_out[r] = Y_in[r] M (M = MC[0..d^2), the Cholesky-QR factor of the filtered block): keeps the
// previous Chebyshev iterate in the same basis as the orthonormalised new one.
template <typename T>
__global__ void cheb_apply_kernel(int d, int64_t row0, int64_t rows, const double *MC, const T *Yin, T *Yout,
                                  int64_t rows_local, int64_t tpr) {
  const int64_t rl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (rl >= rows) return;
  const int64_t r = row0 + rl;
  double y[kMaxD];
  for (int k = 0; k < d; ++k) y[k] = (double)Yin[tile_index(r, k, d, rows_local, tpr)];
  for (int b = 0; b < d; ++b) {
    double v = 0.0;
    for (int k = 0; k < d; ++k) v += y[k] * MC[k * d + b];
    Yout[tile_index(r, b, d, rows_local, tpr)] = (T)v;
  }
}

// ----------------------------------------------------------------------------------------
// a8: F(X^t) = 1/2(||X^T X||^2 - sum_i ||X_i^T X_i||^2) - <X, AX> + 1/2 ||A||^2 for every
// slot t of res[T][npart] = [X^T X (DD) | unused (DD) | s_own | xb].
__global__ void objective_final_kernel(int d, int T, const double *res, int npart, const double *a_fro2,
                                       double *F) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const double *r = res + (int64_t)t * npart;
  double g2 = 0.0;
  for (int e = 0; e < d * d; ++e) g2 += r[e] * r[e];
  F[t] = 0.5 * (g2 - r[2 * d * d]) - r[2 * d * d + 1] + 0.5 * a_fro2[0];
}

// a9: Gram partials [Z^T Z | X^T X | Z^T X] (3 d^2 entries).  Node-parallel: a CTA takes
// `npb` nodes; its 256 threads form G = 256 / (3 d^2) node groups x the 3 d^2 entries (for
// d^2 > 85 one group, threads stride over the entries), each group sums its nodes, and the
// groups are summed in fixed order through smem -> one deterministic partial row per CTA.
// (The round-1 kernel gave each thread one entry and walked 256 nodes serially: 121 us at
// n = 100, 0.38 ms at n = 2000.)
template <typename T, int D>
__global__ void metrics_kernel(int64_t n, const T *X, const T *Z, int64_t rows_local, int64_t tpr, int npb,
                               double *part) {
  constexpr int DD = D * D, E3 = 3 * DD;
  extern __shared__ double msh[];
  const int G = blockDim.x >= E3 ? (int)blockDim.x / E3 : 1;
  const int64_t i0 = (int64_t)blockIdx.x * npb, i1 = min(n, i0 + npb);
  for (int t = threadIdx.x; t < G * E3; t += blockDim.x) {
    const int g = t / E3, e = t - g * E3;
    const int which = e / DD, a = (e / D) % D, b = e % D;
    double s = 0.0;
    for (int64_t i = i0 + g; i < i1; i += G)
#pragma unroll
      for (int k = 0; k < D; ++k) {
        const int64_t r = i * D + k;
        const double u = which == 1 ? (double)X[tile_index(r, a, D, rows_local, tpr)] : (double)Z[r * D + a];
        const double v = which == 0 ? (double)Z[r * D + b] : (double)X[tile_index(r, b, D, rows_local, tpr)];
        s += u * v;
      }
    msh[t] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < E3; e += blockDim.x) {
    double v = 0.0;
    for (int g = 0; g < G; ++g) v += msh[g * E3 + e];
    part[(int64_t)blockIdx.x * E3 + e] = v;
  }
}

// Rel.Err. (Gram identity), nuclear norm of Z^T X by cyclic Jacobi on (Z^T X)^T (Z^T X),
// d_F^2 = ||X||^2 + ||Z||^2 - 2||Z^T X||_*, MSE = d_F^2 / n.
template <int D>
__global__ void metrics_final_kernel(int64_t n, const double *g, double *out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double *ZZ = g, *XX = g + D * D, *ZX = g + 2 * D * D;
  double zz = 0, xx = 0, zx = 0, trz = 0, trx = 0;
  for (int e = 0; e < D * D; ++e) { zz += ZZ[e] * ZZ[e]; xx += XX[e] * XX[e]; zx += ZX[e] * ZX[e]; }
  for (int a = 0; a < D; ++a) { trz += ZZ[a * D + a]; trx += XX[a * D + a]; }
  double S[D][D];
  for (int a = 0; a < D; ++a)
    for (int b = 0; b < D; ++b) {
      double v = 0.0;
      for (int k = 0; k < D; ++k) v += ZX[k * D + a] * ZX[k * D + b];
      S[a][b] = v;
    }
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < D; ++p)
      for (int q = p + 1; q < D; ++q) off += S[p][q] * S[p][q];
    if (off < 1e-30) break;
    for (int p = 0; p < D; ++p)
      for (int q = p + 1; q < D; ++q) {
        if (S[p][q] == 0.0) continue;
        const double th = (S[q][q] - S[p][p]) / (2.0 * S[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < D; ++k) {
          const double skp = S[k][p], skq = S[k][q];
          S[k][p] = c * skp - s * skq;
          S[k][q] = s * skp + c * skq;
        }
        for (int k = 0; k < D; ++k) {
          const double spk = S[p][k], sqk = S[q][k];
          S[p][k] = c * spk - s * sqk;
          S[q][k] = s * spk + c * sqk;
        }
      }
  }
  double nuc = 0.0;
  for (int a = 0; a < D; ++a) nuc += sqrt(fmax(S[a][a], 0.0));
  const double rel = sqrt(fmax(zz + xx - 2.0 * zx, 0.0)) / sqrt(zz);
  const double df2 = fmax(trx + trz - 2.0 * nuc, 0.0);
  out[0] = rel;
  out[1] = sqrt(df2);
  out[2] = df2 / (double)n;
}

// ----------------------------------------------------------------------------------------
// Runtime-d variants for wide blocks (d in (10, 32], wide.cu): same definitions as the
// templated kernels above, loops not unrolled, small arrays in local memory (one-time work).
__global__ void gen_Z_rt(int64_t n, int d, uint64_t seed, double *Z64) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double G[kMaxD * kMaxD];
  for (int q = 0; q < (d * d + 1) / 2; ++q) {
    double z0, z1;
    normal_pair(seed, (uint32_t)i, 0u, (uint32_t)q, 1u, z0, z1);
    G[2 * q] = z0;
    if (2 * q + 1 < d * d) G[2 * q + 1] = z1;
  }
  for (int j = 0; j < d; ++j) {           // modified Gram-Schmidt on the columns (sign fix: R_jj > 0)
    for (int k = 0; k < j; ++k) {
      double r = 0.0;
      for (int a = 0; a < d; ++a) r += G[a * d + k] * G[a * d + j];
      for (int a = 0; a < d; ++a) G[a * d + j] -= r * G[a * d + k];
    }
    double nr = 0.0;
    for (int a = 0; a < d; ++a) nr += G[a * d + j] * G[a * d + j];
    nr = 1.0 / sqrt(nr);
    for (int a = 0; a < d; ++a) G[a * d + j] *= nr;
  }
  for (int e = 0; e < d * d; ++e) Z64[i * d * d + e] = G[e];
}

template <typename T>
__global__ void gen_A_rt(int64_t n, int d, int64_t node0, int64_t n_local, uint64_t seed, double sigma, double p_obs,
                         const double *Z64, T *A, int64_t lda, double *part) {
  __shared__ double sh[32];
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double ss = 0.0;
  for (int64_t il = blockIdx.y; il < n_local; il += gridDim.y) {
    const int64_t i = node0 + il;
    if (j >= n) continue;
    T *Ab = A + (il * d) * lda + j * d;
    bool zero = (j == i);
    const uint32_t lo = (uint32_t)min(i, j), hi = (uint32_t)max(i, j);
    if (!zero && p_obs < 1.0) {
      const U4 v = philox4x32_10(lo, hi, 0u, 4u, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
      zero = !(uniform53(v.x, v.y) < p_obs);
    }
    if (zero) {
      for (int a = 0; a < d; ++a)
        for (int b = 0; b < d; ++b) Ab[a * lda + b] = T(0);
      continue;
    }
    const double *Zi = Z64 + i * d * d, *Zj = Z64 + j * d * d;
    const bool tr = i > j;
    for (int q = 0; q < (d * d + 1) / 2; ++q) {
      double w[2];
      normal_pair(seed, lo, hi, (uint32_t)q, 2u, w[0], w[1]);
      for (int h = 0; h < 2; ++h) {
        const int e = 2 * q + h;
        if (e < d * d) {
          const int a = tr ? e % d : e / d, b = tr ? e / d : e % d;
          double v = 0.0;
          for (int k = 0; k < d; ++k) v += Zi[a * d + k] * Zj[b * d + k];
          v += sigma * w[h];
          const T tv = (T)v;
          Ab[a * lda + b] = tv;
          ss += (double)tv * (double)tv;
        }
      }
    }
  }
  const double t = block_sum<T>(ss, sh);
  if (threadIdx.x == 0) part[(int64_t)blockIdx.y * gridDim.x + blockIdx.x] = t;
}

template <typename T>
__global__ void gen_Y0_rt(int64_t N, int d, uint64_t seed, T *Y, int64_t rows_local, int64_t tpr) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= N) return;
  for (int q = 0; q < (d + 1) / 2; ++q) {
    double z0, z1;
    normal_pair(seed, (uint32_t)r, 0u, (uint32_t)q, 3u, z0, z1);
    Y[tile_index(r, 2 * q, d, rows_local, tpr)] = (T)z0;
    if (2 * q + 1 < d) Y[tile_index(r, 2 * q + 1, d, rows_local, tpr)] = (T)z1;
  }
}

// One warp: right-looking Cholesky of the d x d Gram (the same subtraction order per entry as the
// sequential left-looking form), column-parallel forward substitution for L^{-1}, then M = L^{-T}
// and CM = Cm M entry-parallel.  (The single-thread version took 439 us at d = 25.)
__global__ void chol_rt(int d, const double *res, double *MC, int *err) {
  __shared__ double L[kMaxD][kMaxD + 1], Li[kMaxD][kMaxD + 1];
  __shared__ int bad;
  const int lane = threadIdx.x;
  if (blockIdx.x != 0 || lane >= 32) return;
  if (lane == 0) bad = 0;
  for (int e = lane; e < kMaxD * kMaxD; e += 32) {
    const int i = e / kMaxD, j = e % kMaxD;
    L[i][j] = (i < d && j < d && j <= i) ? res[i * d + j] : 0.0;
    Li[i][j] = 0.0;
  }
  __syncwarp();
  for (int j = 0; j < d; ++j) {
    if (lane == 0) {
      double s = L[j][j];
      if (!(s > 0.0)) { bad = 1; s = 1.0; }
      L[j][j] = sqrt(s);
    }
    __syncwarp();
    const int i = lane;
    if (i > j && i < d) L[i][j] /= L[j][j];
    __syncwarp();
    if (i > j && i < d)   // trailing update of row i: L[i][k] -= L[i][j] L[k][j], j < k <= i
      for (int k = j + 1; k <= i; ++k) L[i][k] -= L[i][j] * L[k][j];
    __syncwarp();
  }
  {
    const int c = lane;   // column c of L^{-1}
    if (c < d) {
      Li[c][c] = 1.0 / L[c][c];
      for (int i = c + 1; i < d; ++i) {
        double t = 0.0;
        for (int k = c; k < i; ++k) t += L[i][k] * Li[k][c];
        Li[i][c] = -t / L[i][i];
      }
    }
  }
  __syncwarp();
  const double *Cm = res + d * d;
  for (int e = lane; e < d * d; e += 32) {
    const int a2 = e / d, b2 = e % d;
    MC[e] = Li[b2][a2];
    double t = 0.0;
    for (int k = 0; k < d; ++k) t += Cm[a2 * d + k] * Li[b2][k];
    MC[d * d + e] = t;
  }
  if (lane == 0 && bad) atomicOr(err, kErrSingular);
}

template <typename T>
__global__ void scale_rt(int d, int64_t row0, int64_t rows, const double *MC, T *W, const T *Yold, int64_t rows_local,
                         int64_t tpr, double *part) {
  __shared__ double sh[32];
  const int64_t rl = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double ss = 0.0;
  if (rl < rows) {
    const int64_t r = row0 + rl;
    double w[kMaxD], y[kMaxD];
    for (int k = 0; k < d; ++k) {
      w[k] = (double)W[tile_index(r, k, d, rows_local, tpr)];
      y[k] = (double)Yold[tile_index(r, k, d, rows_local, tpr)];
    }
    for (int b = 0; b < d; ++b) {
      double v = 0.0, pr = 0.0;
      for (int k = 0; k < d; ++k) {
        v += w[k] * MC[k * d + b];
        pr += y[k] * MC[d * d + k * d + b];
      }
      const T tv = (T)v;
      W[tile_index(r, b, d, rows_local, tpr)] = tv;
      const double dl = (double)tv - pr;
      ss += dl * dl;
    }
  }
  const double t = block_sum<T>(ss, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

template <typename T>
__global__ void metrics_rt(int64_t n, int d, const T *X, const T *Z, int64_t rows_local, int64_t tpr, int npb,
                           double *part) {   // d > 10: as metrics_kernel with one node group
  const int DD = d * d, E3 = 3 * DD;
  const int64_t i0 = (int64_t)blockIdx.x * npb, i1 = min(n, i0 + npb);
  for (int e = threadIdx.x; e < E3; e += blockDim.x) {
    const int which = e / DD, a = (e / d) % d, b = e % d;
    double s = 0.0;
    for (int64_t i = i0; i < i1; ++i)
      for (int k = 0; k < d; ++k) {
        const int64_t r = i * d + k;
        const double u = which == 1 ? (double)X[tile_index(r, a, d, rows_local, tpr)] : (double)Z[r * d + a];
        const double v = which == 0 ? (double)Z[r * d + b] : (double)X[tile_index(r, b, d, rows_local, tpr)];
        s += u * v;
      }
    part[(int64_t)blockIdx.x * E3 + e] = s;
  }
}

__global__ void metrics_final_rt(int64_t n, int d, const double *g, double *out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double *ZZ = g, *XX = g + d * d, *ZX = g + 2 * d * d;
  double zz = 0, xx = 0, zx = 0, trz = 0, trx = 0;
  for (int e = 0; e < d * d; ++e) { zz += ZZ[e] * ZZ[e]; xx += XX[e] * XX[e]; zx += ZX[e] * ZX[e]; }
  for (int a = 0; a < d; ++a) { trz += ZZ[a * d + a]; trx += XX[a * d + a]; }
  double S[kMaxD * kMaxD];
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      double v = 0.0;
      for (int k = 0; k < d; ++k) v += ZX[k * d + a] * ZX[k * d + b];
      S[a * d + b] = v;
    }
  for (int sweep = 0; sweep < 100; ++sweep) {   // cyclic Jacobi eigenvalues of (Z^T X)^T (Z^T X)
    double off = 0.0;
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) off += S[p * d + q] * S[p * d + q];
    if (off < 1e-30) break;
    for (int p = 0; p < d; ++p)
      for (int q = p + 1; q < d; ++q) {
        if (S[p * d + q] == 0.0) continue;
        const double th = (S[q * d + q] - S[p * d + p]) / (2.0 * S[p * d + q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < d; ++k) {
          const double skp = S[k * d + p], skq = S[k * d + q];
          S[k * d + p] = c * skp - s * skq;
          S[k * d + q] = s * skp + c * skq;
        }
        for (int k = 0; k < d; ++k) {
          const double spk = S[p * d + k], sqk = S[q * d + k];
          S[p * d + k] = c * spk - s * sqk;
          S[q * d + k] = s * spk + c * sqk;
        }
      }
  }
  double nuc = 0.0;
  for (int a = 0; a < d; ++a) nuc += sqrt(fmax(S[a * d + a], 0.0));
  const double rel = sqrt(fmax(zz + xx - 2.0 * zx, 0.0)) / sqrt(zz);
  const double df2 = fmax(trx + trz - 2.0 * nuc, 0.0);
  out[0] = rel;
  out[1] = sqrt(df2);
  out[2] = df2 / (double)n;
}

// ----------------------------------------------------------------------------------------
// dispatchers
#define NSRGS_D_SWITCH(d, CALL)                   \
  switch (d) {                                   \
    case 2: { constexpr int D = 2; CALL; } break; \
    case 3: { constexpr int D = 3; CALL; } break; \
    case 4: { constexpr int D = 4; CALL; } break; \
    case 5: { constexpr int D = 5; CALL; } break; \
    case 6: { constexpr int D = 6; CALL; } break; \
    case 7: { constexpr int D = 7; CALL; } break; \
    case 8: { constexpr int D = 8; CALL; } break; \
    case 9: { constexpr int D = 9; CALL; } break; \
    case 10: { constexpr int D = 10; CALL; } break; \
    default: return cudaErrorInvalidValue;        \
  }

static inline unsigned nblk(int64_t count, int threads) { return (unsigned)((count + threads - 1) / threads); }

cudaError_t launch_gen_Z(int dtype, int d, int64_t n, uint64_t seed, double *Z64, void *Zt, cudaStream_t s) {
  if (d > kMaxNarrowD) {
    gen_Z_rt<<<nblk(n, 64), 64, 0, s>>>(n, d, seed, Z64);
  } else {
    NSRGS_D_SWITCH(d, (gen_Z_kernel<D><<<nblk(n, 128), 128, 0, s>>>(n, seed, Z64)));
  }
  if (Zt) {
    const int64_t cnt = n * d * d;
    if (dtype == 0) cast_kernel<float><<<nblk(cnt, 256), 256, 0, s>>>(Z64, (float *)Zt, cnt);
    else cast_kernel<double><<<nblk(cnt, 256), 256, 0, s>>>(Z64, (double *)Zt, cnt);
  }
  return cudaGetLastError();
}

cudaError_t launch_gen_A(int dtype, int d, int64_t n, int64_t node0, int64_t n_local, uint64_t seed, double sigma,
                         double p_obs, const double *Z64, void *A, int64_t lda, double *part, int *nblocks,
                         cudaStream_t s) {
  dim3 grid(nblk(n, 128), (unsigned)(n_local < 32768 ? n_local : 32768));
  *nblocks = (int)(grid.x * grid.y);
  if (d > kMaxNarrowD) {
    if (dtype == 0) gen_A_rt<float><<<grid, 128, 0, s>>>(n, d, node0, n_local, seed, sigma, p_obs, Z64, (float *)A, lda, part);
    else gen_A_rt<double><<<grid, 128, 0, s>>>(n, d, node0, n_local, seed, sigma, p_obs, Z64, (double *)A, lda, part);
    return cudaGetLastError();
  }
  if (dtype == 0) {
    NSRGS_D_SWITCH(d, (gen_A_kernel<float, D><<<grid, 128, 0, s>>>(n, node0, n_local, seed, sigma, p_obs, Z64, (float *)A, lda, part)));
  } else {
    NSRGS_D_SWITCH(d, (gen_A_kernel<double, D><<<grid, 128, 0, s>>>(n, node0, n_local, seed, sigma, p_obs, Z64, (double *)A, lda, part)));
  }
  return cudaGetLastError();
}

cudaError_t launch_gen_Y0(int dtype, int d, int64_t n, uint64_t seed, void *Y, int64_t rows_local, int64_t tpr,
                          cudaStream_t s) {
  const int64_t N = n * d;
  if (d > kMaxNarrowD) {
    if (dtype == 0) gen_Y0_rt<float><<<nblk(N, 256), 256, 0, s>>>(N, d, seed, (float *)Y, rows_local, tpr);
    else gen_Y0_rt<double><<<nblk(N, 256), 256, 0, s>>>(N, d, seed, (double *)Y, rows_local, tpr);
    return cudaGetLastError();
  }
  if (dtype == 0) {
    NSRGS_D_SWITCH(d, (gen_Y0_kernel<float, D><<<nblk(N, 256), 256, 0, s>>>(N, seed, (float *)Y, rows_local, tpr)));
  } else {
    NSRGS_D_SWITCH(d, (gen_Y0_kernel<double, D><<<nblk(N, 256), 256, 0, s>>>(N, seed, (double *)Y, rows_local, tpr)));
  }
  return cudaGetLastError();
}

cudaError_t launch_sumsq(int dtype, const void *A, int64_t rows, int64_t cols, int64_t lda, double *part, int *nblocks,
                         cudaStream_t s) {
  dim3 grid(8, (unsigned)(rows < 4096 ? rows : 4096));
  *nblocks = (int)(grid.x * grid.y);
  if (dtype == 0) sumsq_kernel<float><<<grid, kRedThreads, 0, s>>>((const float *)A, rows, cols, lda, part);
  else sumsq_kernel<double><<<grid, kRedThreads, 0, s>>>((const double *)A, rows, cols, lda, part);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const double *part, int nblocks, int width, double *out, cudaStream_t s) {
  reduce_kernel<<<width == 1 ? 1 : width, width == 1 ? 1024 : 256, 0, s>>>(part, nblocks, width, out);
  return cudaGetLastError();
}

cudaError_t launch_pack(int dtype, int d, int64_t n, const void *stack, void *tiled, int64_t rows_local, int64_t tpr,
                        int unpack, cudaStream_t s) {
  const int64_t N = n * d;
  if (dtype == 0)
    pack_kernel<float><<<nblk(N * d, 256), 256, 0, s>>>(d, N, (float *)stack, (float *)tiled, rows_local, tpr, unpack);
  else
    pack_kernel<double><<<nblk(N * d, 256), 256, 0, s>>>(d, N, (double *)stack, (double *)tiled, rows_local, tpr, unpack);
  return cudaGetLastError();
}

cudaError_t launch_chol(int d, const double *res, double *MC, int *err, cudaStream_t s) {
  if (d > kMaxNarrowD) {
    chol_rt<<<1, 32, 0, s>>>(d, res, MC, err);
    return cudaGetLastError();
  }
  NSRGS_D_SWITCH(d, (chol_kernel<D><<<1, 32, 0, s>>>(res, MC, err)));
  return cudaGetLastError();
}

cudaError_t launch_scale(int dtype, int d, int64_t node0, int64_t n_local, const double *MC, void *W, const void *Yold,
                         int64_t rows_local, int64_t tpr, double *part, int *nblocks, cudaStream_t s) {
  const int64_t rows = n_local * d, row0 = node0 * d;
  *nblocks = (int)nblk(rows, 256);
  if (d > kMaxNarrowD) {
    if (dtype == 0)
      scale_rt<float><<<nblk(rows, 256), 256, 0, s>>>(d, row0, rows, MC, (float *)W, (const float *)Yold, rows_local, tpr, part);
    else
      scale_rt<double><<<nblk(rows, 256), 256, 0, s>>>(d, row0, rows, MC, (double *)W, (const double *)Yold, rows_local, tpr, part);
    return cudaGetLastError();
  }
  if (dtype == 0) {
    NSRGS_D_SWITCH(d, (scale_kernel<float, D><<<nblk(rows, 256), 256, 0, s>>>(row0, rows, MC, (float *)W,
                                                                             (const float *)Yold, rows_local, tpr, part)));
  } else {
    NSRGS_D_SWITCH(d, (scale_kernel<double, D><<<nblk(rows, 256), 256, 0, s>>>(row0, rows, MC, (double *)W,
                                                                              (const double *)Yold, rows_local, tpr, part)));
  }
  return cudaGetLastError();
}

cudaError_t launch_cheb_combine(int dtype, int d, int64_t node0, int64_t n_local, double alpha, double beta, void *W,
                                const void *Yprev, const void *Ycur, int64_t rows_local, int64_t tpr, double *part,
                                int *nblocks, cudaStream_t s) {
  const int64_t rows = n_local * d, row0 = node0 * d;
  const unsigned grid = nblk(rows, kChebRows);
  *nblocks = (int)grid;   // partial slots (one per CTA)
  if (dtype == 0)
    cheb_combine_kernel<float><<<grid, kChebRows, 0, s>>>(d, row0, rows, alpha, beta, (float *)W,
                                                                (const float *)Yprev, (const float *)Ycur, rows_local,
                                                                tpr, part);
  else
    cheb_combine_kernel<double><<<grid, kChebRows, 0, s>>>(d, row0, rows, alpha, beta, (double *)W,
                                                                 (const double *)Yprev, (const double *)Ycur,
                                                                 rows_local, tpr, part);
  return cudaGetLastError();
}

cudaError_t launch_cheb_apply(int dtype, int d, int64_t node0, int64_t n_local, const double *MC, const void *Yin,
                              void *Yout, int64_t rows_local, int64_t tpr, cudaStream_t s) {
  const int64_t rows = n_local * d, row0 = node0 * d;
  if (dtype == 0)
    cheb_apply_kernel<float><<<nblk(rows, 256), 256, 0, s>>>(d, row0, rows, MC, (const float *)Yin, (float *)Yout,
                                                              rows_local, tpr);
  else
    cheb_apply_kernel<double><<<nblk(rows, 256), 256, 0, s>>>(d, row0, rows, MC, (const double *)Yin,
                                                               (double *)Yout, rows_local, tpr);
  return cudaGetLastError();
}

cudaError_t launch_objective_final(int d, int T, const double *res, int npart, const double *a_fro2, double *F,
                                   cudaStream_t s) {
  objective_final_kernel<<<nblk(T, 128), 128, 0, s>>>(d, T, res, npart, a_fro2, F);
  return cudaGetLastError();
}

// Partial rows: one per CTA; the caller reduces *nblocks rows of width 3 d^2 (launch_reduce).
int metrics_blocks(int d, int64_t n) {
  const int E3 = 3 * d * d, G = E3 <= 256 ? 256 / E3 : 1;
  const int npb = 4 * G;
  return (int)((n + npb - 1) / npb);
}

cudaError_t launch_metrics(int dtype, int d, int64_t n, const void *X, const void *Z, int64_t rows_local, int64_t tpr,
                           double *part, int *nblocks, cudaStream_t s) {
  const int E3 = 3 * d * d, G = E3 <= 256 ? 256 / E3 : 1;
  const int npb = 4 * G;   // ~4 nodes per group
  *nblocks = (int)nblk(n, npb);
  if (d > kMaxNarrowD) {
    if (dtype == 0)
      metrics_rt<float><<<*nblocks, 256, 0, s>>>(n, d, (const float *)X, (const float *)Z, rows_local, tpr, npb, part);
    else
      metrics_rt<double><<<*nblocks, 256, 0, s>>>(n, d, (const double *)X, (const double *)Z, rows_local, tpr, npb, part);
    return cudaGetLastError();
  }
  const size_t sh = sizeof(double) * (size_t)(G * E3 > 256 ? G * E3 : 256);
  if (dtype == 0) {
    NSRGS_D_SWITCH(d, (metrics_kernel<float, D><<<*nblocks, 256, sh, s>>>(n, (const float *)X, (const float *)Z,
                                                                         rows_local, tpr, npb, part)));
  } else {
    NSRGS_D_SWITCH(d, (metrics_kernel<double, D><<<*nblocks, 256, sh, s>>>(n, (const double *)X, (const double *)Z,
                                                                          rows_local, tpr, npb, part)));
  }
  return cudaGetLastError();
}

cudaError_t launch_metrics_final(int d, int64_t n, const double *grams, double *out3, cudaStream_t s) {
  if (d > kMaxNarrowD) {
    metrics_final_rt<<<1, 32, 0, s>>>(n, d, grams, out3);
    return cudaGetLastError();
  }
  NSRGS_D_SWITCH(d, (metrics_final_kernel<D><<<1, 32, 0, s>>>(n, grams, out3)));
  return cudaGetLastError();
}

}  // namespace nsrgs
