// bsr.cu — block-sparse (BSR) storage of an incompletely observed instance
// (§4.1: the pair {i, j} is observed with probability p,
// unobserved blocks are zero; step size mu = 1/(np)).
//
// Storage: for every local node row i, only its observed blocks A_ij (j != i) are kept, in
// ascending j, each d x d row-major and contiguous; each row's block list is padded with zero
// blocks (column index = the row's own node, values 0) to a multiple of 4 blocks.  An A pass
// therefore reads ~p of the dense bytes.
//
// Generator (bsr_count / bsr_scan / bsr_fill): the same instance as the dense generator
// (aux.cu gen_A_*): observation test on Philox counter (min, max, 0, 4), W_ij from
// (min, max, q, 2) transposed for i > j, A_ij = round(Z_i Z_j^T + sigma W_ij) with the same
// fp64 expression, so every stored block is bitwise the dense block (tested).
//
// Pass, d <= 10 (bsr_kernel): one warp per node row, streamed in chunks of CH blocks through a
// per-warp software pipeline: the next chunk's A blocks arrive by one bulk copy (cp.async.bulk,
// mbarrier, L2 evict-first) into the other half of a double buffer, and the next chunk's X_j
// records by a cooperative gather into registers (consecutive lanes load consecutive float4 of
// one record of a padded node-major copy of X — 128 B = one L2 line per node at d = 5 — so
// every request is whole lines; per-lane scattered loads of X_j made the first version
// L1-bound at 98 % with 15 sectors per block), column indices two chunks ahead; meanwhile lane
// l multiplies block l/LPB of the current chunk by its X_j (record stride 4 mod 8 words:
// conflict-free per-lane LDS.64), accumulating B_i in registers as FFMA2 component
// pairs (LPB = 2 lanes per block for d >= 7, each owning half of the pairs).  The lanes'
// partial B_i are summed with shuffles and the per-node epilogue (epilogue.cuh) runs as in the
// dense kernel.  A caller's ragged rows (chunks not 16-byte aligned) are copied through
// registers instead of the bulk copy.  d > 10 (bsr_wide_kernel): lane = output component k, A
// blocks broadcast from smem, X_j column k read coalesced from the (row-major) wide X layout.
// Partials (objective / Gram terms): per-CTA slots, last CTA reduces in fixed order
// (bitwise-deterministic; the node -> warp assignment is static).
#include <cstdlib>

#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace nsrgs {

namespace {

__device__ __forceinline__ bool bsr_observed(int64_t i, int64_t j, uint64_t seed, double p_obs) {
  if (i == j) return false;
  if (p_obs >= 1.0) return true;
  const uint32_t lo = (uint32_t)min(i, j), hi = (uint32_t)max(i, j);
  const U4 v = philox4x32_10(lo, hi, 0u, 4u, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
  return uniform53(v.x, v.y) < p_obs;
}

__device__ __forceinline__ uint64_t bpack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void bunpack(uint64_t v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t bffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

constexpr int kGenThreads = 256;

// observed blocks per local row, padded to a multiple of 4
__global__ void bsr_count_kernel(int64_t n, int64_t node0, uint64_t seed, double p_obs, int64_t *cnt) {
  __shared__ int sh[kGenThreads / 32];
  const int64_t il = blockIdx.x, i = node0 + il;
  int c = 0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) c += bsr_observed(i, j, seed, p_obs) ? 1 : 0;
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kGenThreads / 32; ++w) t += sh[w];
    cnt[il] = (t + 3) & ~3;
  }
}

// rowptr[0] = 0, rowptr[il + 1] = sum_{m <= il} cnt[m]  (one CTA, 1024 threads, contiguous segments)
__global__ void bsr_scan_kernel(const int64_t *cnt, int64_t m, int64_t *rowptr) {
  __shared__ int64_t sh[1024];
  const int t = threadIdx.x;
  const int64_t seg = (m + 1023) / 1024, a = (int64_t)t * seg, b = min(m, a + seg);
  int64_t s = 0;
  for (int64_t k = a; k < b; ++k) s += cnt[k];
  sh[t] = s;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {   // Hillis-Steele inclusive scan of the segment sums
    const int64_t v = t >= off ? sh[t - off] : 0;
    __syncthreads();
    sh[t] += v;
    __syncthreads();
  }
  int64_t run = sh[t] - s;
  if (t == 0) rowptr[0] = 0;
  for (int64_t k = a; k < b; ++k) {
    run += cnt[k];
    rowptr[k + 1] = run;
  }
}

// Fill row il: observed j in ascending order (block prefix of the observation flags per chunk
// of 256 columns), values by the dense generator's expression; zero padding blocks at the end.
// ||A||_F^2 partial of the row -> part[il].
template <typename T>
__global__ void bsr_fill_kernel(int64_t n, int d, int64_t node0, uint64_t seed, double sigma, double p_obs,
                                const double *Z64, const int64_t *rowptr, int *col, T *vals, double *part) {
  __shared__ double Zi[kMaxD * kMaxD];
  __shared__ int woff[kGenThreads / 32 + 1];
  __shared__ double sh[32];
  const int64_t il = blockIdx.x, i = node0 + il;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int DD = d * d;
  for (int e = threadIdx.x; e < DD; e += blockDim.x) Zi[e] = Z64[i * DD + e];
  int64_t pos0 = rowptr[il];
  const int64_t end = rowptr[il + 1];
  double ss = 0.0;
  for (int64_t j0 = 0; j0 < n; j0 += blockDim.x) {
    const int64_t j = j0 + threadIdx.x;
    const bool obs = j < n && bsr_observed(i, j, seed, p_obs);
    const unsigned bal = __ballot_sync(0xffffffffu, obs);
    __syncthreads();   // Zi ready (first pass) / previous chunk's woff consumed
    if (lane == 0) woff[warp] = __popc(bal);
    __syncthreads();
    if (threadIdx.x == 0) {
      int run = 0;
      for (int w = 0; w <= kGenThreads / 32; ++w) {
        const int c = w < kGenThreads / 32 ? woff[w] : 0;
        woff[w] = run;
        run += c;
      }
    }
    __syncthreads();
    if (obs) {
      const int64_t pos = pos0 + woff[warp] + __popc(bal & ((1u << lane) - 1u));
      col[pos] = (int)j;
      T *Ab = vals + pos * DD;
      const double *Zj = Z64 + j * DD;
      const uint32_t lo = (uint32_t)min(i, j), hi = (uint32_t)max(i, j);
      const bool tr = i > j;
      for (int q = 0; q < (DD + 1) / 2; ++q) {
        double w[2];
        normal_pair(seed, lo, hi, (uint32_t)q, 2u, w[0], w[1]);
        for (int h = 0; h < 2; ++h) {
          const int e = 2 * q + h;
          if (e < DD) {
            const int a = tr ? e % d : e / d, b = tr ? e / d : e % d;   // position in A_ij
            double v = 0.0;
            for (int k = 0; k < d; ++k) v += Zi[a * d + k] * Zj[b * d + k];
            v += sigma * w[h];
            const T tv = (T)v;
            Ab[a * d + b] = tv;
            ss += (double)tv * (double)tv;
          }
        }
      }
    }
    pos0 += woff[kGenThreads / 32];
  }
  // zero padding blocks (contribute nothing): column = the row's last observed column (rows
  // stay sorted), or the row's own node if it observed none
  __syncthreads();
  const int pad_col = pos0 > rowptr[il] ? col[pos0 - 1] : (int)i;
  for (int64_t pos = pos0 + threadIdx.x; pos < end; pos += blockDim.x) {
    col[pos] = pad_col;
    for (int e = 0; e < DD; ++e) vals[pos * DD + e] = T(0);
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) sh[warp] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kGenThreads / 32; ++w) t += sh[w];
    part[il] = t;
  }
}

// sum of squares of a user-attached BSR value array (fp64 partial per CTA)
__global__ void bsr_sumsq_kernel(const float *vals, int64_t count, double *part) {
  __shared__ double sh[32];
  double ss = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x) {
    const double v = (double)vals[e];
    ss += v * v;
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

// ---------------------------------------------------------------------------------- pass
template <int D>
struct BsrCfg {
  static constexpr int DD = D * D;
  static constexpr int DP = D + (D & 1);                // even row stride of the padded X record
  static constexpr int DS = (D * DP + 3) / 4 * 4;       // node stride of the padded X copy (16 B;
                                                        // 128 B = one L2 line at d = 5)
  static constexpr int DSS = (DS % 8 == 4) ? DS : DS + 4;   // slab pass: 4 mod 8 words, so records
                                                        // read straight from a linear slab copy
                                                        // spread over the banks
  static constexpr int XSS = DSS;                       // smem record stride = 4 mod 8 words:
                                                        // conflict-free LDS.64 / LDS.128 per lane
  static constexpr int Q4 = DS / 4;                     // float4 per record
  static constexpr int KP = DP / 2;                     // component pairs
  static constexpr int LPB = D <= 6 ? 1 : 2;            // lanes per block
  static constexpr int NKP = (KP + LPB - 1) / LPB;      // pairs per lane
  static constexpr int CH = 32 / LPB;                   // blocks per chunk
  static constexpr int LX = (CH * Q4 + 31) / 32;        // chunk X float4 per lane (cooperative gather)
  static constexpr int W = D <= 6 ? 4 : 2;              // warps (nodes) per CTA
  static constexpr int E = DD, EP = (DD + 3) / 4 * 4;
  static constexpr int DDL = (DD + 31) / 32;
  static constexpr int NPART = 2 * DD + 2;
  static constexpr int SAB = (CH * DD + 3) / 4 * 4;     // one A chunk buffer (blocks contiguous)
  static constexpr int SXB = CH * XSS;                  // X record buffer
  static constexpr int SA = 2 * SAB + SXB;              // floats per warp: double-buffered A, one X buffer
  static constexpr int SMEM = W * (SA + 5 * EP) * 4 + W * NPART * 8 + W * 16 + 16;
};

// per-CTA partial slot + last-CTA fixed-order reduction (as wide.cu)
template <int NPART, int W>
__device__ __forceinline__ void bsr_partials(const PanelParams &p, double *red, int *flag, int warp, int lane,
                                             const double *g1s, const double *g2s, int DD, int DDL, double so,
                                             double xs) {
  so = warp_sum(so);
  xs = warp_sum(xs);
  double *rw = red + warp * NPART;
  for (int m = 0; m < DDL; ++m) {
    const int e2 = lane + 32 * m;
    if (e2 < DD) { rw[e2] = g1s[m]; rw[DD + e2] = g2s[m]; }
  }
  if (lane == 0) { rw[2 * DD] = so; rw[2 * DD + 1] = xs; }
  __syncthreads();
  for (int i = threadIdx.x; i < NPART; i += W * 32) {
    double v = 0.0;
    for (int w = 0; w < W; ++w) v += red[w * NPART + i];
    __stcg(p.cta_part + (int64_t)blockIdx.x * NPART + i, v);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_gpu();
    const int is_last = (atomicAdd(p.done_cnt, 1u) == gridDim.x - 1);
    if (is_last) fence_acq_rel_gpu();
    *flag = is_last;
  }
  __syncthreads();
  if (*flag) {
    for (int i = warp; i < NPART; i += W) {
      double v = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(p.cta_part + (int64_t)b * NPART + i);
      v = warp_sum(v);
      if (lane == 0) p.result[i] = v;
    }
    if (threadIdx.x == 0) *p.done_cnt = 0u;
  }
}

template <int D, int MODE>
__global__ void __launch_bounds__(32 * BsrCfg<D>::W) bsr_kernel(const BsrParams bp) {
  using C = BsrCfg<D>;
  extern __shared__ float4 smem4[];
  float *smem = reinterpret_cast<float *>(smem4);
  const PanelParams &p = bp.e;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float *sA = smem + warp * C::SA;          // [2][SAB]: A chunks (double-buffered, bulk-copy target)
  float *sXr = sA + 2 * C::SAB;             // [2][CH][XSS]: X_j records of the chunk (bulk-copy target)
  float *scr = smem + C::W * C::SA + warp * 5 * C::EP;
  double *red = reinterpret_cast<double *>(smem + C::W * (C::SA + 5 * C::EP));
  uint64_t *bar = reinterpret_cast<uint64_t *>(red + C::W * C::NPART) + 2 * warp;
  int *flag = reinterpret_cast<int *>(reinterpret_cast<uint64_t *>(red + C::W * C::NPART) + 2 * C::W);
  const int64_t il = (int64_t)blockIdx.x * C::W + warp;
  const int nvalid = il < p.n_local ? 1 : 0;
  const int h = lane % C::LPB, blane = lane / C::LPB;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncwarp();

  uint64_t acc2[D][C::NKP];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int t = 0; t < C::NKP; ++t) acc2[a][t] = 0ull;
  if (nvalid) {
    const int64_t r0 = bp.rowptr[il], r1 = bp.rowptr[il + 1];
    const int nb = (int)(r1 - r0), nch = (nb + C::CH - 1) / C::CH;
    // whole-chunk bulk copies of A need 16-byte aligned chunks: rows padded to 4 blocks (the
    // generator's layout) when d is odd, any row when d is even; otherwise (a caller's ragged
    // BSR) the A chunk is copied through registers
    const bool tma = ((r0 * C::DD) & 3) == 0 && (((int64_t)nb * C::DD) & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(bp.vals) & 15) == 0;
    const uint64_t pol_a = policy_evict_first(), pol_x = policy_evict_last();
    auto cnt_of = [&](int k) { return min(C::CH, nb - k * C::CH); };
    auto col_of = [&](int k) -> int {
      if (k >= nch) return 0;
      return blane < cnt_of(k) ? __ldg(bp.col + r0 + (int64_t)k * C::CH + blane) : 0;
    };
    // chunk k -> A buffer buf: one bulk copy (or the register path for ragged rows)
    auto load_A = [&](int k, int buf) {
      const int cnt = cnt_of(k);
      const float *src = bp.vals + (r0 + (int64_t)k * C::CH) * C::DD;
      float *dst = sA + buf * C::SAB;
      if (tma) {
        if (lane == 0) {
          // the buffer's previous contents were read through the generic proxy (chunk k - 2)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive_expect_tx(&bar[buf], (uint32_t)(cnt * C::DD * 4));
          bulk_load(dst, src, (uint32_t)(cnt * C::DD * 4), &bar[buf], pol_a);
        }
      } else {
        for (int e = lane; e < cnt * C::DD; e += 32) dst[e] = __ldcs(src + e);
      }
    };
    // X_j records of chunk k, gathered cooperatively into registers: consecutive lanes load
    // consecutive float4 of one record (whole 128-byte lines per request).  Unconditional: slots
    // past the chunk read a valid record (col_of gives node 0) that is never stored — a
    // predicated select would make the consumer wait for the load.  (One bulk copy per record
    // instead was 1.5-2x slower: the TMA unit takes ~5 cycles per small copy.)
    auto gather_X = [&](int jk, float4 (&xv)[C::LX]) {
#pragma unroll
      for (int m = 0; m < C::LX; ++m) {
        const int sl = lane + 32 * m, r = sl / C::Q4, q = sl - r * C::Q4;
        const int jr = __shfl_sync(0xffffffffu, jk, (r * C::LPB) & 31);
        xv[m] = __ldg(reinterpret_cast<const float4 *>(bp.Xs + (int64_t)jr * C::DS) + q);
      }
    };
    auto store_X = [&](int k, const float4 (&xv)[C::LX]) {
      const int cnt = cnt_of(k);
#pragma unroll
      for (int m = 0; m < C::LX; ++m) {
        const int sl = lane + 32 * m, r = sl / C::Q4, q = sl - r * C::Q4;
        if (r < cnt) *reinterpret_cast<float4 *>(sXr + r * C::XSS + 4 * q) = xv[m];
      }
    };
    // software pipeline: column indices two chunks ahead, A one chunk ahead (bulk copy into the
    // other buffer), X_j of the next chunk in registers while the current chunk is multiplied
    int jn = col_of(1);
    load_A(0, 0);
    {
      float4 xv[C::LX];
      gather_X(col_of(0), xv);
      store_X(0, xv);
    }
    __syncwarp();
    for (int k = 0; k < nch; ++k) {
      const int buf = k & 1;
      const int jnn = col_of(k + 2);
      float4 xv[C::LX];
      if (k + 1 < nch) {
        load_A(k + 1, buf ^ 1);
        gather_X(jn, xv);
      }
      if (tma) mbar_wait(&bar[buf], (uint32_t)((k >> 1) & 1));
      if (blane < cnt_of(k)) {
        const float *xr = sXr + blane * C::XSS;
        uint64_t xp[D][C::NKP];
        if constexpr (C::LPB == 1) {
          // whole record as LDS.128 (record stride 4 mod 8 words: conflict-free per quarter warp);
          // every pair (2kp, 2kp+1) sits at an even offset, i.e. inside one float4
          uint64_t rec[C::DS / 2];
#pragma unroll
          for (int q = 0; q < C::Q4; ++q) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(xr + 4 * q);
            rec[2 * q] = v.x;
            rec[2 * q + 1] = v.y;
          }
#pragma unroll
          for (int c = 0; c < D; ++c)
#pragma unroll
            for (int t = 0; t < C::NKP; ++t) xp[c][t] = rec[(c * C::DP) / 2 + t];
        } else {
#pragma unroll
          for (int c = 0; c < D; ++c)
#pragma unroll
            for (int t = 0; t < C::NKP; ++t) {
              const int kp = h + t * C::LPB;
              xp[c][t] = kp < C::KP ? *reinterpret_cast<const unsigned long long *>(xr + c * C::DP + 2 * kp) : 0ull;
            }
        }
        const float *ab = sA + buf * C::SAB + blane * C::DD;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const float av = ab[a * D + c];
            const uint64_t b2 = bpack(av, av);
#pragma unroll
            for (int t = 0; t < C::NKP; ++t) acc2[a][t] = bffma2(b2, xp[c][t], acc2[a][t]);
          }
      }
      __syncwarp();   // A buffer `buf` and the X records are free
      if (k + 1 < nch) store_X(k + 1, xv);
      __syncwarp();
      jn = jnn;
    }
  }
  // sum the lanes' partial B_i over lanes with the same pair set (h)
  float *sX = scr, *sG = sX + C::EP, *sH = sG + C::EP, *sS = sH + C::EP, *sM = sS + C::EP;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int t = 0; t < C::NKP; ++t) {
      float lo, hi;
      bunpack(acc2[a][t], lo, hi);
#pragma unroll
      for (int o = 16; o >= C::LPB; o >>= 1) {
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
      }
      const int kp = h + t * C::LPB;
      if (lane < C::LPB && kp < C::KP) {
        sG[a * D + 2 * kp] = lo;
        if (2 * kp + 1 < D) sG[a * D + 2 * kp + 1] = hi;
      }
    }
  __syncwarp();
  double g1s[C::DDL], g2s[C::DDL], so = 0.0, xs = 0.0;
  float ns_region = 0.f;
  int err = 0;
  node_epilogue<float, D, 1, MODE>(p, static_cast<const float *>(p.X), p.Xout, lane, il, nvalid, sX, sG, sH, sS, sM,
                                   g1s, g2s, so, xs, ns_region, err);
  if (err) atomicOr(p.err, err);
  if (lane == 0 && ns_region > 0.f) atomicMax(p.ns_region, __float_as_uint(ns_region));
  bsr_partials<C::NPART, C::W>(p, red, flag, warp, lane, g1s, g2s, C::DD, C::DDL, so, xs);
}

// ---------------------------------------------------------------------------------- gather4 pass
// As bsr_kernel, but the chunk's X_j records arrive by TMA tile::gather4 (UTMALDG.2D.GATHER4:
// 4 rows of the padded X copy, viewed as an n x DSS tensor, by row index per instruction) into a
// double-buffered smem area at the conflict-free record stride, on the same mbarrier as the
// chunk's A bulk copy: 8 + 1 TMA operations per 32 blocks, no LSU gather, no register staging.
template <int D>
struct BsrG4Cfg {
  using B = BsrCfg<D>;
  static constexpr int W = 4;
  // TMA tensor destinations are 128-byte aligned: a gather group (4 records of DSS floats) starts
  // at a multiple of 32 floats, so record r sits at (r / 4) GS + (r % 4) DSS (<= 2-way bank
  // conflicts on the per-lane record reads)
  static constexpr int GS = (4 * B::DSS + 31) / 32 * 32;
  static constexpr int SXB = (B::CH / 4) * GS;
  static constexpr int SAB = (B::SAB + 31) / 32 * 32;   // keeps every buffer 128-byte aligned
  static constexpr int SA = 2 * SXB + 2 * SAB;
  static constexpr int SMEM = 128 + W * (SA + 5 * B::EP) * 4 + W * B::NPART * 8 + W * 16 + 16;
};

__device__ __forceinline__ void tma_gather4(void *smem_dst, const void *tmap, uint64_t *bar, int c0, int r0, int r1,
                                            int r2, int r3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "l"(policy)
      : "memory");
}

template <int D, int MODE>
__global__ void __launch_bounds__(32 * BsrG4Cfg<D>::W) bsr_g4_kernel(const __grid_constant__ CUtensorMap tmX,
                                                                     const BsrParams bp) {
  using B = BsrCfg<D>;
  using C = BsrG4Cfg<D>;
  extern __shared__ float4 smem4[];
  uint8_t *raw = reinterpret_cast<uint8_t *>(smem4);
  float *smem = reinterpret_cast<float *>(raw + (((smem_u32(raw) + 127u) & ~127u) - smem_u32(raw)));   // 128 B
  const PanelParams &p = bp.e;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float *sXr = smem + warp * C::SA;         // [2][CH/4][GS]: gather4 targets
  float *sA = sXr + 2 * C::SXB;             // [2][SAB]
  float *scr = smem + C::W * C::SA + warp * 5 * B::EP;
  double *red = reinterpret_cast<double *>(smem + C::W * (C::SA + 5 * B::EP));
  uint64_t *bar = reinterpret_cast<uint64_t *>(red + C::W * B::NPART) + 2 * warp;
  int *flag = reinterpret_cast<int *>(reinterpret_cast<uint64_t *>(red + C::W * B::NPART) + 2 * C::W);
  const int64_t il = (int64_t)blockIdx.x * C::W + warp;
  const int nvalid = il < p.n_local ? 1 : 0;
  if (lane == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    prefetch_tmap(&tmX);
  }
  __syncwarp();

  uint64_t acc2[D][B::NKP];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int t = 0; t < B::NKP; ++t) acc2[a][t] = 0ull;
  if (nvalid) {
    const int64_t r0 = bp.rowptr[il], r1 = bp.rowptr[il + 1];
    const int nb = (int)(r1 - r0), nch = (nb + B::CH - 1) / B::CH;
    const bool tma = ((r0 * B::DD) & 3) == 0 && (((int64_t)nb * B::DD) & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(bp.vals) & 15) == 0;
    const uint64_t pol_a = policy_evict_first(), pol_x = policy_evict_last();
    auto cnt_of = [&](int k) { return min(B::CH, nb - k * B::CH); };
    auto col_of = [&](int k) -> int {
      if (k >= nch) return 0;
      const int c = cnt_of(k);
      return __ldg(bp.col + r0 + (int64_t)k * B::CH + min(lane, c - 1));   // past the chunk: its last column
    };
    // chunk k -> buffers buf: A (one bulk copy, or registers for ragged rows) and the X records
    // (gather4 by groups of 4 blocks), all completing on bar[buf]
    auto issue = [&](int k, int buf, int jk) {
      const int cnt = cnt_of(k), ng = (cnt + 3) >> 2;
      const float *src = bp.vals + (r0 + (int64_t)k * B::CH) * B::DD;
      float *dst = sA + buf * C::SAB;
      const int g0 = __shfl_sync(0xffffffffu, jk, (4 * lane) & 31), g1 = __shfl_sync(0xffffffffu, jk, (4 * lane + 1) & 31);
      const int g2 = __shfl_sync(0xffffffffu, jk, (4 * lane + 2) & 31), g3 = __shfl_sync(0xffffffffu, jk, (4 * lane + 3) & 31);
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(&bar[buf], (uint32_t)((tma ? cnt * B::DD * 4 : 0) + ng * 4 * B::DSS * 4));
      }
      __syncwarp();
      if (lane < ng) tma_gather4(sXr + buf * C::SXB + lane * C::GS, &tmX, &bar[buf], 0, g0, g1, g2, g3, pol_x);
      if (tma) {
        if (lane == 0) bulk_load(dst, src, (uint32_t)(cnt * B::DD * 4), &bar[buf], pol_a);
      } else {
        for (int e = lane; e < cnt * B::DD; e += 32) dst[e] = __ldcs(src + e);
      }
    };
    int jn = col_of(1);
    issue(0, 0, col_of(0));
    for (int k = 0; k < nch; ++k) {
      const int buf = k & 1;
      const int jnn = col_of(k + 2);
      if (k + 1 < nch) issue(k + 1, buf ^ 1, jn);
      mbar_wait(&bar[buf], (uint32_t)((k >> 1) & 1));
      __syncwarp();   // register-path A stores of this chunk (ragged rows) visible to all lanes
      if (lane < cnt_of(k)) {
        const float *xr = sXr + buf * C::SXB + (lane >> 2) * C::GS + (lane & 3) * B::DSS;
        uint64_t rec[B::DS / 2];
#pragma unroll
        for (int q = 0; q < B::Q4; ++q) {
          const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(xr + 4 * q);
          rec[2 * q] = v.x;
          rec[2 * q + 1] = v.y;
        }
        const float *ab = sA + buf * C::SAB + lane * B::DD;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int c = 0; c < D; ++c) {
            const float av = ab[a * D + c];
            const uint64_t b2 = bpack(av, av);
#pragma unroll
            for (int t = 0; t < B::NKP; ++t) acc2[a][t] = bffma2(b2, rec[(c * B::DP) / 2 + t], acc2[a][t]);
          }
      }
      __syncwarp();   // buffers `buf` are free for chunk k + 2
      jn = jnn;
    }
  }
  float *sX = scr, *sG = sX + B::EP, *sH = sG + B::EP, *sS = sH + B::EP, *sM = sS + B::EP;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int t = 0; t < B::NKP; ++t) {
      float lo, hi;
      bunpack(acc2[a][t], lo, hi);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
      }
      if (lane == 0 && t < B::KP) {
        sG[a * D + 2 * t] = lo;
        if (2 * t + 1 < D) sG[a * D + 2 * t + 1] = hi;
      }
    }
  __syncwarp();
  double g1s[B::DDL], g2s[B::DDL], so = 0.0, xs = 0.0;
  float ns_region = 0.f;
  int err = 0;
  node_epilogue<float, D, 1, MODE>(p, static_cast<const float *>(p.X), p.Xout, lane, il, nvalid, sX, sG, sH, sS, sM,
                                   g1s, g2s, so, xs, ns_region, err);
  if (err) atomicOr(p.err, err);
  if (lane == 0 && ns_region > 0.f) atomicMax(p.ns_region, __float_as_uint(ns_region));
  bsr_partials<B::NPART, C::W>(p, red, flag, warp, lane, g1s, g2s, B::DD, B::DDL, so, xs);
}

// ---------------------------------------------------------------------------------- slab pass
// Rows sorted by column (the generator's layout), d <= 6: the CTA's W rows walk their sorted
// block lists in lockstep, and one producer warp streams the X records of each column group of
// G nodes ONCE per CTA as a single bulk copy into an S-slot ring (full / empty mbarriers), which
// every row's lanes read directly (record stride 4 mod 8 words).  A chunks arrive per warp by
// bulk copy as in bsr_kernel.  Against bsr_kernel this removes the per-block X gather from the
// LSU pipe (LDG + STS + LDS, ~96 wavefronts per 32 blocks -> LDS only) and divides the L2->SM X
// traffic by the number of CTA rows observing each column (~W p).
// Group g lives in slot g % S; a warp releases group g (arrives on empty) only after waiting for
// its slab (full), so arrivals never run ahead of the slot's phase; it waits at most for groups
// below its own release point + S - 1 (chunks spanning more groups are processed in windows),
// so the ring cannot deadlock.
// Two ring shapes (same 36 KB): 4 slots of 9 KB (G <= 64 at d = 5), the default for p >= 0.75,
// and 8 slots of 4.5 KB (G <= 32: more groups of slack between the CTA's rows), opt-in.
template <int D, int RS = 4>
struct BsrSlabCfg {
  using B = BsrCfg<D>;
  static constexpr int W = 8;                  // consumer warps (rows) per CTA
  static constexpr int NW = W + 1;             // + producer warp
  static constexpr int S = RS;                 // slab slots
  static constexpr int SLAB = RS == 4 ? 2304 : 1152;   // floats per slot (9 KB / 4.5 KB)
  static constexpr int GMAX = SLAB / B::DSS;    // nodes per column group, at most
  static constexpr int SMEM = (S * SLAB + W * (2 * B::SAB + 5 * B::EP)) * 4 + NW * B::NPART * 8 + (2 * S + 2 * W) * 8 + 16;
};

template <int D, int MODE, int RS>
__global__ void __launch_bounds__(32 * BsrSlabCfg<D, RS>::NW) bsr_slab_kernel(const BsrParams bp, int lg2g) {
  using B = BsrCfg<D>;
  using C = BsrSlabCfg<D, RS>;
  extern __shared__ float4 smem4[];
  float *smem = reinterpret_cast<float *>(smem4);
  const PanelParams &p = bp.e;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float *slab = smem;                                          // [S][SLAB]
  float *sAw = smem + C::S * C::SLAB + warp * (2 * B::SAB);    // this warp's A double buffer
  float *scr = smem + C::S * C::SLAB + C::W * 2 * B::SAB + warp * 5 * B::EP;
  double *red = reinterpret_cast<double *>(smem + C::S * C::SLAB + C::W * (2 * B::SAB + 5 * B::EP));
  uint64_t *full = reinterpret_cast<uint64_t *>(red + C::NW * B::NPART);
  uint64_t *empty = full + C::S;
  uint64_t *abar = empty + C::S + 2 * warp;
  int *flag = reinterpret_cast<int *>(empty + C::S + 2 * C::W);
  const int G = 1 << lg2g;
  const int ngroups = (int)((p.n + G - 1) >> lg2g);
  if (threadIdx.x == 0) {
    for (int k = 0; k < C::S; ++k) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], C::W);
    }
  }
  if (warp < C::W && lane == 0) {
    mbar_init(&abar[0], 1);
    mbar_init(&abar[1], 1);
  }
  if (threadIdx.x == 0) fence_mbar_init();
  __syncthreads();

  double g1s[B::DDL], g2s[B::DDL], so = 0.0, xs = 0.0;
#pragma unroll
  for (int m = 0; m < B::DDL; ++m) g1s[m] = g2s[m] = 0.0;
  if (warp == C::W) {   // ------------------------------------------------ slab producer
    if (lane == 0) {
      const uint64_t pol_x = policy_evict_last();
      for (int g = 0; g < ngroups; ++g) {
        const int slot = g % C::S;
        if (g >= C::S) mbar_wait(&empty[slot], (uint32_t)(((g / C::S) - 1) & 1));
        const int64_t n0 = (int64_t)g << lg2g;
        const int cntn = (int)min((int64_t)G, p.n - n0);
        const uint32_t bytes = (uint32_t)(cntn * B::DSS * 4);
        mbar_arrive_expect_tx(&full[slot], bytes);
        bulk_load(slab + slot * C::SLAB, bp.Xs + n0 * B::DSS, bytes, &full[slot], pol_x);
      }
    }
    __syncwarp();
    bsr_partials<B::NPART, C::NW>(p, red, flag, warp, lane, g1s, g2s, B::DD, B::DDL, so, xs);
    return;
  }

  // ------------------------------------------------------------------ consumer warp = one row
  const int64_t il = (int64_t)blockIdx.x * C::W + warp;
  const int nvalid = il < p.n_local ? 1 : 0;
  int gdone = 0;   // groups < gdone released by this warp
  auto release_to = [&](int gend) {   // release groups [gdone, gend): wait for the slab, then arrive
    if (lane == 0)
      for (int g = gdone; g < gend; ++g) {
        mbar_wait(&full[g % C::S], (uint32_t)((g / C::S) & 1));
        mbar_arrive(&empty[g % C::S]);
      }
    gdone = max(gdone, gend);
  };
  uint64_t acc2[D][B::NKP];
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int t = 0; t < B::NKP; ++t) acc2[a][t] = 0ull;
  if (nvalid) {
    const int64_t r0 = bp.rowptr[il], r1 = bp.rowptr[il + 1];
    const int nb = (int)(r1 - r0), nch = (nb + B::CH - 1) / B::CH;
    const bool tma = ((r0 * B::DD) & 3) == 0 && (((int64_t)nb * B::DD) & 3) == 0 &&
                     (reinterpret_cast<uintptr_t>(bp.vals) & 15) == 0;
    const uint64_t pol_a = policy_evict_first();
    auto cnt_of = [&](int k) { return min(B::CH, nb - k * B::CH); };
    auto load_A = [&](int k, int buf) {
      const int cnt = cnt_of(k);
      const float *src = bp.vals + (r0 + (int64_t)k * B::CH) * B::DD;
      float *dst = sAw + buf * B::SAB;
      if (tma) {
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive_expect_tx(&abar[buf], (uint32_t)(cnt * B::DD * 4));
          bulk_load(dst, src, (uint32_t)(cnt * B::DD * 4), &abar[buf], pol_a);
        }
      } else {
        for (int e = lane; e < cnt * B::DD; e += 32) dst[e] = __ldcs(src + e);
      }
    };
    auto col_of = [&](int k) -> int {
      if (k >= nch) return 0;
      const int c = cnt_of(k);
      return __ldg(bp.col + r0 + (int64_t)k * B::CH + min(lane, c - 1));   // past the chunk: its last column
    };
    int jc = col_of(0), jn = col_of(1);
    load_A(0, 0);
    for (int k = 0; k < nch; ++k) {
      const int buf = k & 1;
      const int jnn = col_of(k + 2);
      if (k + 1 < nch) load_A(k + 1, buf ^ 1);
      const int cnt = cnt_of(k);
      const int gl = __shfl_sync(0xffffffffu, jc, cnt - 1) >> lg2g;
      int glo = __shfl_sync(0xffffffffu, jc, 0) >> lg2g;
      release_to(glo);
      if (tma) mbar_wait(&abar[buf], (uint32_t)((k >> 1) & 1));
      __syncwarp();
      const int gme = jc >> lg2g;
      const float *ab = sAw + buf * B::SAB + lane * B::DD;
      while (glo <= gl) {   // windows of at most S - 1 groups
        const int ghi = min(gl, glo + C::S - 2);
        for (int g = glo; g <= ghi; ++g) mbar_wait(&full[g % C::S], (uint32_t)((g / C::S) & 1));
        if (lane < cnt && gme >= glo && gme <= ghi) {
          const float *xr = slab + (gme % C::S) * C::SLAB + (jc - (gme << lg2g)) * B::DSS;
          uint64_t rec[B::DSS / 2];
#pragma unroll
          for (int q = 0; q < B::Q4; ++q) {
            const ulonglong2 v = *reinterpret_cast<const ulonglong2 *>(xr + 4 * q);
            rec[2 * q] = v.x;
            rec[2 * q + 1] = v.y;
          }
#pragma unroll
          for (int a = 0; a < D; ++a)
#pragma unroll
            for (int c = 0; c < D; ++c) {
              const float av = ab[a * D + c];
              const uint64_t b2 = bpack(av, av);
#pragma unroll
              for (int t = 0; t < B::NKP; ++t) acc2[a][t] = bffma2(b2, rec[(c * B::DP) / 2 + t], acc2[a][t]);
            }
        }
        __syncwarp();
        if (ghi < gl) release_to(ghi + 1);
        glo = ghi + 1;
      }
      jc = jn;
      jn = jnn;
    }
  }
  release_to(ngroups);
  // sum the lanes' partial B_i, then the per-node epilogue and the CTA partials
  float *sX = scr, *sG = sX + B::EP, *sH = sG + B::EP, *sS = sH + B::EP, *sM = sS + B::EP;
#pragma unroll
  for (int a = 0; a < D; ++a)
#pragma unroll
    for (int t = 0; t < B::NKP; ++t) {
      float lo, hi;
      bunpack(acc2[a][t], lo, hi);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lo += __shfl_xor_sync(0xffffffffu, lo, o);
        hi += __shfl_xor_sync(0xffffffffu, hi, o);
      }
      if (lane == 0 && t < B::KP) {
        sG[a * D + 2 * t] = lo;
        if (2 * t + 1 < D) sG[a * D + 2 * t + 1] = hi;
      }
    }
  __syncwarp();
  float ns_region = 0.f;
  int err = 0;
  node_epilogue<float, D, 1, MODE>(p, static_cast<const float *>(p.X), p.Xout, lane, il, nvalid, sX, sG, sH, sS, sM,
                                   g1s, g2s, so, xs, ns_region, err);
  if (err) atomicOr(p.err, err);
  if (lane == 0 && ns_region > 0.f) atomicMax(p.ns_region, __float_as_uint(ns_region));
  bsr_partials<B::NPART, C::NW>(p, red, flag, warp, lane, g1s, g2s, B::DD, B::DDL, so, xs);
}

// d > 10: lane = output component; CHW blocks per chunk staged in smem with a 16-byte row stride
template <int D>
struct BsrWideCfg {
  static constexpr int DD = D * D;
  static constexpr int D4 = (D + 3) / 4 * 4;            // smem row stride (float4 broadcast reads)
  static constexpr int CHW = 2;                          // blocks per chunk (per warp)
  static constexpr int LD = (CHW * DD + 31) / 32;
  static constexpr int W = 8;                            // warps splitting ONE node row (CTA = node)
  static constexpr int E = DD, EP = (DD + 3) / 4 * 4;
  static constexpr int DDL = (DD + 31) / 32;
  static constexpr int NPART = 2 * DD + 2;
  static constexpr int SA = CHW * D * D4;
  static constexpr int SRED = W * D * 32;                // per-warp partial B rows (lane = component)
  static constexpr int SMEM = (W * SA + SRED + 5 * EP) * 4 + W * NPART * 8 + 16;
};

// One CTA per node row; its W warps take the row's blocks round-robin by chunks of CHW (the
// Table 1 sizes have n = 500 rows: one warp per row left ~3 warps per SM), and warp 0 sums the
// W partial B_i in fixed order and runs the epilogue.
template <int D, int MODE>
__global__ void __launch_bounds__(32 * BsrWideCfg<D>::W) bsr_wide_kernel(const BsrParams bp) {
  using C = BsrWideCfg<D>;
  extern __shared__ float4 smem4[];
  float *smem = reinterpret_cast<float *>(smem4);
  const PanelParams &p = bp.e;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float *sA = smem + warp * C::SA;
  float *sred = smem + C::W * C::SA;                     // [W][D][32]
  float *scr = sred + C::SRED;
  double *red = reinterpret_cast<double *>(scr + 5 * C::EP);
  int *flag = reinterpret_cast<int *>(red + C::W * C::NPART);
  const int64_t il = blockIdx.x;
  const int nvalid = il < p.n_local ? 1 : 0;
  const int kk = lane < D ? lane : D - 1;
  // zero the row padding columns once (never written by the chunk copies)
  for (int e = lane; e < C::SA; e += 32) sA[e] = 0.f;
  __syncwarp();
  uint64_t acc2[D];   // (even-column, odd-column) partial sums of row a, component `lane`
#pragma unroll
  for (int a = 0; a < D; ++a) acc2[a] = 0ull;
  const float *Xg = static_cast<const float *>(p.X);
  if (nvalid) {
    const int64_t r0 = bp.rowptr[il], r1 = bp.rowptr[il + 1];
    for (int64_t b0 = r0 + (int64_t)warp * C::CHW; b0 < r1; b0 += (int64_t)C::W * C::CHW) {
      const int cnt = (int)min((int64_t)C::CHW, r1 - b0);
      const int tot = cnt * C::DD;
      const float *src = bp.vals + b0 * C::DD;
      float v[C::LD];
#pragma unroll
      for (int m = 0; m < C::LD; ++m) {
        const int e = lane + 32 * m;
        v[m] = e < tot ? __ldcs(src + e) : 0.f;
      }
#pragma unroll
      for (int m = 0; m < C::LD; ++m) {
        const int e = lane + 32 * m;
        if (e < tot) {
          const int blk = e / C::DD, r = e - blk * C::DD, a = r / D, c = r - a * D;
          sA[(blk * D + a) * C::D4 + c] = v[m];
        }
      }
      __syncwarp();
      for (int bb = 0; bb < cnt; ++bb) {
        const int j = __ldg(bp.col + b0 + bb);
        // X_j rows are contiguous in the wide layout (a node never straddles a rank slice)
        const int g = j / (int)p.n_local, jl = j - g * (int)p.n_local;
        const float *xj = Xg + ((int64_t)g * p.tiles_per_rank * kWideColTile + (int64_t)jl * D) * D + kk;
        uint64_t xq[C::D4 / 2];
#pragma unroll
        for (int c2 = 0; c2 < C::D4 / 2; ++c2) {
          const int c0 = 2 * c2, c1 = 2 * c2 + 1;
          const float x0 = c0 < D ? __ldg(xj + c0 * D) : 0.f;
          const float x1 = c1 < D ? __ldg(xj + c1 * D) : 0.f;
          xq[c2] = bpack(x0, x1);
        }
        const float *ab = sA + bb * D * C::D4;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
          for (int c4 = 0; c4 < C::D4 / 4; ++c4) {
            const ulonglong2 av = *reinterpret_cast<const ulonglong2 *>(ab + a * C::D4 + 4 * c4);   // broadcast
            acc2[a] = bffma2(av.x, xq[2 * c4], acc2[a]);
            acc2[a] = bffma2(av.y, xq[2 * c4 + 1], acc2[a]);
          }
      }
      __syncwarp();
    }
  }
  // the W partial rows -> smem; warp 0 sums them in warp order (deterministic)
#pragma unroll
  for (int a = 0; a < D; ++a) {
    float lo, hi;
    bunpack(acc2[a], lo, hi);
    sred[(warp * D + a) * 32 + lane] = lo + hi;
  }
  __syncthreads();
  double g1s[C::DDL], g2s[C::DDL], so = 0.0, xs = 0.0;
#pragma unroll
  for (int m = 0; m < C::DDL; ++m) g1s[m] = g2s[m] = 0.0;
  if (warp == 0) {
    float *sX = scr, *sG = sX + C::EP, *sH = sG + C::EP, *sS = sH + C::EP, *sM = sS + C::EP;
    for (int a = 0; a < D; ++a) {
      float t = 0.f;
      for (int w = 0; w < C::W; ++w) t += sred[(w * D + a) * 32 + lane];
      if (lane < D) sG[a * D + lane] = t;   // entry (a, b = lane) of B_i
    }
    __syncwarp();
    float ns_region = 0.f;
    int err = 0;
    node_epilogue<float, D, 1, MODE>(p, Xg, p.Xout, lane, il, nvalid, sX, sG, sH, sS, sM, g1s, g2s, so, xs, ns_region,
                                     err);
    if (err) atomicOr(p.err, err);
    if (lane == 0 && ns_region > 0.f) atomicMax(p.ns_region, __float_as_uint(ns_region));
  }
  bsr_partials<C::NPART, C::W>(p, red, flag, warp, lane, g1s, g2s, C::DD, C::DDL, so, xs);
}

// tile layout X -> padded node-major copy (record of DS floats per node, row stride DP, zeros
// in the padding), d <= 10
template <int D>
__global__ void bsr_pack_x_kernel(const float *X, float *Xs, int64_t n, int64_t rows_local, int64_t tpr, int ds) {
  using C = BsrCfg<D>;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * ds) return;
  const int64_t j = idx / ds;
  const int r = (int)(idx - j * ds), c = r / C::DP, k = r - c * C::DP;
  Xs[idx] = (c < D && k < D) ? X[tile_index(j * D + c, k, D, rows_local, tpr)] : 0.f;
}

template <int D, int MODE>
cudaError_t bsr_launch(const BsrParams &bp, cudaStream_t s) {
  if constexpr (D <= kMaxNarrowD) {
    using C = BsrCfg<D>;
    auto kern = bsr_kernel<D, MODE>;
    static bool attr[64] = {};
    {
      const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void *>(kern), C::SMEM, attr);
      if (e != cudaSuccess) return e;
    }
    const unsigned grid = (unsigned)((bp.e.n_local + C::W - 1) / C::W);
    kern<<<grid, 32 * C::W, C::SMEM, s>>>(bp);
  } else {
    using C = BsrWideCfg<D>;
    auto kern = bsr_wide_kernel<D, MODE>;
    static bool attr[64] = {};
    {
      const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void *>(kern), C::SMEM, attr);
      if (e != cudaSuccess) return e;
    }
    const unsigned grid = (unsigned)bp.e.n_local;   // one CTA per node row
    kern<<<grid, 32 * C::W, C::SMEM, s>>>(bp);
  }
  return cudaGetLastError();
}

template <int D, int MODE, int RS>
cudaError_t bsr_slab_launch(const BsrParams &bp, int lg2g, cudaStream_t s) {
  if constexpr (D <= 6) {
    using C = BsrSlabCfg<D, RS>;
    auto kern = bsr_slab_kernel<D, MODE, RS>;
    static bool attr[64] = {};
    {
      const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void *>(kern), C::SMEM, attr);
      if (e != cudaSuccess) return e;
    }
    const unsigned grid = (unsigned)((bp.e.n_local + C::W - 1) / C::W);
    kern<<<grid, 32 * C::NW, C::SMEM, s>>>(bp, lg2g);
    return cudaGetLastError();
  } else {
    return cudaErrorInvalidValue;
  }
}

template <int D, int MODE>
cudaError_t bsr_g4_launch(const BsrParams &bp, const CUtensorMap *tmX, cudaStream_t s) {
  if constexpr (D <= 6) {
    using C = BsrG4Cfg<D>;
    auto kern = bsr_g4_kernel<D, MODE>;
    static bool attr[64] = {};
    {
      const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void *>(kern), C::SMEM, attr);
      if (e != cudaSuccess) return e;
    }
    const unsigned grid = (unsigned)((bp.e.n_local + C::W - 1) / C::W);
    kern<<<grid, 32 * C::W, C::SMEM, s>>>(*tmX, bp);
    return cudaGetLastError();
  } else {
    return cudaErrorInvalidValue;
  }
}

template <int D>
cudaError_t bsr_mode_switch(int mode, const BsrParams &bp, int lg2g, const CUtensorMap *tmX, cudaStream_t s) {
  if (lg2g < 0 && tmX && D <= 6) {
    switch (mode) {
      case kModeRgs: return bsr_g4_launch<D, kModeRgs>(bp, tmX, s);
      case kModeObjective: return bsr_g4_launch<D, kModeObjective>(bp, tmX, s);
      case kModeGpm: return bsr_g4_launch<D, kModeGpm>(bp, tmX, s);
      default: return bsr_g4_launch<D, kModeProduct>(bp, tmX, s);
    }
  }
  if (lg2g >= 0) {   // bits 0-7: log2 group size; bit 8: 8-slot ring
    const int lg = lg2g & 0xff;
    if (lg2g & 0x100) {
      switch (mode) {
        case kModeRgs: return bsr_slab_launch<D, kModeRgs, 8>(bp, lg, s);
        case kModeObjective: return bsr_slab_launch<D, kModeObjective, 8>(bp, lg, s);
        case kModeGpm: return bsr_slab_launch<D, kModeGpm, 8>(bp, lg, s);
        default: return bsr_slab_launch<D, kModeProduct, 8>(bp, lg, s);
      }
    }
    switch (mode) {
      case kModeRgs: return bsr_slab_launch<D, kModeRgs, 4>(bp, lg, s);
      case kModeObjective: return bsr_slab_launch<D, kModeObjective, 4>(bp, lg, s);
      case kModeGpm: return bsr_slab_launch<D, kModeGpm, 4>(bp, lg, s);
      default: return bsr_slab_launch<D, kModeProduct, 4>(bp, lg, s);
    }
  }
  switch (mode) {
    case kModeRgs: return bsr_launch<D, kModeRgs>(bp, s);
    case kModeObjective: return bsr_launch<D, kModeObjective>(bp, s);
    case kModeGpm: return bsr_launch<D, kModeGpm>(bp, s);
    default: return bsr_launch<D, kModeProduct>(bp, s);
  }
}

}  // namespace

int bsr_xs_stride(int d, bool slab) {   // floats per node record of the padded X copy (d <= 10)
  const int dp = d + (d & 1);
  const int ds = (d * dp + 3) / 4 * 4;
  return (!slab || ds % 8 == 4) ? ds : ds + 4;
}

int bsr_grid(int d, int64_t n_local) {
  const int w = d <= 6 ? 4 : d <= kMaxNarrowD ? 2 : 1;   // wide: one CTA per node row
  return (int)((n_local + w - 1) / w);
}

// Pass selection for sorted rows (d <= 6) observed with probability ~p_eff.  Returns -1 for the
// per-block gather pass (bsr_kernel), else (ring << 8) | log2 G for the slab pass: G ~ 32 / p
// nodes per column group (about one 32-block chunk of observed blocks), capped by the slot size.
// Measured at n 20000 (bsr_bench, one box): d 5 p 0.9: slab-4 6.73-6.85 ms, slab-8 6.89, gather
// 7.7-8.8; d 5 p 0.5: slab-8 4.01, slab-4 4.25, gather 4.18-4.29; d 5 p 0.3: gather 2.57, slab-8
// 2.83; d 6 p 0.5: gather 6.16, slab-8 7.04; d 4 p 0.5: gather 3.78, slab-8 4.11; d 5 p 0.1:
// gather 1.23, slab-4 1.76; d 3 p 0.5: gather 1.86, slab-8 2.33 (the rows advance in lockstep
// through the ring, and two 9-warp CTAs per SM hide less latency than four 4-warp ones).  So the
// slab pass (4 slots) is the default for p >= 0.75 only; the 8-slot ring is opt-in.
int bsr_slab_lg2g(int d, double p_eff) {
  const char *force = std::getenv("NSRGS_BSR_SLAB");   // "4" / "8": force that ring (experiments)
  int ring = p_eff >= 0.75 ? 4 : 0;
  if (force && (force[0] == '4' || force[0] == '8')) ring = force[0] - '0';
  if (!ring) return -1;
  int gmax = 0;
  switch (d) {
    case 2: gmax = (ring == 4 ? BsrSlabCfg<2, 4>::GMAX : BsrSlabCfg<2, 8>::GMAX); break;
    case 3: gmax = (ring == 4 ? BsrSlabCfg<3, 4>::GMAX : BsrSlabCfg<3, 8>::GMAX); break;
    case 4: gmax = (ring == 4 ? BsrSlabCfg<4, 4>::GMAX : BsrSlabCfg<4, 8>::GMAX); break;
    case 5: gmax = (ring == 4 ? BsrSlabCfg<5, 4>::GMAX : BsrSlabCfg<5, 8>::GMAX); break;
    case 6: gmax = (ring == 4 ? BsrSlabCfg<6, 4>::GMAX : BsrSlabCfg<6, 8>::GMAX); break;
    default: return -1;
  }
  const double want = p_eff > 0.0 ? 32.0 / p_eff : 1e9;
  int lg = 3;
  while ((2 << lg) <= gmax && (double)(2 << lg) <= want) ++lg;
  return (ring == 8 ? 0x100 : 0) | lg;
}

cudaError_t bsr_dispatch(int d, int mode, const BsrParams *bp, int lg2g, const CUtensorMap *tmX, cudaStream_t s) {
  switch (d) {
#define NSRGS_BSR_CASE(DV) \
  case DV: return bsr_mode_switch<DV>(mode, *bp, lg2g, tmX, s);
    NSRGS_BSR_CASE(2)
    NSRGS_BSR_CASE(3)
    NSRGS_BSR_CASE(4)
    NSRGS_BSR_CASE(5)
    NSRGS_BSR_CASE(6)
    NSRGS_BSR_CASE(7)
    NSRGS_BSR_CASE(8)
    NSRGS_BSR_CASE(9)
    NSRGS_BSR_CASE(10)
    NSRGS_BSR_CASE(11)
    NSRGS_BSR_CASE(12)
    NSRGS_BSR_CASE(13)
    NSRGS_BSR_CASE(14)
    NSRGS_BSR_CASE(15)
    NSRGS_BSR_CASE(16)
    NSRGS_BSR_CASE(20)
    NSRGS_BSR_CASE(24)
    NSRGS_BSR_CASE(25)
    NSRGS_BSR_CASE(32)
#undef NSRGS_BSR_CASE
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_bsr_pack_x(int d, const void *X, float *Xs, int64_t n, int64_t rows_local, int64_t tpr, bool slab,
                              cudaStream_t s) {
  const int ds = bsr_xs_stride(d, slab);
  const int64_t cnt = n * ds;
  const unsigned grid = (unsigned)((cnt + 255) / 256);
  switch (d) {
#define NSRGS_PACK_CASE(DV) \
  case DV: bsr_pack_x_kernel<DV><<<grid, 256, 0, s>>>(static_cast<const float *>(X), Xs, n, rows_local, tpr, ds); break;
    NSRGS_PACK_CASE(2)
    NSRGS_PACK_CASE(3)
    NSRGS_PACK_CASE(4)
    NSRGS_PACK_CASE(5)
    NSRGS_PACK_CASE(6)
    NSRGS_PACK_CASE(7)
    NSRGS_PACK_CASE(8)
    NSRGS_PACK_CASE(9)
    NSRGS_PACK_CASE(10)
#undef NSRGS_PACK_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_bsr_count(int64_t n, int64_t node0, int64_t n_local, uint64_t seed, double p_obs, int64_t *cnt,
                             int64_t *rowptr, cudaStream_t s) {
  bsr_count_kernel<<<(unsigned)n_local, kGenThreads, 0, s>>>(n, node0, seed, p_obs, cnt);
  bsr_scan_kernel<<<1, 1024, 0, s>>>(cnt, n_local, rowptr);
  return cudaGetLastError();
}

cudaError_t launch_bsr_fill(int d, int64_t n, int64_t node0, int64_t n_local, uint64_t seed, double sigma, double p_obs,
                            const double *Z64, const int64_t *rowptr, int *col, float *vals, double *part,
                            cudaStream_t s) {
  bsr_fill_kernel<float><<<(unsigned)n_local, kGenThreads, 0, s>>>(n, d, node0, seed, sigma, p_obs, Z64, rowptr, col,
                                                                    vals, part);
  return cudaGetLastError();
}

cudaError_t launch_bsr_sumsq(const float *vals, int64_t count, double *part, int *nblocks, cudaStream_t s) {
  const int grid = 1024;
  *nblocks = grid;
  bsr_sumsq_kernel<<<grid, 256, 0, s>>>(vals, count, part);
  return cudaGetLastError();
}

}  // namespace nsrgs

namespace nsrgs {
// Caller-attached block-sparse arrays (nsrgs_attach_A_bsr): rowptr[0] = 0, rowptr non-decreasing,
// rowptr[n_local] = nnzb and every col in [0, n).  The passes address X_j directly from col[b]
// (bsr.cu gathers), so a bad index would read outside X: bit 1 = bad rowptr, bit 2 = bad col.
__global__ void bsr_validate_kernel(const int64_t *rowptr, const int *col, int64_t n_local, int64_t nnzb, int64_t n,
                                    int *bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int b = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n_local; i += stride) {
    const int64_t r = rowptr[i];
    if (i == 0 && r != 0) b |= 1;
    if (i == n_local && r != nnzb) b |= 1;
    if (i < n_local && rowptr[i + 1] < r) b |= 1;
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnzb; i += stride) {
    const int c = col[i];
    if (c < 0 || (int64_t)c >= n) b |= 2;
  }
  if (b) atomicOr(bad, b);
}

cudaError_t launch_bsr_validate(const int64_t *rowptr, const int *col, int64_t n_local, int64_t nnzb, int64_t n,
                                int *bad, cudaStream_t s) {
  bsr_validate_kernel<<<592, 256, 0, s>>>(rowptr, col, n_local, nnzb, n, bad);
  return cudaGetLastError();
}
}  // namespace nsrgs
