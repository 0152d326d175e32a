// wide.cu — the two fallback A.X passes for wide blocks, d in {11, ..., 16, 20, 24, 25, 32}
// (the paper's experiments use d = 25; §8(b) asks for d <= 16).
// The DEFAULT wide pass is wide_tc.cu (tcgen05, NSRGS_WIDE_MMA=2 / unset); the passes here are
// selected with NSRGS_WIDE_MMA=1 / 0 and kept as independent implementations for the variant
// parity tests (tests/test_gpu_parity.py::test_wide_pass_variants) and as A/B baselines.
//
// With d > 10 the narrow kernel's register tile (RT rows x d accumulators per lane) no longer
// fits, so a consumer warp owns ONE node (d rows of A).  4 consumer warps + 1 TMA producer warp
// per CTA, one CTA per row panel (4 nodes), the same mbarrier ring, tensor map and per-node
// epilogue (epilogue.cuh) as the narrow kernel.  Two inner products:
//
//  * MMA = true (NSRGS_WIDE_MMA=1): 3xTF32 on the tensor cores with legacy mma.sync m16n8k8 — A
//    fragments read from the stage through the 128-byte TMA swizzle (so the runtime's tensor map
//    MUST be encoded with CU_TENSOR_MAP_SWIZZLE_128B whenever a tensor-core variant runs:
//    build_tmap couples the two through ctx->wide_mma != 0), X fragments from the row-major
//    32 x d slab, hi/lo splits on the fly, and the MMA accumulator drained into a CUDA-core fp32
//    sum after every 32-column tile (the tensor core's fp32 accumulation does not round to
//    nearest; bounding each chain to one tile keeps the step error at <= 3.1e-7, below the
//    CUDA-core pass's 8.4e-7, profiles/r01c_wide_variants.txt).
//  * MMA = false (NSRGS_WIDE_MMA=0): CUDA cores, lane k owns output component k,
//    acc[r] += A[r][c] X[c][k] with A row pieces as 128-bit smem broadcasts and FFMA2 on column
//    pairs (even / odd partial sums).
//
// Measured on B200 (same box, mean pass of a 20-iteration run, profiles/r02_wide_ab.log): d = 25,
// n = 4000: 19.1 ms (mma.sync) vs 7.6 ms (tcgen05); d = 16, n = 8000: 19.2 vs 10.5 ms; the
// CUDA-core pass is another 1.07-1.9x slower than mma.sync (profiles/r01c_wide_variants.txt).
#include <cuda.h>

#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace nsrgs {

template <int D, bool MMA = false>
struct WideCfg {
  static constexpr int W = 4;                          // consumer warps = nodes per panel
  static constexpr int THREADS = 32 * (W + 1);
  static constexpr int ROWS = W * D;
  static constexpr int CW = kWideColTile;
  static constexpr int A_BYTES = ROWS * CW * 4;
  static constexpr int X_BYTES = CW * D * 4;
  // = 128 (ROWS + D): TMA-aligned; the tensor-core variant reads A through the 128-byte TMA
  // swizzle, whose pattern needs 1024-byte aligned stages
  static constexpr int STAGE_BYTES = MMA ? (A_BYTES + X_BYTES + 1023) / 1024 * 1024 : A_BYTES + X_BYTES;
  static constexpr int DD = D * D, E = DD, DDL = (DD + 31) / 32;
  static constexpr int NPART = 2 * DD + 2;
  static constexpr int SCR = W * 5 * E * 4;
  static constexpr int RED = W * NPART * 8;
  static constexpr int FIXED = 1024 + 128 + SCR + RED + 64;
  static constexpr int BUDGET = 222 * 1024;
  static constexpr int STAGES_RAW = (BUDGET - FIXED) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static_assert(STAGES >= 2, "ring");
  static constexpr int SMEM = FIXED + STAGES * STAGE_BYTES;
  // The MMA variant reads A fragment rows warp*D .. warp*D + 16*MT - 1: for d not a multiple of
  // 16 the last rows are the next node's (warp 3: bytes of the X slab).  Their products land in
  // accumulator rows a >= D, which are dropped; the reads must stay inside the stage.
  static constexpr int MT = (D + 15) / 16;
  static_assert(!MMA || ((W - 1) * D + 16 * MT) * CW * 4 <= STAGE_BYTES,
                "MMA fragment rows past the panel must stay inside the stage");
};

__device__ __forceinline__ uint64_t wpack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t wffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// ---- tensor-core path (3xTF32 on mma.sync m16n8k8): fp32 x = hi + lo with hi = tf32(x),
// lo = tf32(x - hi); A X ~ A_lo X_hi + A_hi X_lo + A_hi X_hi (the dropped A_lo X_lo is ~2^-22
// relative), accumulated in fp32.
__device__ __forceinline__ void split_tf32(float x, uint32_t &hi, uint32_t &lo) {
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hi) : "f"(x));
  const float r = x - __uint_as_float(hi);
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(lo) : "f"(r));
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
               "{%0, %1, %2, %3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// element (r, c) of a 128-byte-swizzled [rows][32] fp32 TMA tile (1024-byte aligned base)
__device__ __forceinline__ float lds_sw128(const uint8_t *base, int r, int c) {
  const uint32_t off = (uint32_t)r * 128u + ((((uint32_t)(c >> 2) ^ (uint32_t)(r & 7)) << 4) | ((uint32_t)(c & 3) << 2));
  return *reinterpret_cast<const float *>(base + off);
}

template <int D, int MODE, bool MMA>
__global__ void __launch_bounds__(WideCfg<D, MMA>::THREADS, 1)
    wide_kernel(const __grid_constant__ CUtensorMap tmA, const PanelParams p) {
  using C = WideCfg<D, MMA>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *empty = full + 8;
  float *scr = reinterpret_cast<float *>(smem + C::STAGES * C::STAGE_BYTES + 128);
  double *red = reinterpret_cast<double *>(reinterpret_cast<uint8_t *>(scr) + C::SCR);
  int *flag = reinterpret_cast<int *>(red + C::W * C::NPART);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::W);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const float *Xg = static_cast<const float *>(p.X);
  const int panel = blockIdx.x;
  const int tpr = (int)p.tiles_per_rank;

  if (warp == C::W) {   // ------------------------------------------------ TMA producer
    if (lane == 0) {
      prefetch_tmap(&tmA);
      const uint64_t pol_a = p.a_keep > 0.f ? policy_keep_fraction(p.a_keep) : policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 0; t < p.total_tiles; ++t) {
        const int g0 = t / tpr;
        const int g = (g0 + p.rank) % p.world, jt = t - g0 * tpr;     // own rank slice first
        const int tt = g * tpr + jt;
        mbar_wait(&empty[stage], phase ^ 1u);
        uint8_t *sb = smem + stage * C::STAGE_BYTES;
        mbar_arrive_expect_tx(&full[stage], C::A_BYTES + C::X_BYTES);   // STAGE_BYTES may include alignment padding
        tma_load_3d(sb, &tmA, &full[stage], jt * C::CW, g, panel * C::ROWS, pol_a);
        bulk_load(sb + C::A_BYTES, Xg + (int64_t)tt * C::CW * D, C::X_BYTES, &full[stage], pol_x);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumer warp = one node
  float *sX = scr + warp * 5 * C::E, *sG = sX + C::E, *sH = sG + C::E, *sS = sH + C::E, *sM = sS + C::E;
  if constexpr (MMA) {
    // tensor cores: B_i[a][k] = sum_c A[a][c] X[c][k] as m16 (node rows) x n8 (components) x k8
    // (columns) tiles; A fragments from the swizzled tile (conflict-free), X fragments from the
    // row-major [32][d] slab; rows / components past d are computed on padding and dropped
    constexpr int MT = (D + 15) / 16, NT = (D + 7) / 8;
    // acc: the tensor core's accumulator, restarted every tile (32 columns = 12 MMAs): its fp32
    // accumulation does not round to nearest, so a chain over all N columns drifts (error ∝ N);
    // tot: the running sum in CUDA-core fp32 (round to nearest), one FADD per entry per tile
    float acc[MT][NT][4], tot[MT][NT][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) { acc[mt][nt][e] = 0.f; tot[mt][nt][e] = 0.f; }
    const int g = lane >> 2, tq = lane & 3;
    int stage = 0;
    uint32_t phase = 0;
    for (int t = 0; t < p.total_tiles; ++t) {
      mbar_wait(&full[stage], phase);
      const uint8_t *Ab = smem + stage * C::STAGE_BYTES;
      const float *Xs = reinterpret_cast<const float *>(smem + stage * C::STAGE_BYTES + C::A_BYTES);
#pragma unroll
      for (int k0 = 0; k0 < C::CW; k0 += 8) {
        uint32_t bh[NT][2], bl[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int n = nt * 8 + g;
          const float x0 = n < D ? Xs[(k0 + tq) * D + n] : 0.f;
          const float x1 = n < D ? Xs[(k0 + tq + 4) * D + n] : 0.f;
          split_tf32(x0, bh[nt][0], bl[nt][0]);
          split_tf32(x1, bh[nt][1], bl[nt][1]);
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const int r0 = warp * D + mt * 16 + g;
          uint32_t ah[4], al[4];
          split_tf32(lds_sw128(Ab, r0, k0 + tq), ah[0], al[0]);
          split_tf32(lds_sw128(Ab, r0 + 8, k0 + tq), ah[1], al[1]);
          split_tf32(lds_sw128(Ab, r0, k0 + tq + 4), ah[2], al[2]);
          split_tf32(lds_sw128(Ab, r0 + 8, k0 + tq + 4), ah[3], al[3]);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            mma_tf32(acc[mt][nt], al, bh[nt][0], bh[nt][1]);
            mma_tf32(acc[mt][nt], ah, bl[nt][0], bl[nt][1]);
            mma_tf32(acc[mt][nt], ah, bh[nt][0], bh[nt][1]);
          }
        }
      }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) { tot[mt][nt][e] += acc[mt][nt][e]; acc[mt][nt][e] = 0.f; }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
    }
    // C fragment (row g / g + 8, columns 2 tq, 2 tq + 1) -> B_i entries (a, k) inside d x d
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int a = mt * 16 + g + (e >> 1) * 8, k = nt * 8 + 2 * tq + (e & 1);
          if (a < D && k < D) sG[a * D + k] = tot[mt][nt][e];
        }
    __syncwarp();
  } else {
  const int kk = lane < D ? lane : D - 1;
  uint64_t acc2[D];   // (even-column, odd-column) partial sums of row r, component `lane`
#pragma unroll
  for (int r = 0; r < D; ++r) acc2[r] = 0ull;
  int stage = 0;
  uint32_t phase = 0;
  for (int t = 0; t < p.total_tiles; ++t) {
    mbar_wait(&full[stage], phase);
    const float *As = reinterpret_cast<const float *>(smem + stage * C::STAGE_BYTES) + warp * D * C::CW;
    const float *Xs = reinterpret_cast<const float *>(smem + stage * C::STAGE_BYTES + C::A_BYTES) + kk;
#pragma unroll
    for (int c4 = 0; c4 < C::CW / 4; ++c4) {
      const uint64_t xa = wpack(Xs[(4 * c4 + 0) * D], Xs[(4 * c4 + 1) * D]);
      const uint64_t xb = wpack(Xs[(4 * c4 + 2) * D], Xs[(4 * c4 + 3) * D]);
#pragma unroll
      for (int r = 0; r < D; ++r) {
        const ulonglong2 a = *reinterpret_cast<const ulonglong2 *>(As + r * C::CW + 4 * c4);   // broadcast
        acc2[r] = wffma2(a.x, xa, acc2[r]);
        acc2[r] = wffma2(a.y, xb, acc2[r]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
  }

#pragma unroll
  for (int r = 0; r < D; ++r) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(acc2[r]));
    if (lane < D) sG[r * D + lane] = lo + hi;   // entry (a = r, b = lane) of B_i
  }
  __syncwarp();
  }
  const int64_t node = (int64_t)panel * C::W + warp;
  const int nvalid = node < p.n_local ? 1 : 0;
  double g1s[C::DDL], g2s[C::DDL], so = 0.0, xs = 0.0;
  float ns_region = 0.f;
  int err = 0;
  node_epilogue<float, D, 1, MODE>(p, Xg, p.Xout, lane, node, nvalid, sX, sG, sH, sS, sM, g1s, g2s, so, xs, ns_region, err);
  if (err) atomicOr(p.err, err);
  if (lane == 0 && ns_region > 0.f) atomicMax(p.ns_region, __float_as_uint(ns_region));

  // per-CTA partials (fixed warp order) -> slot, last CTA reduces all slots in order
  so = warp_sum(so);
  xs = warp_sum(xs);
  double *rw = red + warp * C::NPART;
#pragma unroll
  for (int m = 0; m < C::DDL; ++m) {
    const int e2 = lane + 32 * m;
    if (e2 < C::DD) { rw[e2] = g1s[m]; rw[C::DD + e2] = g2s[m]; }
  }
  if (lane == 0) { rw[2 * C::DD] = so; rw[2 * C::DD + 1] = xs; }
  named_bar_sync(1, C::W * 32);
  for (int i = threadIdx.x; i < C::NPART; i += C::W * 32) {
    double v = 0.0;
    for (int w = 0; w < C::W; ++w) v += red[w * C::NPART + i];
    __stcg(p.cta_part + (int64_t)blockIdx.x * C::NPART + i, v);
  }
  named_bar_sync(1, C::W * 32);
  if (threadIdx.x == 0) {   // one fence per CTA (bar.sync + cumulative fence), see panel.cu
    fence_acq_rel_gpu();
    const int is_last = (atomicAdd(p.done_cnt, 1u) == gridDim.x - 1);
    if (is_last) fence_acq_rel_gpu();
    *flag = is_last;
  }
  named_bar_sync(1, C::W * 32);
  if (*flag) {
    for (int i = warp; i < C::NPART; i += C::W) {
      double v = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(p.cta_part + (int64_t)b * C::NPART + i);
      v = warp_sum(v);
      if (lane == 0) p.result[i] = v;
    }
    if (threadIdx.x == 0) *p.done_cnt = 0u;
  }
}

template <int D, int MODE, bool MMA>
static cudaError_t wide_launch(const CUtensorMap *tm, const PanelParams &p, int grid, cudaStream_t s) {
  using C = WideCfg<D, MMA>;
  auto kern = wide_kernel<D, MODE, MMA>;
  static bool attr[64] = {};
  {
    const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void *>(kern), C::SMEM, attr);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid, C::THREADS, C::SMEM, s>>>(*tm, p);
  return cudaGetLastError();
}

template <int D, bool MMA>
static cudaError_t wide_mode(int mode, const CUtensorMap *tm, const PanelParams &p, int grid, cudaStream_t s) {
  if (mode == kModeRgs) return wide_launch<D, kModeRgs, MMA>(tm, p, grid, s);
  if (mode == kModeObjective) return wide_launch<D, kModeObjective, MMA>(tm, p, grid, s);
  if (mode == kModeGpm) return wide_launch<D, kModeGpm, MMA>(tm, p, grid, s);
  return wide_launch<D, kModeProduct, MMA>(tm, p, grid, s);
}

bool wide_supported(int d) { return (d >= 11 && d <= 16) || d == 20 || d == 24 || d == 25 || d == 32; }

// mma: the 3xTF32 tensor-core variant (the caller's tensor map must then use the 128-byte swizzle)
cudaError_t wide_dispatch(int d, int mode, bool shape_only, PanelShape *shape, const CUtensorMap *tm,
                          const PanelParams *p, int grid, cudaStream_t s, bool mma) {
#define NSRGS_WIDE_CASE(DV)                                                                        \
  case DV: {                                                                                       \
    if (shape_only) {                                                                              \
      if (mma) {                                                                                   \
        using C = WideCfg<DV, true>;                                                               \
        *shape = PanelShape{C::ROWS, C::W, C::STAGES, C::SMEM, C::NPART, C::THREADS, C::W};        \
      } else {                                                                                     \
        using C = WideCfg<DV, false>;                                                              \
        *shape = PanelShape{C::ROWS, C::W, C::STAGES, C::SMEM, C::NPART, C::THREADS, C::W};        \
      }                                                                                            \
      return cudaSuccess;                                                                          \
    }                                                                                              \
    return mma ? wide_mode<DV, true>(mode, tm, *p, grid, s) : wide_mode<DV, false>(mode, tm, *p, grid, s); \
  }
  switch (d) {
    NSRGS_WIDE_CASE(11)
    NSRGS_WIDE_CASE(12)
    NSRGS_WIDE_CASE(13)
    NSRGS_WIDE_CASE(14)
    NSRGS_WIDE_CASE(15)
    NSRGS_WIDE_CASE(16)
    NSRGS_WIDE_CASE(20)
    NSRGS_WIDE_CASE(24)
    NSRGS_WIDE_CASE(25)
    NSRGS_WIDE_CASE(32)
    default: return cudaErrorInvalidValue;
  }
#undef NSRGS_WIDE_CASE
}

}  // namespace nsrgs
