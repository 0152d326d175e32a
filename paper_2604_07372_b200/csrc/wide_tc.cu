// wide_tc.cu — the A.X pass + fused epilogue for wide blocks (d in [11, 32], SURVEY §8(f) row 4:
// the paper's experiments use d = 25) on the 5th-generation tensor cores:
// tcgen05.mma kind::tf32, 3xTF32, accumulators in TMEM.  Default for d > 10 (NSRGS_WIDE_MMA=2).
//
// Why tensor cores here and not for d <= 10: at d = 25 the contraction needs 12.5 flop per byte of
// A, i.e. 87 TFLOP/s of fp32 at the HBM rate — more than the CUDA cores deliver — so the pass is
// only HBM-bound on the tensor cores.  fp32 parity (1e-6 per step) is kept by
//   * 3xTF32: kind::tf32 reads the top 19 bits of an fp32 operand (truncation, pinned by
//     tools/micro/umma_tf32.cu), so the raw fp32 tile IS the hi part; lo = x - trunc(x) is exact.
//     A X = A_hi X_hi + A_lo X_hi + A_hi X_lo (+ A_lo X_lo ~ 2^-22, dropped);
//   * draining: the tensor core's fp32 accumulation does not round to nearest, so one accumulator
//     over all N columns drifts ∝ N.  The main accumulator (hi·hi + lo·hi) is double
//     buffered in TMEM and after every `drain` column tiles it is read back (tcgen05.ld) and added
//     into a CUDA-core fp32 sum (round to nearest) while the MMAs fill the other buffer.  The hi·lo
//     term is 2^-11 smaller; it has its own TMEM accumulator, read once per segment.
//
// CTA = 10 warps: 4 split warps, 4 drain/epilogue warps, 1 TMA producer, 1 MMA issuer.
//   producer  A tile (ROWS x 32 fp32, 128-byte swizzle, 3-D tensor map) + the X slab (32 x d) per
//             stage into an mbarrier ring;
//   split     A_lo of the stage straight into TMEM (thread = row: 8 conflict-free LDS.128 through
//             the swizzle, tcgen05.st) — A_lo never touches shared memory, the MMA takes it as
//             its TMEM A operand — and the X slab transposed into K-major swizzled X^T_hi / X^T_lo
//             tiles (the B operands);
//   MMA       per stage and 128-row half: 4 K-steps x {A·X_hi, A_lo·X_hi -> main; A·X_lo -> hilo},
//             tcgen05.commit releases the stage, the X^T buffer and (per drain period) the
//             accumulator buffer;
//   drain     tcgen05.ld of the main buffer -> fp32 sums in registers (thread = panel row); at
//             the end of a segment the node epilogue (epilogue.cuh), 4 nodes at a time.
// Work: persistent grid; the (panel, column tile) space is cut into equal contiguous ranges
// (stream-K).  A CTA's first segment may continue a panel (contribution: partial B rows to a
// per-CTA slot + flag) and its last may start one (head: waits for the later CTAs' slots, which
// they produced FIRST, adds them in CTA order — deterministic — and runs the epilogue).
#include <cuda.h>

#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace nsrgs {

template <int D, int MH, int EWT>
struct TcCfgE {
  static constexpr int NP = D <= 16 ? 16 : 32;         // MMA N: components padded
  static constexpr int MROWS = 128 * MH;               // MMA rows per stage (MH M = 128 instructions)
  static constexpr int NPP = MROWS / D;                // whole nodes per panel
  static constexpr int ROWS = NPP * D;
  static constexpr int CW = kWideColTile;
  static constexpr int A_BYTES = ROWS * CW * 4;
  static constexpr int X_BYTES = CW * D * 4;
  static constexpr int STAGE_BYTES = (A_BYTES + X_BYTES + 1023) / 1024 * 1024;
  static constexpr int NXB = 2;                        // X^T (hi, lo) buffers
  static constexpr int XT_BYTES = NP * 128;
  static constexpr int XBUF_BYTES = 2 * XT_BYTES;
  static constexpr int DD = D * D, E = DD, DDL = (DD + 31) / 32;
  static constexpr int NPART = 2 * DD + 2;
  static constexpr int EW = EWT;                       // nodes in the epilogue at a time (one warp each)
  static constexpr int SCR = EW * 5 * E * 4;
  static constexpr int RED = NPART * 8;
  static constexpr int BARS = 512;
  static constexpr int FIXED = 1024 + NXB * XBUF_BYTES + SCR + RED + BARS;
  static constexpr int BUDGET = 227 * 1024;
  static constexpr int STAGES_RAW = (BUDGET - FIXED) / STAGE_BYTES;
  static constexpr int STAGES_CAP = 10 / MH;           // TMEM: 32 A_lo columns per (stage, half)
  static constexpr int STAGES = STAGES_RAW > STAGES_CAP ? STAGES_CAP : STAGES_RAW;
  static constexpr int SMEM = FIXED + STAGES * STAGE_BYTES;
  static constexpr int THREADS = 320;
  // TMEM columns (512 allocated): main[h][b] | hilo[h] | alo[stage][h]
  static constexpr int TM_MAIN = 0, TM_HILO = 128, TM_ALO = 192;
  static_assert(MH * 2 * NP <= 128 && MH * NP <= 64 && TM_ALO + STAGES * MH * 32 <= 512, "TMEM map");
  // the MMA and the split warps read rows up to MROWS - 1 of a stage (rows >= ROWS are padding
  // whose products land in accumulator rows nobody reads): stay inside the stage
  static_assert(MROWS * 128 <= STAGE_BYTES, "padding rows must stay inside the stage");
};
template <int D, int MH>
struct TcCfg : TcCfgE<D, MH, (TcCfgE<D, MH, 4>::STAGES_RAW >= 4 ? 4 : 2)> {};

// ---- tcgen05 helpers; descriptor encodings pinned by tools/micro/umma_tf32.cu -----------------
// shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: D f32, A / B tf32, both K-major, M = 128
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void umma_ss(uint32_t d_tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d_tmem), "l"(da), "l"(db), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t db, uint32_t idesc, uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d_tmem), "r"(a_tmem), "l"(db), "r"(idesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ float tf32_lo(float x) {   // x - trunc_tf32(x): exact
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&w)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
               "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
               "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
               ::"r"(taddr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
               "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]),
               "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]),
               "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31])
               : "memory");
}
template <int NP>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&v)[NP]) {
  if constexpr (NP == 32) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                 "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                   "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                   "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                   "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(taddr) : "memory");
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 "
                 "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                   "=r"(v[15])
                 : "r"(taddr) : "memory");
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// the CTA's contiguous range of (panel, column tile) units, walked as segments of one panel
struct TcRange {
  int64_t u, u1;
  int TT;
  __device__ __forceinline__ bool next(int &panel, int &t0, int &t1) {
    if (u >= u1) return false;
    panel = (int)(u / TT);
    t0 = (int)(u - (int64_t)panel * TT);
    const int64_t left = u1 - u;
    t1 = left < (int64_t)(TT - t0) ? t0 + (int)left : TT;
    u += t1 - t0;
    return true;
  }
};
__device__ __forceinline__ int64_t tc_start(int64_t U, int c, int G) { return U * c / G; }

template <int D, int MODE, int MH>
__global__ void __launch_bounds__(TcCfg<D, MH>::THREADS, 1)
    wide_tc_kernel(const __grid_constant__ CUtensorMap tmA, const PanelParams p) {
  using C = TcCfg<D, MH>;
  constexpr int NP = C::NP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
  uint8_t *xbuf = smem + C::STAGES * C::STAGE_BYTES;
  float *scr = reinterpret_cast<float *>(xbuf + C::NXB * C::XBUF_BYTES);
  double *red = reinterpret_cast<double *>(reinterpret_cast<uint8_t *>(scr) + C::SCR);
  uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(red) + C::RED);
  uint64_t *empty = full + 10, *split_full = empty + 10, *xfree = split_full + 10;
  uint64_t *acc_full = xfree + 2, *acc_free = acc_full + 2, *seg_free = acc_free + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(seg_free + 1);
  int *flag = reinterpret_cast<int *>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&split_full[s], 4);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&xfree[b], 1);
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_free[b], 4);
    }
    mbar_init(seg_free, 4);
    fence_mbar_init();
  }
  // zero the ring, the X^T tiles (component rows >= d stay zero) and the partial sums once: the
  // MMA also reads the padding rows of a stage, which must hold finite numbers
  for (int i = threadIdx.x; i < (C::STAGES * C::STAGE_BYTES + C::NXB * C::XBUF_BYTES) / 16; i += C::THREADS)
    reinterpret_cast<float4 *>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = threadIdx.x; i < C::NPART; i += C::THREADS) red[i] = 0.0;
  fence_proxy_async_smem();
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const float *Xg = static_cast<const float *>(p.X);
  const int TT = p.total_tiles, tpr = (int)p.tiles_per_rank, G = (int)gridDim.x;
  const int64_t U = (int64_t)p.panels * TT;
  TcRange rng{tc_start(U, (int)blockIdx.x, G), tc_start(U, (int)blockIdx.x + 1, G), TT};
  const int DP = p.drain_tiles > 0 ? p.drain_tiles : 1;
  int panel, t0, t1;

  if (warp == 8) {   // ----------------------------------------------------------- TMA producer
    if (lane == 0) {
      prefetch_tmap(&tmA);
      const uint64_t pol_a = p.a_keep > 0.f ? policy_keep_fraction(p.a_keep) : policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      while (rng.next(panel, t0, t1)) {
        for (int t = t0; t < t1; ++t) {
          const int g0 = t / tpr;
          const int g = (g0 + p.rank) % p.world, jt = t - g0 * tpr;     // own rank slice first
          const int tt = g * tpr + jt;
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t *sb = smem + stage * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], C::A_BYTES + C::X_BYTES);
          tma_load_3d(sb, &tmA, &full[stage], jt * C::CW, g, panel * C::ROWS, pol_a);
          bulk_load(sb + C::A_BYTES, Xg + (int64_t)tt * C::CW * D, C::X_BYTES, &full[stage], pol_x);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else if (warp == 9) {   // ---------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = umma_idesc_tf32(NP);
      int stage = 0;
      uint32_t phase = 0;
      unsigned i = 0, pc = 0, sc = 0;
      while (rng.next(panel, t0, t1)) {
        if (sc > 0) mbar_wait(seg_free, (sc - 1u) & 1u);   // hilo of the previous segment has been read
        int b = 0;
        for (int t = t0; t < t1; ++t, ++i) {
          const int j = t - t0;
          const bool pfirst = j % DP == 0;
          mbar_wait(&full[stage], phase);
          mbar_wait(&split_full[stage], phase);
          if (pfirst) {
            b = (int)(pc & 1u);
            mbar_wait(&acc_free[b], ((pc >> 1) & 1u) ^ 1u);
          }
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t xh = smem_u32(xbuf + (i % C::NXB) * C::XBUF_BYTES), xl = xh + C::XT_BYTES;
#pragma unroll
          for (int h = 0; h < MH; ++h) {
            const uint32_t dmain = tmem + C::TM_MAIN + (uint32_t)(h * 2 + b) * NP;
            const uint32_t dhilo = tmem + C::TM_HILO + (uint32_t)h * NP;
            const uint32_t alo = tmem + C::TM_ALO + (uint32_t)(stage * MH + h) * 32u;
#pragma unroll
            for (int ks = 0; ks < C::CW / 8; ++ks) {
              const uint64_t da = umma_sdesc(sa + h * 16384 + ks * 32);
              const uint64_t dxh = umma_sdesc(xh + ks * 32), dxl = umma_sdesc(xl + ks * 32);
              umma_ts(dmain, alo + ks * 8, dxh, idesc, !(pfirst && ks == 0));
              umma_ss(dmain, da, dxh, idesc, 1u);
              umma_ss(dhilo, da, dxl, idesc, !(j == 0 && ks == 0));
            }
          }
          umma_commit(&empty[stage]);
          umma_commit(&xfree[i % C::NXB]);
          if (j % DP == DP - 1 || t == t1 - 1) {
            umma_commit(&acc_full[b]);
            ++pc;
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
        }
        ++sc;
      }
    }
  } else if (warp < 4) {   // ------------------------------------------------------ split warps
    const int r = warp * 32 + lane;
    int stage = 0;
    uint32_t phase = 0;
    unsigned i = 0;
    while (rng.next(panel, t0, t1)) {
      for (int t = t0; t < t1; ++t, ++i) {
        mbar_wait(&full[stage], phase);
        const uint8_t *sb = smem + stage * C::STAGE_BYTES;
        // A_lo row by row into TMEM (thread = row; the swizzle makes the 8 LDS.128 conflict-free)
#pragma unroll
        for (int h = 0; h < MH; ++h) {
          const int row = h * 128 + r;
          const uint8_t *rb = sb + row * 128;
          uint32_t w[32];
#pragma unroll
          for (int jc = 0; jc < 8; ++jc) {
            const float4 v = *reinterpret_cast<const float4 *>(rb + ((jc ^ (row & 7)) << 4));
            w[4 * jc + 0] = __float_as_uint(tf32_lo(v.x));
            w[4 * jc + 1] = __float_as_uint(tf32_lo(v.y));
            w[4 * jc + 2] = __float_as_uint(tf32_lo(v.z));
            w[4 * jc + 3] = __float_as_uint(tf32_lo(v.w));
          }
          tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + C::TM_ALO + (uint32_t)(stage * MH + h) * 32u, w);
        }
        // X slab (32 columns x d, row-major) -> K-major swizzled X^T (raw = hi) and X^T_lo
        const unsigned xb = i % C::NXB;
        mbar_wait(&xfree[xb], ((i / C::NXB) & 1u) ^ 1u);
        const float *Xs = reinterpret_cast<const float *>(sb + C::A_BYTES);
        uint8_t *XH = xbuf + xb * C::XBUF_BYTES, *XL = XH + C::XT_BYTES;
        if constexpr (D & 1) {   // lane = column k: stride-d reads are conflict-free for odd d
          for (int n = warp; n < D; n += 4) {
            const float x = Xs[lane * D + n];
            const uint32_t off = (uint32_t)n * 128u + ((uint32_t)((lane >> 2) ^ (n & 7)) << 4) + (uint32_t)(lane & 3) * 4u;
            *reinterpret_cast<float *>(XH + off) = x;
            *reinterpret_cast<float *>(XL + off) = tf32_lo(x);
          }
        } else {                 // lane = component n: contiguous reads, 4-way conflicting stores
          for (int k = warp; k < C::CW; k += 4) {
            if (lane < D) {
              const float x = Xs[k * D + lane];
              const uint32_t off = (uint32_t)lane * 128u + ((uint32_t)((k >> 2) ^ (lane & 7)) << 4) + (uint32_t)(k & 3) * 4u;
              *reinterpret_cast<float *>(XH + off) = x;
              *reinterpret_cast<float *>(XL + off) = tf32_lo(x);
            }
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&split_full[stage]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
      }
    }
  } else {   // ------------------------------------------------------ drain + epilogue warps 4..7
    const int wq = warp - 4, r = wq * 32 + lane, tid = threadIdx.x - 128;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    float *Bp = static_cast<float *>(p.Bpart);
    unsigned *flags = p.ucnt;
    unsigned pc = 0;
    float ns_region = 0.f;
    int err = 0;
    while (rng.next(panel, t0, t1)) {
      float tot[MH][NP];
#pragma unroll
      for (int h = 0; h < MH; ++h)
#pragma unroll
        for (int k = 0; k < NP; ++k) tot[h][k] = 0.f;
      const int nper = (t1 - t0 + DP - 1) / DP;
      for (int per = 0; per < nper; ++per, ++pc) {
        const int b = (int)(pc & 1u);
        mbar_wait(&acc_full[b], (pc >> 1) & 1u);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < MH; ++h) {
          uint32_t v[NP];
          tmem_ld<NP>(tmem + lane_base + C::TM_MAIN + (uint32_t)(h * 2 + b) * NP, v);
#pragma unroll
          for (int k = 0; k < NP; ++k) tot[h][k] += __uint_as_float(v[k]);
        }
        if (per == nper - 1) {
#pragma unroll
          for (int h = 0; h < MH; ++h) {
            uint32_t v[NP];
            tmem_ld<NP>(tmem + lane_base + C::TM_HILO + (uint32_t)h * NP, v);
#pragma unroll
            for (int k = 0; k < NP; ++k) tot[h][k] += __uint_as_float(v[k]);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&acc_free[b]);
          if (per == nper - 1) mbar_arrive(seg_free);
        }
      }
      const bool head = t0 == 0, tail = t1 == TT;
      if (!head) {   // contribution: partial rows -> this CTA's slot ([k][row]: coalesced), then the flag
        float *bp = Bp + (size_t)blockIdx.x * (C::MROWS * NP);
#pragma unroll
        for (int h = 0; h < MH; ++h)
#pragma unroll
          for (int k = 0; k < NP; ++k) __stcg(bp + k * C::MROWS + h * 128 + r, tot[h][k]);
        named_bar_sync(2, 128);
        if (tid == 0) {
          fence_acq_rel_gpu();
          atomicExch(flags + blockIdx.x, p.epoch);
        }
        continue;
      }
      if (!tail) {   // head of a split panel: add the later CTAs' partial rows in CTA order
        const int64_t last = (int64_t)(panel + 1) * TT - 1;
        for (int cc = (int)blockIdx.x + 1; cc < G && tc_start(U, cc, G) <= last; ++cc) {
          while (ld_acquire_gpu(flags + cc) != p.epoch) __nanosleep(64);
          const float *bp = Bp + (size_t)cc * (C::MROWS * NP);
#pragma unroll
          for (int h = 0; h < MH; ++h)
#pragma unroll
            for (int k = 0; k < NP; ++k) tot[h][k] += __ldcg(bp + k * C::MROWS + h * 128 + r);
        }
      }
      // node epilogue, EW nodes at a time (warp wq takes node q0 + wq)
      for (int q0 = 0; q0 < C::NPP; q0 += C::EW) {
#pragma unroll
        for (int h = 0; h < MH; ++h) {
          const int row = h * 128 + r;
          const int q = row / D, a = row - q * D;
          if (row < C::ROWS && q >= q0 && q < q0 + C::EW) {
            float *g = scr + (q - q0) * 5 * C::E + C::E + a * D;
#pragma unroll
            for (int k = 0; k < NP; ++k)
              if (k < D) g[k] = tot[h][k];
          }
        }
        named_bar_sync(2, 128);
        const bool active = wq < C::EW && q0 + wq < C::NPP;
        double g1s[C::DDL], g2s[C::DDL], so = 0.0, xs = 0.0;
        if (active) {
          float *sX = scr + wq * 5 * C::E, *sG = sX + C::E, *sH = sG + C::E, *sS = sH + C::E, *sM = sS + C::E;
          const int64_t node = (int64_t)panel * C::NPP + q0 + wq;
          const int nvalid = node < p.n_local ? 1 : 0;
          node_epilogue<float, D, 1, MODE>(p, Xg, p.Xout, lane, node, nvalid, sX, sG, sH, sS, sM, g1s, g2s, so, xs,
                                           ns_region, err);
          so = warp_sum(so);
          xs = warp_sum(xs);
        }
        // objective / Gram partials into the CTA's sums, one warp after the other (fixed order)
        for (int w = 0; w < C::EW; ++w) {
          if (w == wq && active) {
#pragma unroll
            for (int m = 0; m < C::DDL; ++m) {
              const int e2 = lane + 32 * m;
              if (e2 < C::DD) { red[e2] += g1s[m]; red[C::DD + e2] += g2s[m]; }
            }
            if (lane == 0) { red[2 * C::DD] += so; red[2 * C::DD + 1] += xs; }
          }
          named_bar_sync(2, 128);
        }
      }
    }
    if (err) atomicOr(p.err, err);
    if (lane == 0 && ns_region > 0.f) atomicMax(p.ns_region, __float_as_uint(ns_region));
    // per-CTA partials -> slot; the last CTA reduces all slots in order
    for (int i = tid; i < C::NPART; i += 128) __stcg(p.cta_part + (int64_t)blockIdx.x * C::NPART + i, red[i]);
    named_bar_sync(2, 128);
    if (tid == 0) {
      fence_acq_rel_gpu();
      const int is_last = (atomicAdd(p.done_cnt, 1u) == gridDim.x - 1);
      if (is_last) fence_acq_rel_gpu();
      *flag = is_last;
    }
    named_bar_sync(2, 128);
    if (*flag) {
      for (int i = wq; i < C::NPART; i += 4) {
        double v = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(p.cta_part + (int64_t)b * C::NPART + i);
        v = warp_sum(v);
        if (lane == 0) p.result[i] = v;
      }
      if (tid == 0) *p.done_cnt = 0u;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 9) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

template <int D, int MODE, int MH>
static cudaError_t tc_launch(const CUtensorMap *tm, const PanelParams &p, int grid, cudaStream_t s) {
  using C = TcCfg<D, MH>;
  auto kern = wide_tc_kernel<D, MODE, MH>;
  static bool attr[64] = {};
  {
    const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void *>(kern), C::SMEM, attr);
    if (e != cudaSuccess) return e;
  }
  kern<<<grid, C::THREADS, C::SMEM, s>>>(*tm, p);
  return cudaGetLastError();
}

template <int D, int MH>
static cudaError_t tc_mode(int mode, const CUtensorMap *tm, const PanelParams &p, int grid, cudaStream_t s) {
  if (mode == kModeRgs) return tc_launch<D, kModeRgs, MH>(tm, p, grid, s);
  if (mode == kModeObjective) return tc_launch<D, kModeObjective, MH>(tm, p, grid, s);
  if (mode == kModeGpm) return tc_launch<D, kModeGpm, MH>(tm, p, grid, s);
  return tc_launch<D, kModeProduct, MH>(tm, p, grid, s);
}

// shape->nw reports MROWS * NP floats / 1024 (the per-CTA partial slot, for the runtime's allocation)
cudaError_t wide_tc_dispatch(int d, int mode, bool shape_only, PanelShape *shape, int *slot_floats,
                             const CUtensorMap *tm, const PanelParams *p, int grid, cudaStream_t s) {
#define NSRGS_TC_CASE(DV)                                                                          \
  case DV: {                                                                                       \
    using C = TcCfg<DV, 2>;                                                                        \
    if (shape_only) {                                                                              \
      *shape = PanelShape{C::ROWS, C::NPP, C::STAGES, C::SMEM, C::NPART, C::THREADS, 4};          \
      if (slot_floats) *slot_floats = C::MROWS * C::NP;                                            \
      return cudaSuccess;                                                                          \
    }                                                                                              \
    return tc_mode<DV, 2>(mode, tm, *p, grid, s);                                                  \
  }
  switch (d) {
    NSRGS_TC_CASE(11)
    NSRGS_TC_CASE(12)
    NSRGS_TC_CASE(13)
    NSRGS_TC_CASE(14)
    NSRGS_TC_CASE(15)
    NSRGS_TC_CASE(16)
    NSRGS_TC_CASE(20)
    NSRGS_TC_CASE(24)
    NSRGS_TC_CASE(25)
    NSRGS_TC_CASE(32)
    default: return cudaErrorInvalidValue;
  }
#undef NSRGS_TC_CASE
}

}  // namespace nsrgs
