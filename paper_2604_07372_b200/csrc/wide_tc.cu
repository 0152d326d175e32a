// wide_tc.cu — the A.X pass + fused epilogue on the 5th-generation tensor cores (tcgen05.mma
// kind::tf32, 3xTF32, operands and accumulators in TMEM) for wide blocks, d in [11, 32] (SURVEY
// §8(f) row 4: the paper's experiments use d = 25; default, NSRGS_WIDE_MMA=2), and
// for d = 10 with X in the narrow tile layout (template flag NL: config c4 on large shards).
//
// Why tensor cores here and not for small d: at d = 25 the contraction needs 12.5 flop per byte of
// A, i.e. 87 TFLOP/s of fp32 at the HBM rate — more than the CUDA cores deliver — so the pass is
// only HBM-bound on the tensor cores (d = 10 is FMA co-limited under the power cap).  fp32 parity
// (1e-6 per step) is kept by
//   * 3xTF32: kind::tf32 reads the top 19 bits of an fp32 operand (truncation, pinned by
//     tools/micro/umma_tf32.cu), so the raw fp32 value IS the hi part; lo = x - trunc(x) is exact.
//     A X = A_lo X_hi + A X_lo + A X_hi (+ A_lo X_lo ~ 2^-20, dropped);
//   * draining: the tensor core's fp32 accumulation does not round to nearest, so one accumulator
//     over all N columns drifts ∝ N.  The accumulator of each 128-row half is double
//     buffered in TMEM and after every `drain` column tiles it is read back (tcgen05.ld) and added
//     into a CUDA-core fp32 sum (round to nearest) while the MMAs fill the other buffer.
//
// CTA = 16 warps in 4 warpgroups, registers re-dealt with setmaxnreg (104 / 104 / 232 / 72): two
// split warpgroups (alternate tiles), one drain/epilogue warpgroup, and a control group (TMA
// producer warp, MMA issuer warp, 2 idle warps).
//   producer  A tile (ROWS x 32 fp32, 128-byte swizzle, 3-D tensor map) + the X slab (32 x d) per
//             stage into an mbarrier ring (a pure landing buffer: free again once it is read);
//   split     thread = row: 8 conflict-free LDS.128 through the swizzle, then the row goes into
//             TMEM twice with tcgen05.st — raw (= A_hi, the tensor core truncates) and A_lo — as
//             the MMAs' TMEM A operands (3 operand buffers); the X slab is transposed into K-major
//             swizzled X^T_hi / X^T_lo smem tiles (the B operands).  No MMA reads A from shared
//             memory: measured (tools/micro/umma_rate.cu) an M 128 x N 32 x K 8 kind::tf32 MMA
//             takes 42 cycles with A in smem (the 4 KB A read is exposed) and 17 from TMEM;
//   MMA       per operand buffer and 128-row half: {A_lo·X_hi, A·X_lo, A·X_hi} x 4 K-steps into the
//             half's accumulator (small terms first); tcgen05.commit releases the operand buffer
//             and (per drain period) the accumulator buffer.  Issued under elect.sync so the
//             UTCHMMAs are straight-line; per-tile descriptors are one base descriptor + constants;
//   drain     tcgen05.ld of the accumulator -> fp32 sums in registers (thread = panel row); at
//             the end of a whole panel the node epilogue (epilogue.cuh), 4 nodes at a time.
// Work: persistent grid (one CTA per SM, cooperative launch); the (panel, column tile) space is cut
// into equal contiguous ranges (stream-K).  A partial segment of a panel — a CTA's first segment
// may continue a panel, its last may start one — goes to a per-CTA slot + epoch flag; after its
// range every CTA sharing a split panel takes every np-th node of it, sums that node's partial
// rows over all sharers' slots in CTA order (deterministic) and runs its epilogue — so at small n
// (Table 1: 50 panels for 148 SMs) the epilogues are spread over all CTAs.  Objective / Gram
// partials: per-CTA slots, reduced in two fixed-order levels by the last CTA of each group.
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
  static constexpr int NXB = 3;                        // operand buffers: X^T (hi, lo) in smem, A (hi, lo) in TMEM
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
  static constexpr int STAGES = STAGES_RAW > 6 ? 6 : STAGES_RAW;
  static constexpr int SMEM = FIXED + STAGES * STAGE_BYTES;
  // 16 warps: split WG 0 (warps 0-3), split WG 1 (4-7), drain/epilogue WG (8-11), producer (12),
  // MMA issuer (13), 2 idle; launched at 128 registers, re-dealt with setmaxnreg
  static constexpr int THREADS = 512;
  static constexpr int REG_SPLIT = 104, REG_DRAIN = 232, REG_CTRL = 72;
  static_assert(2 * REG_SPLIT + REG_DRAIN + REG_CTRL <= 512, "register file: 4 warpgroups x 128 threads");
  // TMEM columns (512 allocated): accumulators acc[h][b] | A operand buffers [ob][h] = (A_hi 32 | A_lo 32)
  static constexpr int TM_MAIN = 0, TM_A = 128;
  static_assert(MH * 2 * NP <= 128 && TM_A + NXB * MH * 64 <= 512, "TMEM map");
  // the MMA and the split warps read rows up to MROWS - 1 of a stage (rows >= ROWS are padding
  // whose products land in accumulator rows nobody reads): stay inside the stage
  static_assert(MROWS * 128 <= STAGE_BYTES, "padding rows must stay inside the stage");
};
template <int D, int MH>
struct TcCfg : TcCfgE<D, MH, (TcCfgE<D, MH, 4>::STAGES_RAW >= 4 ? 4 : 2)> {
  static_assert(TcCfgE<D, MH, (TcCfgE<D, MH, 4>::STAGES_RAW >= 4 ? 4 : 2)>::STAGES >= 3, "ring");
};

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
template <int R> __device__ __forceinline__ void reg_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(R)); }
template <int R> __device__ __forceinline__ void reg_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(R)); }
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&w)[16]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
               "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               ::"r"(taddr), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
               "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15])
               : "memory");
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

// try_wait without the long suspend hint of common.cuh's mbar_wait: the handshakes of this
// pipeline (split -> MMA -> drain) are latency-critical
__device__ __forceinline__ void mbar_wait_spin(uint64_t *bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITS_%=;\n\t}" ::"r"(addr), "r"(parity)
      : "memory");
}
template <bool SPIN = true>
__device__ __forceinline__ void mbar_wait_t(uint64_t *bar, uint32_t parity, bool timed, long long &acc) {
  const long long t = timed ? clock64() : 0;
  if constexpr (SPIN) mbar_wait_spin(bar, parity);
  else mbar_wait(bar, parity);   // suspended wait (common.cuh)
  if (timed) acc += clock64() - t;
}
constexpr int kTcGroup = 12;   // CTAs per first-level group of the final partial-sum reduction

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

// NL: X in the narrow tile layout of d <= 10 (common.cuh tile_index: 128-column tiles of component
// pair blocks) — the same kernel then serves d = 10 (c4), whose CUDA-core pass is FMA co-limited
template <int D, int MODE, int MH, bool NL>
__global__ void __launch_bounds__(TcCfg<D, MH>::THREADS, 1)
    wide_tc_kernel(const __grid_constant__ CUtensorMap tmA, const PanelParams p) {
  using C = TcCfg<D, MH>;
  static_assert(!NL || (D % 2 == 0 && D <= kMaxNarrowD), "narrow layout: even d <= 10 (pair blocks only)");
  constexpr int NP = C::NP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
  uint8_t *xbuf = smem + C::STAGES * C::STAGE_BYTES;
  float *scr = reinterpret_cast<float *>(xbuf + C::NXB * C::XBUF_BYTES);
  double *red = reinterpret_cast<double *>(reinterpret_cast<uint8_t *>(scr) + C::SCR);
  uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(red) + C::RED);
  uint64_t *empty = full + 10, *split_full = empty + 10, *bfree = split_full + 4;
  uint64_t *acc_full = bfree + 4, *acc_free = acc_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_free + 2);
  int *flag = reinterpret_cast<int *>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    for (int b = 0; b < C::NXB; ++b) {
      mbar_init(&split_full[b], 4);
      mbar_init(&bfree[b], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_free[b], 4);
    }
    fence_mbar_init();
  }
  // zero the ring, the X^T tiles (component rows >= d stay zero) and the partial sums once: the
  // MMA also reads the padding rows of a stage, which must hold finite numbers
  for (int i = threadIdx.x; i < (C::STAGES * C::STAGE_BYTES + C::NXB * C::XBUF_BYTES) / 16; i += C::THREADS)
    reinterpret_cast<float4 *>(smem)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = threadIdx.x; i < C::NPART; i += C::THREADS) red[i] = 0.0;
  fence_proxy_async_smem();
  if (warp == 13) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const float *Xg = static_cast<const float *>(p.X);
  // 32-column tiles: the narrow layout's plan counts 128-column tiles
  const int TT = NL ? 4 * p.total_tiles : p.total_tiles, tpr = NL ? 4 * (int)p.tiles_per_rank : (int)p.tiles_per_rank;
  const int G = (int)gridDim.x;
  const int64_t U = (int64_t)p.panels * TT;
  TcRange rng{tc_start(U, (int)blockIdx.x, G), tc_start(U, (int)blockIdx.x + 1, G), TT};
  const int DP = p.drain_tiles > 0 ? p.drain_tiles : 1;
  const bool timed = p.ts != nullptr;   // debug: per-role wait / busy cycles into ts[cta][slot]
  int panel, t0, t1;

  if (warp >= 12) {   // ---------------------------------- control warpgroup: producer, MMA issuer, 2 idle
    reg_dec<C::REG_CTRL>();
  if (warp == 12) {   // ---------------------------------------------------------- TMA producer
    if (elect_one()) {
      prefetch_tmap(&tmA);
      const uint64_t pol_a = p.a_keep > 0.f ? policy_keep_fraction(p.a_keep) : policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      long long tw = 0;
      const long long tb = timed ? clock64() : 0;
      while (rng.next(panel, t0, t1)) {
        for (int t = t0; t < t1; ++t) {
          const int g0 = t / tpr;
          const int g = (g0 + p.rank) % p.world, jt = t - g0 * tpr;     // own rank slice first
          const int tt = g * tpr + jt;
          mbar_wait_t<false>(&empty[stage], phase ^ 1u, timed, tw);
          uint8_t *sb = smem + stage * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], C::A_BYTES + C::X_BYTES);
          tma_load_3d(sb, &tmA, &full[stage], jt * C::CW, g, panel * C::ROWS, pol_a);
          if constexpr (NL) {   // 32 columns of every component pair block: d/2 runs of 64 floats
            const float *xt = Xg + (int64_t)(tt >> 2) * (D * kColTile) + (tt & 3) * 64;
#pragma unroll
            for (int kp = 0; kp < D / 2; ++kp)
              bulk_load(sb + C::A_BYTES + kp * 256, xt + kp * 2 * kColTile, 256, &full[stage], pol_x);
          } else {
            bulk_load(sb + C::A_BYTES, Xg + (int64_t)tt * C::CW * D, C::X_BYTES, &full[stage], pol_x);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
        }
      }
      if (timed) {
        p.ts[(size_t)blockIdx.x * kTsSlots + 0] = (unsigned long long)(clock64() - tb);
        p.ts[(size_t)blockIdx.x * kTsSlots + 1] = (unsigned long long)tw;
      }
    }
  } else if (warp == 13) {   // --------------------------------------------------- MMA issuer
    if (elect_one()) {
      constexpr uint32_t idesc = umma_idesc_tf32(NP);
      // descriptor of X^T buffer 0, K-step 0; every other one is this + a constant: the start
      // address field counts 16-byte units and cannot carry out of its 14 bits (smem < 256 KB),
      // so the per-tile uniform-datapath work is a handful of adds, not 16 descriptor builds
      const uint64_t dx0 = umma_sdesc(smem_u32(xbuf));
      unsigned pc = 0, ob = 0, ophase = 0;
      long long tw_in = 0, tw_acc = 0;
      const long long tb = timed ? clock64() : 0;
      while (rng.next(panel, t0, t1)) {
        int b = 0, jp = 0;   // jp: tile index within the drain period
        for (int t = t0; t < t1; ++t) {
          const bool pfirst = jp == 0;
          mbar_wait_t(&split_full[ob], ophase, timed, tw_in);
          if (pfirst) {
            b = (int)(pc & 1u);
            mbar_wait_t(&acc_free[b], ((pc >> 1) & 1u) ^ 1u, timed, tw_acc);
          }
          tc_fence_after();
          const uint64_t dxh = dx0 + (uint64_t)(ob * (C::XBUF_BYTES >> 4)), dxl = dxh + (C::XT_BYTES >> 4);
          const uint32_t abase = tmem + C::TM_A + ob * (MH * 64u);
#pragma unroll
          for (int h = 0; h < MH; ++h) {
            const uint32_t dmain = tmem + C::TM_MAIN + (uint32_t)(h * 2 + b) * NP;
            const uint32_t ahi = abase + (uint32_t)h * 64u, alo = ahi + 32u;
            // all three A operands come from TMEM.  Order: the two small terms (2^-11 of the
            // product) first, A.X_hi last — every accumulation truncates toward zero at the
            // accumulator's magnitude, so only the last 4 of the 12 MMAs of a tile lose an ulp of
            // the full partial sum (measured bias of <X, A X>, n 1100, d 16: 5.1e-7 interleaved)
#pragma unroll
            for (int ks = 0; ks < C::CW / 8; ++ks) umma_ts(dmain, alo + ks * 8, dxh + 2 * ks, idesc, !(pfirst && ks == 0));
#pragma unroll
            for (int ks = 0; ks < C::CW / 8; ++ks) umma_ts(dmain, ahi + ks * 8, dxl + 2 * ks, idesc, 1u);
#pragma unroll
            for (int ks = 0; ks < C::CW / 8; ++ks) umma_ts(dmain, ahi + ks * 8, dxh + 2 * ks, idesc, 1u);
          }
          umma_commit(&bfree[ob]);
          if (++ob == C::NXB) { ob = 0; ophase ^= 1u; }
          if (++jp == DP || t == t1 - 1) {
            umma_commit(&acc_full[b]);
            ++pc;
            jp = 0;
          }
        }
      }
      if (timed) {
        p.ts[(size_t)blockIdx.x * kTsSlots + 5] = (unsigned long long)tw_in;
        p.ts[(size_t)blockIdx.x * kTsSlots + 6] = (unsigned long long)tw_acc;
        p.ts[(size_t)blockIdx.x * kTsSlots + 7] = (unsigned long long)(clock64() - tb);
      }
    }
  }
  } else if (warp < 8) {   // ------------------- split warps: warpgroup g takes the tiles i = g (mod 2)
    reg_dec<C::REG_SPLIT>();
    const int wg = warp >> 2, wq = warp & 3, r = wq * 32 + lane;
    unsigned i = 0;
    long long tw_full = 0, tw_x = 0;
    const long long tb = timed ? clock64() : 0;
    while (rng.next(panel, t0, t1)) {
      for (int t = t0; t < t1; ++t, ++i) {
        if ((int)(i & 1u) != wg) continue;
        const unsigned xb = i % C::NXB;
        const int stage = (int)(i % C::STAGES);
        const uint32_t phase = (i / C::STAGES) & 1u;
        mbar_wait_t<false>(&full[stage], phase, timed, tw_full);   // TMA arrival: suspended wait (A/B neutral vs spinning)
        const uint8_t *sb = smem + stage * C::STAGE_BYTES;
        // the X slab (32 columns x d, row-major) of the stage into registers first
        const float *Xs = reinterpret_cast<const float *>(sb + C::A_BYTES);
        constexpr int NI = (D & 1) ? (D + 3) / 4 : C::CW / 4;
        float xv[NI];
#pragma unroll
        for (int it = 0; it < NI; ++it) {
          if constexpr (D & 1) {   // lane = column k: stride-d reads are conflict-free for odd d
            const int n = wq + 4 * it;
            xv[it] = n < D ? Xs[lane * D + n] : 0.f;
          } else if constexpr (NL) {   // lane = component n of pair block n / 2: (column, pair) interleaved
            xv[it] = lane < D ? Xs[(lane >> 1) * 64 + 2 * (wq + 4 * it) + (lane & 1)] : 0.f;
          } else {                 // lane = component n: contiguous reads
            xv[it] = lane < D ? Xs[(wq + 4 * it) * D + lane] : 0.f;
          }
        }
        mbar_wait_t(&bfree[xb], ((i / C::NXB) & 1u) ^ 1u, timed, tw_x);   // MMAs of tile i - NXB are done
        tc_fence_after();
        // A (raw = hi) and A_lo row by row into TMEM (thread = row; the swizzle makes the 8
        // LDS.128 conflict-free): the MMA reads both as TMEM A operands, never from smem
#pragma unroll
        for (int h = 0; h < MH; ++h) {
          const int row = h * 128 + r;
          const uint8_t *rb = sb + row * 128;
          const uint32_t ta = tmem + ((uint32_t)(wq * 32) << 16) + C::TM_A + (uint32_t)(xb * MH + h) * 64u;
#pragma unroll
          for (int c16 = 0; c16 < 2; ++c16) {   // 16 columns at a time: 32 live data registers
            uint32_t wh[16], wl[16];
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
              const int jc = c16 * 4 + jj;
              const float4 v = *reinterpret_cast<const float4 *>(rb + ((jc ^ (row & 7)) << 4));
              wh[4 * jj + 0] = __float_as_uint(v.x); wl[4 * jj + 0] = __float_as_uint(tf32_lo(v.x));
              wh[4 * jj + 1] = __float_as_uint(v.y); wl[4 * jj + 1] = __float_as_uint(tf32_lo(v.y));
              wh[4 * jj + 2] = __float_as_uint(v.z); wl[4 * jj + 2] = __float_as_uint(tf32_lo(v.z));
              wh[4 * jj + 3] = __float_as_uint(v.w); wl[4 * jj + 3] = __float_as_uint(tf32_lo(v.w));
            }
            tmem_st16(ta + 16u * c16, wh);
            tmem_st16(ta + 32u + 16u * c16, wl);
          }
        }
        // every read of the stage has completed (its values fed the stores above): the stage is only
        // a TMA landing buffer, so it goes back to the producer now, not after the fences below
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        // X^T (raw = hi) and X^T_lo as K-major swizzled tiles (4-way conflicting stores for even d)
        uint8_t *XH = xbuf + xb * C::XBUF_BYTES, *XL = XH + C::XT_BYTES;
#pragma unroll
        for (int it = 0; it < NI; ++it) {
          if constexpr (D & 1) {
            const int n = wq + 4 * it;
            if (n < D) {
              const uint32_t off = (uint32_t)n * 128u + ((uint32_t)((lane >> 2) ^ (n & 7)) << 4) + (uint32_t)(lane & 3) * 4u;
              *reinterpret_cast<float *>(XH + off) = xv[it];
              *reinterpret_cast<float *>(XL + off) = tf32_lo(xv[it]);
            }
          } else {
            const int k = wq + 4 * it;
            if (lane < D) {
              const uint32_t off = (uint32_t)lane * 128u + ((uint32_t)((k >> 2) ^ (lane & 7)) << 4) + (uint32_t)(k & 3) * 4u;
              *reinterpret_cast<float *>(XH + off) = xv[it];
              *reinterpret_cast<float *>(XL + off) = tf32_lo(xv[it]);
            }
          }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_proxy_async_smem();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&split_full[xb]);
      }
    }
    if (timed && threadIdx.x == 0) {
      p.ts[(size_t)blockIdx.x * kTsSlots + 2] = (unsigned long long)tw_full;
      p.ts[(size_t)blockIdx.x * kTsSlots + 3] = (unsigned long long)tw_x;
      p.ts[(size_t)blockIdx.x * kTsSlots + 4] = (unsigned long long)(clock64() - tb);
    }
  } else {   // ----------------------------------------------------- drain + epilogue warps 8..11
    reg_inc<C::REG_DRAIN>();
    const int wq = warp - 8, r = wq * 32 + lane, tid = threadIdx.x - 256;
    const uint32_t lane_base = (uint32_t)(wq * 32) << 16;
    float *Bp = static_cast<float *>(p.Bpart);
    unsigned *flags = p.ucnt;
    constexpr int SLOT = C::MROWS * NP;
    unsigned pc = 0;
    float ns_region = 0.f;
    int err = 0;
    int nsplit = 0, sp_panel[2] = {0, 0}, segidx = 0;
    long long t_wait = 0, t_epi = 0;
    const long long t_begin = timed ? clock64() : 0;

    // one epilogue round: warp wq runs node `node_q` of `panel` (B_i already in its sG), then the
    // objective / Gram partials go into the CTA's sums one warp after the other (fixed order)
    auto epilogue_round = [&](int pnl, int node_q) {
      const bool active = wq < C::EW && node_q >= 0 && node_q < C::NPP;
      double g1s[C::DDL], g2s[C::DDL], so = 0.0, xs = 0.0;
      if (active) {
        float *sX = scr + wq * 5 * C::E, *sG = sX + C::E, *sH = sG + C::E, *sS = sH + C::E, *sM = sS + C::E;
        const int64_t node = (int64_t)pnl * C::NPP + node_q;
        const int nvalid = node < p.n_local ? 1 : 0;
        node_epilogue<float, D, 1, MODE>(p, Xg, p.Xout, lane, node, nvalid, sX, sG, sH, sS, sM, g1s, g2s, so, xs,
                                         ns_region, err);
        so = warp_sum(so);
        xs = warp_sum(xs);
      }
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
    };

    while (rng.next(panel, t0, t1)) {
      float tot[MH][NP];
#pragma unroll
      for (int h = 0; h < MH; ++h)
#pragma unroll
        for (int k = 0; k < NP; ++k) tot[h][k] = 0.f;
      const int nper = (t1 - t0 + DP - 1) / DP;
      for (int per = 0; per < nper; ++per, ++pc) {
        const int b = (int)(pc & 1u);
        mbar_wait_t<false>(&acc_full[b], (pc >> 1) & 1u, timed, t_wait);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < MH; ++h) {
          uint32_t v[NP];
          tmem_ld<NP>(tmem + lane_base + C::TM_MAIN + (uint32_t)(h * 2 + b) * NP, v);
#pragma unroll
          for (int k = 0; k < NP; ++k) tot[h][k] += __uint_as_float(v[k]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_free[b]);
      }
      const long long te0 = timed ? clock64() : 0;
      if (t0 == 0 && t1 == TT) {   // whole panel: epilogue straight from the registers, EW nodes at a time
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
          epilogue_round(panel, q0 + wq);
        }
      } else {   // part of a split panel: partial rows -> slot ([k][row]: coalesced), flag; epilogue deferred
        const int si = 2 * (int)blockIdx.x + (segidx == 0 ? 0 : 1);
        float *bp = Bp + (size_t)si * SLOT;
#pragma unroll
        for (int h = 0; h < MH; ++h)
#pragma unroll
          for (int k = 0; k < NP; ++k) __stcg(bp + k * C::MROWS + h * 128 + r, tot[h][k]);
        named_bar_sync(2, 128);
        if (tid == 0) {
          fence_acq_rel_gpu();
          atomicExch(flags + si, p.epoch);
        }
        sp_panel[nsplit++] = panel;
      }
      if (timed) t_epi += clock64() - te0;
      ++segidx;
    }
    const long long t_stream = timed ? clock64() : 0;
    // split panels: the CTAs sharing a panel deal its nodes round-robin; each sums the partial rows
    // of its nodes over all sharers' slots in CTA order (deterministic) and runs their epilogues
    for (int sidx = 0; sidx < nsplit; ++sidx) {
      const int pnl = sp_panel[sidx];
      const int64_t ub = (int64_t)pnl * TT, ue = ub + TT - 1;
      int cf = (int)blockIdx.x, cl = (int)blockIdx.x;
      while (cf > 0 && tc_start(U, cf, G) > ub) --cf;
      while (cl + 1 < G && tc_start(U, cl + 1, G) <= ue) ++cl;
      const int np = cl - cf + 1, pi = (int)blockIdx.x - cf;
      for (int cc = cf; cc <= cl; ++cc) {
        const unsigned *f = flags + 2 * cc + (tc_start(U, cc, G) >= ub ? 0 : 1);
        while (ld_acquire_gpu(f) != p.epoch) __nanosleep(40);
      }
      for (int q0 = pi; q0 < C::NPP; q0 += np * C::EW) {
        constexpr int GPT = (C::EW * C::DD + 127) / 128;   // gathered entries per thread
        float v[GPT];
        int off[GPT];
#pragma unroll
        for (int u = 0; u < GPT; ++u) {
          const int idx = tid + 128 * u;
          const int w = idx / C::DD, e = idx - w * C::DD;
          const int k = e / D, a = e - k * D;
          const int q = q0 + w * np;
          v[u] = 0.f;
          off[u] = (idx < C::EW * C::DD && q < C::NPP) ? k * C::MROWS + q * D + a : -1;
        }
        for (int cc = cf; cc <= cl; ++cc) {   // sharers in CTA order: the fixed summation order
          const float *bp = Bp + (size_t)(2 * cc + (tc_start(U, cc, G) >= ub ? 0 : 1)) * SLOT;
#pragma unroll
          for (int u = 0; u < GPT; ++u)
            if (off[u] >= 0) v[u] += __ldcg(bp + off[u]);
        }
#pragma unroll
        for (int u = 0; u < GPT; ++u) {
          const int idx = tid + 128 * u;
          const int w = idx / C::DD, e = idx - w * C::DD;
          const int k = e / D, a = e - k * D;
          if (off[u] >= 0) scr[w * 5 * C::E + C::E + a * D + k] = v[u];
        }
        named_bar_sync(2, 128);
        epilogue_round(pnl, q0 + wq * np);
      }
    }
    const long long t_shared = timed ? clock64() : 0;
    if (err) atomicOr(p.err, err);
    if (lane == 0 && ns_region > 0.f) atomicMax(p.ns_region, __float_as_uint(ns_region));
    // per-CTA partials -> slot; two-level fixed-order reduction: the last CTA of each group of
    // kTcGroup sums its group's slots, the last group to finish sums the group sums
    double *grp = p.cta_part + (int64_t)G * C::NPART;
    const int gi = (int)blockIdx.x / kTcGroup, ngrp = (G + kTcGroup - 1) / kTcGroup;
    const int gfirst = gi * kTcGroup, gsize = min(kTcGroup, G - gfirst);
    for (int i = tid; i < C::NPART; i += 128) __stcg(p.cta_part + (int64_t)blockIdx.x * C::NPART + i, red[i]);
    named_bar_sync(2, 128);
    if (tid == 0) {
      fence_acq_rel_gpu();
      const int is_last = (atomicAdd(p.done_cnt + 1 + gi, 1u) == (unsigned)gsize - 1u);
      if (is_last) fence_acq_rel_gpu();
      *flag = is_last;
    }
    named_bar_sync(2, 128);
    if (*flag) {
      for (int i = tid; i < C::NPART; i += 128) {
        double v = 0.0;
#pragma unroll
        for (int b = 0; b < kTcGroup; ++b)
          if (b < gsize) v += __ldcg(p.cta_part + (int64_t)(gfirst + b) * C::NPART + i);
        __stcg(grp + (int64_t)gi * C::NPART + i, v);
      }
      named_bar_sync(2, 128);
      if (tid == 0) {
        p.done_cnt[1 + gi] = 0u;
        fence_acq_rel_gpu();
        const int is_last = (atomicAdd(p.done_cnt, 1u) == (unsigned)ngrp - 1u);
        if (is_last) fence_acq_rel_gpu();
        *flag = is_last;
      }
      named_bar_sync(2, 128);
      if (*flag) {
        for (int i = tid; i < C::NPART; i += 128) {
          double v = 0.0;
          for (int g = 0; g < ngrp; ++g) v += __ldcg(grp + (int64_t)g * C::NPART + i);
          p.result[i] = v;
        }
        if (tid == 0) *p.done_cnt = 0u;
      }
    }
    if (timed && tid == 0) {
      unsigned long long *ts = p.ts + (size_t)blockIdx.x * kTsSlots;
      ts[8] = (unsigned long long)t_wait;
      ts[9] = (unsigned long long)(t_stream - t_begin);
      ts[10] = (unsigned long long)t_epi;
      ts[11] = (unsigned long long)(t_shared - t_stream);
      ts[12] = (unsigned long long)(clock64() - t_shared);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 13) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

template <int D, int MODE, int MH, bool NL = false>
static cudaError_t tc_launch(const CUtensorMap *tm, const PanelParams &p, int grid, cudaStream_t s) {
  using C = TcCfg<D, MH>;
  auto kern = wide_tc_kernel<D, MODE, MH, NL>;
  static bool attr[64] = {};
  {
    const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void *>(kern), C::SMEM, attr);
    if (e != cudaSuccess) return e;
  }
  // CTAs sharing a split panel wait for each other's partial rows, so the whole grid (<= one CTA
  // per SM) must be co-resident: a cooperative launch guarantees it (or waits / fails, never hangs)
  CUtensorMap tmv = *tm;
  PanelParams pv = p;
  void *args[] = {&tmv, &pv};
  return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kern), dim3(grid), dim3(C::THREADS), args, C::SMEM, s);
}

template <int D, int MH, bool NL = false>
static cudaError_t tc_mode(int mode, const CUtensorMap *tm, const PanelParams &p, int grid, cudaStream_t s) {
  if (mode == kModeRgs) return tc_launch<D, kModeRgs, MH, NL>(tm, p, grid, s);
  if (mode == kModeObjective) return tc_launch<D, kModeObjective, MH, NL>(tm, p, grid, s);
  if (mode == kModeGpm) return tc_launch<D, kModeGpm, MH, NL>(tm, p, grid, s);
  return tc_launch<D, kModeProduct, MH, NL>(tm, p, grid, s);
}

// The block sizes are instantiated in four translation units (NSRGS_TC_PART = 0..3, balanced by
// compile time: one nvcc run over all of them takes > 8 minutes); part 0 also holds the dispatcher.
#ifndef NSRGS_TC_PART
#define NSRGS_TC_PART 0
#endif
#define NSRGS_TC_CASE(DV)                                                                          \
  case DV: {                                                                                       \
    using C = TcCfg<DV, 2>;                                                                        \
    if (shape_only) {                                                                              \
      *shape = PanelShape{C::ROWS, C::NPP, C::STAGES, C::SMEM, C::NPART, C::THREADS, 4};          \
      if (slot_floats) *slot_floats = C::MROWS * C::NP;                                            \
      *err = cudaSuccess;                                                                          \
      return true;                                                                                 \
    }                                                                                              \
    *err = tc_mode<DV, 2>(mode, tm, *p, grid, s);                                                  \
    return true;                                                                                   \
  }
#define NSRGS_TC_PART_FN(K) wide_tc_part##K
#define NSRGS_TC_PART_NAME(K) NSRGS_TC_PART_FN(K)

// true if this part instantiates block size d (then *err is the shape query's / launch's status)
bool NSRGS_TC_PART_NAME(NSRGS_TC_PART)(int d, int mode, bool shape_only, PanelShape *shape, int *slot_floats,
                                       const CUtensorMap *tm, const PanelParams *p, int grid, cudaStream_t s,
                                       cudaError_t *err) {
  switch (d) {
#if NSRGS_TC_PART == 0
    case 10: {   // d = 10 in the narrow X layout (runtime: ctx->narrow_tc)
      using C = TcCfg<10, 2>;
      if (shape_only) {
        *shape = PanelShape{C::ROWS, C::NPP, C::STAGES, C::SMEM, C::NPART, C::THREADS, 4};
        if (slot_floats) *slot_floats = C::MROWS * C::NP;
        *err = cudaSuccess;
        return true;
      }
      *err = tc_mode<10, 2, true>(mode, tm, *p, grid, s);
      return true;
    }
    NSRGS_TC_CASE(11)
    NSRGS_TC_CASE(12)
    NSRGS_TC_CASE(13)
    NSRGS_TC_CASE(14)
    NSRGS_TC_CASE(15)
#elif NSRGS_TC_PART == 1
    NSRGS_TC_CASE(16)
    NSRGS_TC_CASE(25)
#elif NSRGS_TC_PART == 2
    NSRGS_TC_CASE(20)
    NSRGS_TC_CASE(24)
#else
    NSRGS_TC_CASE(32)
#endif
    default: return false;
  }
}
#undef NSRGS_TC_CASE

#if NSRGS_TC_PART == 0
bool wide_tc_part1(int, int, bool, PanelShape *, int *, const CUtensorMap *, const PanelParams *, int, cudaStream_t, cudaError_t *);
bool wide_tc_part2(int, int, bool, PanelShape *, int *, const CUtensorMap *, const PanelParams *, int, cudaStream_t, cudaError_t *);
bool wide_tc_part3(int, int, bool, PanelShape *, int *, const CUtensorMap *, const PanelParams *, int, cudaStream_t, cudaError_t *);

// slot_floats: floats of one CTA's partial-row slot (the runtime allocates 2 slots + 2 flags per CTA)
cudaError_t wide_tc_dispatch(int d, int mode, bool shape_only, PanelShape *shape, int *slot_floats,
                             const CUtensorMap *tm, const PanelParams *p, int grid, cudaStream_t s) {
  cudaError_t err = cudaErrorInvalidValue;
  if (wide_tc_part0(d, mode, shape_only, shape, slot_floats, tm, p, grid, s, &err) ||
      wide_tc_part1(d, mode, shape_only, shape, slot_floats, tm, p, grid, s, &err) ||
      wide_tc_part2(d, mode, shape_only, shape, slot_floats, tm, p, grid, s, &err) ||
      wide_tc_part3(d, mode, shape_only, shape, slot_floats, tm, p, grid, s, &err))
    return err;
  return cudaErrorInvalidValue;
}
#endif

}  // namespace nsrgs
