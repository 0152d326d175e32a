// panel.cu — the NS-RGS hot path: one streaming pass of the A shard per launch.
//
//   B = A_shard . X            (Alg. 2 "G_i^t = sum_{j!=i}(X_i^t - A_ij X_j^t)")
//   G_i = (n-1) X_i - B_i      (A_ii = 0)
//   P_i = (G_i - X_i G_i^T X_i)/2,  F_i = X_i - eta P_i
//   X_i^{t+1} = S(F_i): K steps S <- 1/2 S (3I - S^T S)
//
// Design: persistent grid, one CTA per SM, 7 consumer warps + 1 TMA
// producer warp.  Work units (a row panel of ROWS = 7 RT rows, or a column range of one) come
// from an atomic queue.  The producer streams A tiles (ROWS x 128, 3-D tensor map over
// (col-in-rank-slice, rank slice, row)) and the matching X tile (d x 128, contiguous in the
// tile layout) into an mbarrier ring, A with an L2 evict-first (or fractional evict-last)
// policy, X evict-last.  Each consumer warp owns RT rows (= whole nodes); lane l owns 4
// columns of every tile and keeps RT x d fp32 accumulators in registers (FFMA2 on component
// pairs), so every X value read from smem is reused RT times and A is read from smem once.
// At the end of a panel the warp reduces its accumulators with shuffles and runs the per-node
// epilogue entry-parallel in warp-private smem; no B is ever written to HBM.  Objective / Gram
// partials are summed exactly in 128-bit fixed point (deterministic under any schedule).
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"
#include "epilogue.cuh"

namespace nsrgs {

template <typename T, int D>
struct PanelCfg {
  static constexpr int RT = (sizeof(T) == 4)
                                ? (D == 2 ? 12 : D == 3 ? 12 : D == 4 ? 12 : D == 5 ? 10 : D == 6 ? 12
                                   : D == 7 ? 7 : D == 8 ? 8 : D == 9 ? 9 : 10)
                                : (D == 2 ? 6 : D == 3 ? 6 : D == 4 ? 4 : D == 5 ? 5 : 6);
  static_assert(RT % D == 0, "warp rows must be whole nodes");
  static constexpr int NPW = RT / D;
  static constexpr int ROWS = RT * kWarps;
  static constexpr int NODES = ROWS / D;
  static constexpr int A_BYTES = ROWS * kColTile * (int)sizeof(T);
  static constexpr int KP = D / 2;                 // component pairs (2kp, 2kp+1)
  static constexpr bool ODD = (D & 1) != 0;        // last component handled with column pairs
  static constexpr int X_BYTES = D * kColTile * (int)sizeof(T);
  static constexpr int STAGE_BYTES = A_BYTES + X_BYTES;
  static constexpr int E = NPW * D * D;          // epilogue entries per warp
  static constexpr int EPL = (E + 31) / 32;      // entries per lane
  static constexpr int DD = D * D;
  static constexpr int DDL = (DD + 31) / 32;     // Gram entries per lane
  static constexpr int NPART = 2 * DD + 2;
  // shared memory after the stages
  static constexpr int BAR_BYTES = 2 * 8 * 8;                         // up to 8 stages
  static constexpr int VW = 16 / (int)sizeof(T);                      // elements per 16 B
  static constexpr int EP = (E + VW - 1) / VW * VW;                  // E padded to 16 B
  static constexpr int SCR_T = 5 * EP;                                // sX sG sH sS sM
  static constexpr int SCR_T_BYTES = (kWarps * SCR_T * (int)sizeof(T) + 15) / 16 * 16;   // keep doubles aligned
  static constexpr int SCR_BYTES = SCR_T_BYTES + kWarps * NPART * 16 + 8 * 8 + 64;   // + fixed-point slices, meta, flag
  static constexpr int BUDGET = 220 * 1024;
  static constexpr int STAGES_RAW = (BUDGET - 1024 - BAR_BYTES - SCR_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static_assert(STAGES >= 2, "need a double-buffered ring");
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + BAR_BYTES + SCR_BYTES;
};


// After warp_sum every lane holds all RT x D sums of the warp; lane 0 writes them (zero-padded
// to 16 B) with vector stores to a 16-byte aligned destination.  (Picking value r*D+k in lane
// (r*D+k)%32 compiles to a divergent switch over the lane id: ~2 us per panel hand-off.)
template <typename T, int RT, int D, bool GLOBAL>
__device__ __forceinline__ void lane0_store_rows(T *dst, const T (&acc)[RT][D], int lane) {
  if (lane != 0) return;
  constexpr int N = RT * D, VW = 16 / (int)sizeof(T);
#pragma unroll
  for (int e = 0; e < N; e += VW) {
    T v[VW];
#pragma unroll
    for (int j = 0; j < VW; ++j) v[j] = (e + j < N) ? acc[(e + j) / D][(e + j) % D] : T(0);
    if constexpr (sizeof(T) == 4) {
      const float4 f = make_float4(v[0], v[1], v[2], v[3]);
      if constexpr (GLOBAL) __stcg(reinterpret_cast<float4 *>(dst + e), f);
      else *reinterpret_cast<float4 *>(dst + e) = f;
    } else {
      const double2 f = make_double2(v[0], v[1]);
      if constexpr (GLOBAL) __stcg(reinterpret_cast<double2 *>(dst + e), f);
      else *reinterpret_cast<double2 *>(dst + e) = f;
    }
  }
}

__device__ __forceinline__ uint64_t pack2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack2(uint64_t v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
// d = a * b + c on two packed fp32 lanes (sm_100a FFMA2; round-to-nearest like fmaf)
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}


// Column-tile order within a panel: this rank's own X slice first (ready earliest under P > 1).
__device__ __forceinline__ int tile_of_step(int t, const PanelParams &p) {
  const int tpr = (int)p.tiles_per_rank;
  const int g = t / tpr;
  return ((g + p.rank) % p.world) * tpr + (t - g * tpr);
}

// ---- exact order-independent fp64 sums: 128-bit fixed point with 40 fraction bits.
// Objective / Gram partials are converted per (panel, warp) epilogue and added as integers, so
// the totals do not depend on which CTA ran which unit (bitwise-deterministic results under
// the dynamic schedule).  |partial| < 2^86; resolution 2^-40 ~ 9e-13 absolute, far below the
// fp64 rounding of the O(1e4..1e10) terms it sums.
constexpr double kFixScale = 1099511627776.0;   // 2^40
constexpr double kTwo64 = 18446744073709551616.0;
__device__ __forceinline__ void fix_from(double v, unsigned long long &lo, long long &hi, int &err) {
  if (!(fabs(v) < 1e25)) {   // non-finite or out of range
    err |= kErrNonfinite;
    v = 0.0;
  }
  const double sc = v * kFixScale;                  // exact (power of two)
  const double h = floor(sc * (1.0 / kTwo64));      // exact
  hi = (long long)h;
  lo = (unsigned long long)(sc - h * kTwo64);       // in [0, 2^64), exact up to sc's own ulp
}
__device__ __forceinline__ void fix_add(unsigned long long &lo, long long &hi, unsigned long long alo, long long ahi) {
  const unsigned long long s = lo + alo;
  hi += ahi + (s < lo ? 1ll : 0ll);
  lo = s;
}
__device__ __forceinline__ void fix_atomic_add(unsigned long long *g, unsigned long long lo, long long hi) {
  if (lo == 0ull && hi == 0ll) return;
  const unsigned long long old = atomicAdd(g, lo);
  atomicAdd(g + 1, (unsigned long long)hi + (old + lo < old ? 1ull : 0ull));
}
__device__ __forceinline__ double fix_to(unsigned long long lo, long long hi) {
  return (double)hi * (kTwo64 / kFixScale) + (double)lo * (1.0 / kFixScale);
}

struct UnitMeta {   // published by the producer per stage: global unit index (-1: no more work), tile step
  int kg, t;
};

// Dense pass.  Persistent CTAs (one per SM) take work units from an atomic queue that runs over
// iters x nunits (iteration-major).  A unit is a whole row panel or, for the tail of the list,
// an equal column range of one; per-SM bandwidth differs by a few % (GPC population), so the
// dynamic queue, not a static split, balances the pass.  Each consumer warp owns RT rows of the
// panel; at the end of a split unit it publishes its partial rows and the last of the panel's
// units to arrive (per warp) sums them in column order and runs the epilogue for its nodes.
template <typename T, int D, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    panel_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ PanelParams p) {
  using C = PanelCfg<T, D>;
  using V = typename Vec4<T>::type;
  extern __shared__ uint8_t smem_raw[];
  // align to 1 KB by offsetting the shared array itself (keeps the shared address space, so
  // every smem access below compiles to LDS/STS rather than generic LD/ST)
  uint8_t *smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *empty = full + 8;
  T *scr_all = reinterpret_cast<T *>(smem + C::STAGES * C::STAGE_BYTES + C::BAR_BYTES);
  unsigned long long *fix_all =
      reinterpret_cast<unsigned long long *>(reinterpret_cast<uint8_t *>(scr_all) + C::SCR_T_BYTES);   // [kWarps][NPART][2]
  UnitMeta *meta = reinterpret_cast<UnitMeta *>(fix_all + kWarps * C::NPART * 2);                     // [8]
  int *flag = reinterpret_cast<int *>(meta + 8);
  unsigned *epi_tot = reinterpret_cast<unsigned *>(flag + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
    *epi_tot = 0u;
  }
  for (int i = threadIdx.x; i < kWarps * C::NPART * 2; i += kThreads) fix_all[i] = 0ull;
  __syncthreads();
  const int total_units = p.iters * p.nunits;
  const unsigned epi_per_iter = (unsigned)p.panels * kWarps;

  // ------------------------------------------------------------------ producer warp
  if (warp == kWarps) {
    if (elect_one()) {   // one lane; the TMA instructions issue straight-line (no per-instruction ELECT loop)
      prefetch_tmap(&tmA);
      const uint64_t pol_frac = p.a_keep > 0.f ? policy_keep_fraction(p.a_keep) : policy_evict_first();
      const uint64_t pol_keep = policy_evict_last(), pol_stream = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      int ready_it = 0;   // X^it known complete for it <= ready_it
      unsigned slice_ready = 0u;   // P2P: rank slices of X^0 known complete
      int ts_it = -1;
      for (;;) {
        const int kg = (int)atomicAdd(&p.ctl[0], 1u);
        if (kg >= total_units) {
          mbar_wait(&empty[stage], phase ^ 1u);
          meta[stage].kg = -1;
          mbar_arrive(&full[stage]);
          break;
        }
        const int it = kg / p.nunits;
        const int4 u = __ldg(p.units + (kg - it * p.nunits));
        const uint64_t pol_a = p.keep_panels > 0 ? (u.x < p.keep_panels ? pol_keep : pol_stream) : pol_frac;
        const T *Xin = static_cast<const T *>((it & 1) ? p.Xout : p.X);
        unsigned long long *ts = p.ts ? p.ts + ((int64_t)it * gridDim.x + blockIdx.x) * kTsSlots : nullptr;
        if (ts && it != ts_it) { ts[0] = globaltimer(); ts_it = it; }
        for (int t = u.y; t < u.z; ++t) {
          const int tt = tile_of_step(t, p);
          const int g = tt / (int)p.tiles_per_rank, jt = tt - g * (int)p.tiles_per_rank;
          mbar_wait(&empty[stage], phase ^ 1u);
          meta[stage].kg = kg;
          meta[stage].t = t;
          uint8_t *sb = smem + stage * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_3d(sb, &tmA, &full[stage], jt * kColTile, g, u.x * C::ROWS, pol_a);
          if (p.p2p && !((slice_ready >> g) & 1u)) {
            // fused exchange: rank g's slice of X^t is complete once all its (panel, warp)
            // epilogues of the previous iteration have been counted here
            unsigned spins = 0;
            while (ld_acquire_sys(p.xcnt + g) < p.xtarget) {
              __nanosleep(128);
              if (++spins > (1u << 26)) { atomicOr(p.err, kErrTimeout); break; }
            }
            fence_proxy_async_global();
            slice_ready |= 1u << g;
          }
          if (it > ready_it) {
            // A of this unit is in flight; X^it needs every (panel, warp) epilogue of it-1
            const unsigned target = (unsigned)it * epi_per_iter;
            unsigned spins = 0;
            while (ld_acquire_gpu(&p.ctl[1]) < target) {
              __nanosleep(64);
              if (++spins > (1u << 26)) { atomicOr(p.err, kErrTimeout); break; }
            }
            fence_proxy_async_global();
            ready_it = it;
            if (ts) ts[1] = globaltimer();
          }
          bulk_load(sb + C::A_BYTES, Xin + (int64_t)tt * D * kColTile, C::X_BYTES, &full[stage], pol_x);
          if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumer warps
  T *sX = scr_all + warp * C::SCR_T;
  T *sG = sX + C::EP;   // 16-byte aligned: lane 0 fills it with vector stores
  T *sH = sG + C::EP;
  T *sS = sH + C::EP;
  T *sM = sS + C::EP;
  unsigned long long *fixw = fix_all + warp * C::NPART * 2;   // this warp's fixed-point sums
  float ns_region = 0.f;
  int err = 0;
  unsigned n_epi = 0;   // (panel, warp) epilogues run by this warp (P2P arrival count)

  // CTA-wide: add the warps' fixed-point sums of iteration `it` to the global accumulators.
  // All consumer warps process the same unit sequence, so they all reach this together.
  auto flush = [&](int it) {
    named_bar_sync(1, kWarps * 32);
    for (int i = threadIdx.x; i < C::NPART; i += kWarps * 32) {
      unsigned long long lo = 0ull;
      long long hi = 0ll;
      for (int w = 0; w < kWarps; ++w) {
        unsigned long long *f = fix_all + (w * C::NPART + i) * 2;
        fix_add(lo, hi, f[0], (long long)f[1]);
        f[0] = 0ull;
        f[1] = 0ull;
      }
      fix_atomic_add(p.acc + ((int64_t)it * C::NPART + i) * 2, lo, hi);
    }
    named_bar_sync(1, kWarps * 32);
  };

  int stage = 0;
  uint32_t phase = 0;
  int cur_it = -1;
  unsigned long long *cts = nullptr;
  for (;;) {
    mbar_wait(&full[stage], phase);
    const int kg = meta[stage].kg;
    if (kg < 0) break;
    const int it = kg / p.nunits;
    if (it != cur_it) {
      if (cur_it >= 0) {
        flush(cur_it);
        if (cts) cts[3] = globaltimer();
      }
      cur_it = it;
      cts = (p.ts && threadIdx.x == 0) ? p.ts + ((int64_t)it * gridDim.x + blockIdx.x) * kTsSlots : nullptr;
      if (cts) {
        cts[2] = globaltimer();
        unsigned sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        cts[11] = sm;
      }
    }
    const int4 u = __ldg(p.units + (kg - it * p.nunits));
    const int panel = u.x, t0 = u.y, t1 = u.z, slot = u.w;
    // iteration it reads X^it and writes X^{it+1} (buffers alternate; no parameter copy)
    const T *Xg = static_cast<const T *>((it & 1) ? p.Xout : p.X);
    void *Xo_it = (it & 1) ? const_cast<void *>(p.X) : p.Xout;
    const int64_t node_base = (int64_t)panel * C::NODES + warp * C::NPW;   // local node of q = 0
    const int64_t rem = p.n_local - node_base;
    const int nvalid = rem <= 0 ? 0 : (rem < C::NPW ? (int)rem : C::NPW);
    // X_i of this warp's nodes for the epilogue, in flight during the stream.  Issued after the
    // unit's first stage has landed: X^it is only guaranteed complete (every epilogue of it-1)
    // once the producer passed its readiness wait and that stage's barrier completed (writers'
    // release -> producer acquire -> mbarrier arrive / wait).
    T xpre[C::EPL];
    epi_load_x<T, D, C::NPW>(p, Xg, lane, node_base, nvalid, xpre);

    // Lane l owns columns {2l, 2l+1, 64+2l, 65+2l} of each 128-column tile: A row pieces are
    // conflict-free 64-bit smem loads, X component pairs conflict-free 128-bit loads.
    T acc[C::RT][D];
    if constexpr (sizeof(T) == 4) {
      // fp32: packed FFMA2 on component pairs (acc[r][2kp], acc[r][2kp+1]) += (x_2kp, x_2kp+1) * a,
      // and for odd d the last component on column pairs (even, odd column sums) += (a_c, a_c+1) * (x_c, x_c+1)
      constexpr int KL = C::ODD ? 1 : 0;
      uint64_t acc2[C::RT][C::KP + KL];
#pragma unroll
      for (int r = 0; r < C::RT; ++r)
#pragma unroll
        for (int kp = 0; kp < C::KP + KL; ++kp) acc2[r][kp] = 0ull;
      for (int t = t0; t < t1; ++t) {
        if (t > t0) mbar_wait(&full[stage], phase);
        const float *As = reinterpret_cast<const float *>(smem + stage * C::STAGE_BYTES) + (warp * C::RT) * kColTile + 2 * lane;
        const float *Xt = reinterpret_cast<const float *>(smem + stage * C::STAGE_BYTES + C::A_BYTES);
        const float *Xs = Xt + 4 * lane;
        uint64_t xp[C::KP + KL][4];   // pairs for the lane's 4 columns (+ last-component column pairs)
#pragma unroll
        for (int kp = 0; kp < C::KP; ++kp) {
          const ulonglong2 lo = *reinterpret_cast<const ulonglong2 *>(Xs + kp * 2 * kColTile);
          const ulonglong2 hi = *reinterpret_cast<const ulonglong2 *>(Xs + kp * 2 * kColTile + kColTile);
          xp[kp][0] = lo.x; xp[kp][1] = lo.y; xp[kp][2] = hi.x; xp[kp][3] = hi.y;
        }
        if constexpr (C::ODD) {
          xp[C::KP][0] = *reinterpret_cast<const uint64_t *>(Xt + (D - 1) * kColTile + 2 * lane);
          xp[C::KP][1] = *reinterpret_cast<const uint64_t *>(Xt + (D - 1) * kColTile + 64 + 2 * lane);
        }
#pragma unroll
        for (int r = 0; r < C::RT; ++r) {
          const uint64_t a0 = *reinterpret_cast<const uint64_t *>(As + r * kColTile);        // (A[r][2l], A[r][2l+1])
          const uint64_t a1 = *reinterpret_cast<const uint64_t *>(As + r * kColTile + 64);   // (.., 64+2l, 65+2l)
          float f0, f1, f2, f3;
          unpack2(a0, f0, f1);
          unpack2(a1, f2, f3);
          const uint64_t b0 = pack2(f0, f0), b1 = pack2(f1, f1);
          const uint64_t b2 = pack2(f2, f2), b3 = pack2(f3, f3);
#pragma unroll
          for (int kp = 0; kp < C::KP; ++kp) {
            uint64_t v = acc2[r][kp];
            v = ffma2(xp[kp][0], b0, v);
            v = ffma2(xp[kp][1], b1, v);
            v = ffma2(xp[kp][2], b2, v);
            v = ffma2(xp[kp][3], b3, v);
            acc2[r][kp] = v;
          }
          if constexpr (C::ODD) {
            uint64_t v = acc2[r][C::KP];
            v = ffma2(a0, xp[C::KP][0], v);
            v = ffma2(a1, xp[C::KP][1], v);
            acc2[r][C::KP] = v;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
      }
#pragma unroll
      for (int r = 0; r < C::RT; ++r) {
#pragma unroll
        for (int kp = 0; kp < C::KP; ++kp) {
          float lo, hi;
          unpack2(acc2[r][kp], lo, hi);
          acc[r][2 * kp] = (T)lo;
          acc[r][2 * kp + 1] = (T)hi;
        }
        if constexpr (C::ODD) {
          float lo, hi;
          unpack2(acc2[r][C::KP], lo, hi);
          acc[r][D - 1] = (T)(lo + hi);
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < C::RT; ++r)
#pragma unroll
        for (int k = 0; k < D; ++k) acc[r][k] = T(0);
      for (int t = t0; t < t1; ++t) {
        if (t > t0) mbar_wait(&full[stage], phase);
        const T *As = reinterpret_cast<const T *>(smem + stage * C::STAGE_BYTES) + (warp * C::RT) * kColTile + 2 * lane;
        const T *Xs = reinterpret_cast<const T *>(smem + stage * C::STAGE_BYTES + C::A_BYTES) + 4 * lane;
        T xv[D][4];
#pragma unroll
        for (int kp = 0; kp < C::KP; ++kp) {
          const V lo = *reinterpret_cast<const V *>(Xs + kp * 2 * kColTile);
          const V hi = *reinterpret_cast<const V *>(Xs + kp * 2 * kColTile + kColTile);
          xv[2 * kp][0] = lo.x; xv[2 * kp + 1][0] = lo.y; xv[2 * kp][1] = lo.z; xv[2 * kp + 1][1] = lo.w;
          xv[2 * kp][2] = hi.x; xv[2 * kp + 1][2] = hi.y; xv[2 * kp][3] = hi.z; xv[2 * kp + 1][3] = hi.w;
        }
        if constexpr (C::ODD) {
          const T *Xl = reinterpret_cast<const T *>(smem + stage * C::STAGE_BYTES + C::A_BYTES) + (D - 1) * kColTile;
          xv[D - 1][0] = Xl[2 * lane]; xv[D - 1][1] = Xl[2 * lane + 1];
          xv[D - 1][2] = Xl[64 + 2 * lane]; xv[D - 1][3] = Xl[65 + 2 * lane];
        }
#pragma unroll
        for (int r = 0; r < C::RT; ++r) {
          T a[4];
          a[0] = As[r * kColTile]; a[1] = As[r * kColTile + 1];
          a[2] = As[r * kColTile + 64]; a[3] = As[r * kColTile + 65];
#pragma unroll
          for (int k = 0; k < D; ++k) {
            T v = acc[r][k];
#pragma unroll
            for (int j = 0; j < 4; ++j) v = tfma(a[j], xv[k][j], v);
            acc[r][k] = v;
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
      }
    }

    if (cts) cts[5] = globaltimer();   // streaming of this unit done
    // ---- reduce the lane-partial sums: every lane ends with the full B rows of the warp
#pragma unroll
    for (int r = 0; r < C::RT; ++r)
#pragma unroll
      for (int k = 0; k < D; ++k) acc[r][k] = warp_sum(acc[r][k]);

    if (slot >= 0) {
      // Split panel: publish this warp's partial rows; the last of the panel's units to arrive
      // (counted per (panel, warp), no CTA barrier) sums all of them in column order.
      T *bp = static_cast<T *>(p.Bpart) + ((int64_t)slot * kWarps + warp) * C::EP;
      lane0_store_rows<T, C::RT, D, true>(bp, acc, lane);
      __syncwarp();
      const int2 pi = __ldg(p.pinfo + panel);   // (units of the panel, first slot)
      int last = 0;
      if (lane == 0) {
        fence_acq_rel_gpu();
        unsigned *cnt = p.ucnt + panel * kWarps + warp;
        last = atomicAdd(cnt, 1u) == (unsigned)(pi.x - 1);
        if (last) {
          fence_acq_rel_gpu();
          *cnt = 0u;   // ready for the next iteration / launch
        }
      }
      if (!__shfl_sync(0xffffffffu, last, 0)) continue;
      const T *bpr = static_cast<const T *>(p.Bpart) + (int64_t)warp * C::EP;
      T v[C::EPL];
#pragma unroll
      for (int m = 0; m < C::EPL; ++m) v[m] = T(0);
      for (int j0 = 0; j0 < pi.x; j0 += 4) {   // 4 slots x EPL independent loads in flight
        T part[4][C::EPL];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const T *src = bpr + (int64_t)(pi.y + j0 + j) * kWarps * C::EP;
#pragma unroll
          for (int m = 0; m < C::EPL; ++m) {
            const int e = lane + 32 * m;
            part[j][m] = (j0 + j < pi.x && e < C::E) ? __ldcg(src + e) : T(0);
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int m = 0; m < C::EPL; ++m) v[m] += part[j][m];
      }
#pragma unroll
      for (int m = 0; m < C::EPL; ++m)
        if (lane + 32 * m < C::E) sG[lane + 32 * m] = v[m];
    } else {
      lane0_store_rows<T, C::RT, D, false>(sG, acc, lane);
    }

    if (cts) cts[6] = globaltimer();   // B rows of the panel complete (combine done)
    // ---- per-node epilogue (epilogue.cuh), entry-parallel in warp-private smem.
    double g1s[C::DDL], g2s[C::DDL], so = 0.0, xs = 0.0;
    node_epilogue<T, D, C::NPW, MODE, true>(p, Xg, Xo_it, lane, node_base, nvalid, sX, sG, sH, sS, sM, g1s, g2s, so, xs,
                                            ns_region, err, xpre);
    // exact partial sums of this (panel, warp) into the warp's fixed-point accumulators
#pragma unroll
    for (int m = 0; m < C::DDL; ++m) {
      const int e = lane + 32 * m;
      if (e < C::DD) {
        unsigned long long lo;
        long long hi;
        fix_from(g1s[m], lo, hi, err);
        fix_add(fixw[2 * e], *reinterpret_cast<long long *>(&fixw[2 * e + 1]), lo, hi);
        fix_from(g2s[m], lo, hi, err);
        fix_add(fixw[2 * (C::DD + e)], *reinterpret_cast<long long *>(&fixw[2 * (C::DD + e) + 1]), lo, hi);
      }
    }
    so = warp_sum(so);
    xs = warp_sum(xs);
    if (lane == 0) {
      unsigned long long lo;
      long long hi;
      fix_from(so, lo, hi, err);
      fix_add(fixw[2 * (2 * C::DD)], *reinterpret_cast<long long *>(&fixw[2 * (2 * C::DD) + 1]), lo, hi);
      fix_from(xs, lo, hi, err);
      fix_add(fixw[2 * (2 * C::DD + 1)], *reinterpret_cast<long long *>(&fixw[2 * (2 * C::DD + 1) + 1]), lo, hi);
    }
    __syncwarp();
    ++n_epi;
    if (p.iters > 1 && lane == 0) {   // this warp's rows of X^{it+1} are written
      fence_acq_rel_gpu();
      atomicAdd(&p.ctl[1], 1u);
    }
  }

  // ------------------------------------------------------------------ exit
  if (cur_it >= 0) {
    flush(cur_it);
    if (cts) cts[3] = globaltimer();
  }
  if (err) atomicOr(p.err, err);
  if (MODE == kModeRgs || MODE == kModeGpm) {
    float mx = ns_region;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0 && mx > 0.f) atomicMax(p.ns_region, __float_as_uint(mx));
  }
  if (p.p2p && lane == 0 && n_epi) atomicAdd(epi_tot, n_epi);
  named_bar_sync(1, kWarps * 32);
  if (threadIdx.x == 0) {
    if (p.p2p && *epi_tot) {
      // every consumer's X^{t+1} stores (local and remote) precede the barrier; one
      // system-scope release, then this CTA's epilogue count to every rank's counter[rank]
      fence_acq_rel_sys();
      for (int g = 0; g < p.world; ++g) red_add_sys(p.peer_cnt[g] + p.rank, *epi_tot);
    }
    fence_acq_rel_gpu();
    const int is_last = atomicAdd(&p.ctl[2], 1u) == gridDim.x - 1;
    if (is_last) fence_acq_rel_gpu();
    *flag = is_last;
  }
  named_bar_sync(1, kWarps * 32);
  if (*flag) {   // last CTA out: fixed point -> fp64 results, re-zero, reset the queue counters
    const int nval = p.iters * C::NPART;
    for (int i = threadIdx.x; i < nval; i += kWarps * 32) {
      unsigned long long *a = p.acc + (int64_t)i * 2;
      const unsigned long long lo = __ldcg(a);
      const long long hi = (long long)__ldcg(a + 1);
      p.result[i] = fix_to(lo, hi);
      a[0] = 0ull;
      a[1] = 0ull;
    }
    if (threadIdx.x == 0) {
      p.ctl[0] = 0u;
      p.ctl[1] = 0u;
      p.ctl[2] = 0u;
    }
  }
  if (cts) cts[4] = globaltimer();
}

// End of a fused-exchange run: every peer's stores into this rank's X buffers have landed once
// all arrival counters reached `target` (so the host may reuse / overwrite X afterwards).
__global__ void p2p_wait_kernel(const unsigned *xcnt, int world, unsigned target, int *err) {
  if (threadIdx.x < world) {
    unsigned spins = 0;
    while (ld_acquire_sys(xcnt + threadIdx.x) < target) {
      __nanosleep(256);
      if (++spins > (1u << 26)) { atomicOr(err, kErrTimeout); break; }
    }
  }
}
cudaError_t launch_p2p_wait(const unsigned *xcnt, int world, unsigned target, int *err, cudaStream_t s) {
  p2p_wait_kernel<<<1, 32, 0, s>>>(xcnt, world, target, err);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ host-side launchers
template <typename T, int D, int MODE>
static cudaError_t launch_impl(const CUtensorMap *tm, const PanelParams &p, int grid, cudaStream_t s) {
  using C = PanelCfg<T, D>;
  auto kern = panel_kernel<T, D, MODE>;
  static bool attr_set[64] = {};
  {
    const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void *>(kern), C::SMEM, attr_set);
    if (e != cudaSuccess) return e;
  }
  if (p.iters > 1) {   // all CTAs must be co-resident for the in-kernel grid barrier
    CUtensorMap tmc = *tm;
    PanelParams pc = p;
    void *args[] = {&tmc, &pc};
    return cudaLaunchCooperativeKernel(reinterpret_cast<const void *>(kern), dim3(grid), dim3(kThreads), args,
                                       (size_t)C::SMEM, s);
  }
  kern<<<grid, kThreads, C::SMEM, s>>>(*tm, p);
  return cudaGetLastError();
}

template <typename T, int D>
static PanelShape shape_impl() {
  using C = PanelCfg<T, D>;
  return PanelShape{C::ROWS, C::NODES, C::STAGES, C::SMEM, C::NPART, kThreads, kWarps};
}

#define NSRGS_PANEL_CASE(T, D)                                                               \
  case D:                                                                                    \
    if (shape_only) { *shape = shape_impl<T, D>(); return cudaSuccess; }                     \
    if (mode == kModeRgs) return launch_impl<T, D, kModeRgs>(tm, *p, grid, s);               \
    if (mode == kModeObjective) return launch_impl<T, D, kModeObjective>(tm, *p, grid, s);   \
    if (mode == kModeGpm) return launch_impl<T, D, kModeGpm>(tm, *p, grid, s);               \
    return launch_impl<T, D, kModeProduct>(tm, *p, grid, s);

cudaError_t panel_dispatch(int dtype, int d, int mode, bool shape_only, PanelShape *shape,
                           const CUtensorMap *tm, const PanelParams *p, int grid, cudaStream_t s) {
  if (dtype == 0) {
    switch (d) {
      NSRGS_PANEL_CASE(float, 2)
      NSRGS_PANEL_CASE(float, 3)
      NSRGS_PANEL_CASE(float, 4)
      NSRGS_PANEL_CASE(float, 5)
      NSRGS_PANEL_CASE(float, 6)
      NSRGS_PANEL_CASE(float, 7)
      NSRGS_PANEL_CASE(float, 8)
      NSRGS_PANEL_CASE(float, 9)
      NSRGS_PANEL_CASE(float, 10)
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (d) {
      NSRGS_PANEL_CASE(double, 2)
      NSRGS_PANEL_CASE(double, 3)
      NSRGS_PANEL_CASE(double, 4)
      NSRGS_PANEL_CASE(double, 5)
      NSRGS_PANEL_CASE(double, 6)
      default: return cudaErrorInvalidValue;
    }
  }
}

}  // namespace nsrgs
