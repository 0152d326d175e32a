// panel.cu — the NS-RGS hot path: one streaming pass of the A shard per launch.
//
//   B = A_shard . X            (Alg. 2 "G_i^t = sum_{j!=i}(X_i^t - A_ij X_j^t)")
//   G_i = (n-1) X_i - B_i      (A_ii = 0)
//   P_i = (G_i - X_i G_i^T X_i)/2,  F_i = X_i - eta P_i
//   X_i^{t+1} = S(F_i): K steps S <- 1/2 S (3I - S^T S)
//
// Design: persistent grid, one CTA per SM, 8 consumer warps + 1 TMA
// producer warp.  Work unit = (row panel of ROWS = 8*RT rows, column split).  The producer
// streams A tiles (ROWS x 128, 3-D tensor map over (col-in-rank-slice, rank slice, row)) and
// the matching X tile (d x 128, contiguous in the tile layout) into an mbarrier ring with an
// L2 evict-first policy on A and evict-last on X.  Each consumer warp owns RT rows (= whole
// nodes); lane l owns columns 4l..4l+3 of every tile and keeps RT x d fp32 accumulators in
// registers, so every X value read from smem is reused RT times and A is read from smem once
// with conflict-free 128-bit loads.  At the end of a panel the warp reduces its accumulators
// with shuffles and runs the per-node epilogue entry-parallel in warp-private smem; no B is
// ever written to HBM.  fp64 partials for the objective / Gram matrices are reduced
// deterministically (fixed order, last-CTA pattern).
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
  static constexpr int SCR_BYTES = SCR_T_BYTES + kWarps * 2 * DD * 8 + kWarps * 2 * 8 + kWarps * NPART * 8 + 64;
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

// Sum nslots partial slots [nslots][NPART] into out[NPART] (consumer warps).  Warp w takes
// entries w, w + kWarps, ...; lane j sums slots j, j + 32, ... in order (loads issued 8 at a
// time: independent L2 round trips), then a fixed butterfly — deterministic.
template <int NPART>
__device__ __forceinline__ void reduce_slots(const double *slots, int nslots, double *out, int warp, int lane) {
  for (int i = warp; i < NPART; i += kWarps) {
    double v = 0.0;
    for (int b0 = lane; b0 < nslots; b0 += 32 * 8) {
      double q[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int b = b0 + 32 * j;
        q[j] = b < nslots ? __ldcg(slots + (int64_t)b * NPART + i) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) v += q[j];
    }
    v = warp_sum(v);
    if (lane == 0) out[i] = v;
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


// Stream-K schedule: the panels x tiles steps are cut into gridDim.x equal contiguous ranges.
__device__ __forceinline__ int64_t sk_bound(int64_t W, int G, int b) { return W * b / G; }
// CTA whose range contains step s: max b with sk_bound(b) <= s.
__device__ __forceinline__ int sk_owner(int64_t s, int64_t W, int G) { return (int)(((s + 1) * G + W - 1) / W - 1); }
// Column-tile order within a panel: this rank's own X slice first (ready earliest under P > 1).
__device__ __forceinline__ int tile_of_step(int t, const PanelParams &p) {
  const int tpr = (int)p.tiles_per_rank;
  const int g = t / tpr;
  return ((g + p.rank) % p.world) * tpr + (t - g * tpr);
}

template <typename T, int D, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    panel_kernel(const __grid_constant__ CUtensorMap tmA, const PanelParams p) {
  using C = PanelCfg<T, D>;
  using V = typename Vec4<T>::type;
  extern __shared__ uint8_t smem_raw[];
  // align to 1 KB by offsetting the shared array itself (keeps the shared address space, so
  // every smem access below compiles to LDS/STS rather than generic LD/ST)
  uint8_t *smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *empty = full + 8;
  T *scr_all = reinterpret_cast<T *>(smem + C::STAGES * C::STAGE_BYTES + C::BAR_BYTES);
  double *gram_all = reinterpret_cast<double *>(reinterpret_cast<uint8_t *>(scr_all) + C::SCR_T_BYTES);
  double *red = gram_all + kWarps * 2 * C::DD;       // [kWarps][2]
  double *xred = red + kWarps * 2;                   // [kWarps][NPART] cut-panel pre-reduction
  int *flag = reinterpret_cast<int *>(xred + kWarps * C::NPART);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // ------------------------------------------------------------------ producer warp
  if (warp == kWarps) {
    if (lane == 0) {
      prefetch_tmap(&tmA);
      const uint64_t pol_a = p.a_keep > 0.f ? policy_keep_fraction(p.a_keep) : policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      const int64_t s_end = sk_bound(p.steps, gridDim.x, blockIdx.x + 1);
      for (int it = 0; it < p.iters; ++it) {
        const T *Xin = static_cast<const T *>((it & 1) ? p.Xout : p.X);
        bool ready = it == 0;
        unsigned long long *ts = p.ts ? p.ts + ((int64_t)it * gridDim.x + blockIdx.x) * kTsSlots : nullptr;
        if (ts) ts[0] = globaltimer();
        for (int64_t st = sk_bound(p.steps, gridDim.x, blockIdx.x); st < s_end; ++st) {
          const int panel = (int)(st / p.total_tiles), t = (int)(st - (int64_t)panel * p.total_tiles);
          const int tt = tile_of_step(t, p);
          const int g = tt / (int)p.tiles_per_rank, jt = tt - g * (int)p.tiles_per_rank;
          mbar_wait(&empty[stage], phase ^ 1u);
          uint8_t *sb = smem + stage * C::STAGE_BYTES;
          mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          tma_load_3d(sb, &tmA, &full[stage], jt * kColTile, g, panel * C::ROWS, pol_a);
          if (!ready) {
            // A of iteration `it` is already in flight; X^it needs every CTA's epilogues of it-1
            const unsigned target = (unsigned)it * gridDim.x;
            unsigned spins = 0;
            while (ld_acquire_gpu(p.iter_cnt) < target) {
              __nanosleep(64);
              if (++spins > (1u << 26)) { atomicOr(p.err, kErrTimeout); break; }
            }
            fence_proxy_async_global();
            ready = true;
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
  double *gram1 = gram_all + warp * 2 * C::DD;
  double *gram2 = gram1 + C::DD;
#pragma unroll
  for (int m = 0; m < C::DDL; ++m) {
    const int e = lane + 32 * m;
    if (e < C::DD) { gram1[e] = 0.0; gram2[e] = 0.0; }
  }
  double s_own = 0.0, xb = 0.0;     // sum_i ||X_i^T X_i||^2, <X, B>
  float ns_region = 0.f;
  int err = 0;

  // Objective / Gram partials.  A panel whose tiles all lie in this CTA's stream-K range is
  // finished here by construction (static) and accumulates into the per-CTA running sums; a
  // panel cut by a CTA boundary is finished by whichever covering CTA arrives last, so its
  // contribution goes to a per-(panel, warp) slot and is summed later in a fixed order
  // (bitwise-deterministic results).
  double *part_base = p.cta_part;   // this iteration's partial slots (see part_iters)
  auto commit = [&](bool split_panel, int panel, const double *g1, const double *g2, double so, double xs) {
    if (!split_panel) {
#pragma unroll
      for (int m = 0; m < C::DDL; ++m) {
        const int e = lane + 32 * m;
        if (e < C::DD) { gram1[e] += g1[m]; gram2[e] += g2[m]; }
      }
      s_own += so;
      xb += xs;
      return;
    }
    // all consumer warps finish the same cut panel together: pre-reduce across warps in smem
    // (fixed warp order), one global slot per cut panel, indexed by the first CTA whose range
    // starts inside it.
    so = warp_sum(so);
    xs = warp_sum(xs);
    double *xw = xred + warp * C::NPART;
#pragma unroll
    for (int m = 0; m < C::DDL; ++m) {
      const int e = lane + 32 * m;
      if (e < C::DD) { xw[e] = g1[m]; xw[C::DD + e] = g2[m]; }
    }
    if (lane == 0) { xw[2 * C::DD] = so; xw[2 * C::DD + 1] = xs; }
    named_bar_sync(1, kWarps * 32);
    const int slot_cta = sk_owner((int64_t)panel * p.total_tiles, p.steps, gridDim.x) + 1;
    double *slot = part_base + ((int64_t)gridDim.x + slot_cta) * C::NPART;
    for (int i = threadIdx.x; i < C::NPART; i += kWarps * 32) {
      double v = 0.0;
      for (int w = 0; w < kWarps; ++w) v += xred[w * C::NPART + i];
      __stcg(slot + i, v);
    }
    named_bar_sync(1, kWarps * 32);
  };

  int stage = 0;
  uint32_t phase = 0;
  for (int it = 0; it < p.iters; ++it) {
  PanelParams pt = p;                 // per-iteration view: X^it in, X^{it+1} out, result slot it
  pt.X = (it & 1) ? p.Xout : p.X;
  pt.Xout = (it & 1) ? const_cast<void *>(p.X) : p.Xout;
  pt.result = p.result + (int64_t)it * C::NPART;
  const bool deferred = p.part_iters != nullptr && p.iters > 1;
  if (deferred) part_base = p.part_iters + (int64_t)it * 2 * gridDim.x * C::NPART;
  const T *Xg = static_cast<const T *>(pt.X);
  unsigned long long *cts = (p.ts && threadIdx.x == 0) ? p.ts + ((int64_t)it * gridDim.x + blockIdx.x) * kTsSlots : nullptr;
  bool first_stage = true;
  if (it > 0) {
#pragma unroll
    for (int m = 0; m < C::DDL; ++m) {
      const int e = lane + 32 * m;
      if (e < C::DD) { gram1[e] = 0.0; gram2[e] = 0.0; }
    }
    s_own = 0.0;
    xb = 0.0;
  }
  const int64_t my_s0 = sk_bound(p.steps, gridDim.x, blockIdx.x);
  const int64_t my_s1 = sk_bound(p.steps, gridDim.x, blockIdx.x + 1);
  const int first_panel = (int)(my_s0 / p.total_tiles);
  for (int64_t st = my_s0; st < my_s1;) {
    const int panel = (int)(st / p.total_tiles);
    const int t0 = (int)(st - (int64_t)panel * p.total_tiles);
    const int64_t t1l = t0 + (my_s1 - st);
    const int t1 = t1l < p.total_tiles ? (int)t1l : p.total_tiles;
    st += t1 - t0;
    const bool split_panel = !(t0 == 0 && t1 == p.total_tiles);
    const int64_t node_base = (int64_t)panel * C::NODES + warp * C::NPW;   // local node of q = 0
    const int64_t rem = p.n_local - node_base;
    const int nvalid = rem <= 0 ? 0 : (rem < C::NPW ? (int)rem : C::NPW);
    // X_i of this warp's nodes for the epilogue, in flight during the stream.  Issued after the
    // segment's first stage has landed: X^it is only guaranteed complete (all CTAs' epilogues
    // of it-1) once the producer passed the grid barrier and that stage's barrier completed
    // (writers' release -> producer acquire -> mbarrier arrive/wait).  The loop's own wait on
    // this phase then returns at once.
    mbar_wait(&full[stage], phase);
    T xpre[C::EPL];
    epi_load_x<T, D, C::NPW>(pt, Xg, lane, node_base, nvalid, xpre);

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
        mbar_wait(&full[stage], phase);
        if (cts && first_stage) { cts[2] = globaltimer(); first_stage = false; }
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
        mbar_wait(&full[stage], phase);
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

    if (cts) cts[5] = globaltimer();   // streaming of this segment done
    // ---- reduce the lane-partial sums: every lane ends with the full B rows of the warp
#pragma unroll
    for (int r = 0; r < C::RT; ++r)
#pragma unroll
      for (int k = 0; k < D; ++k) acc[r][k] = warp_sum(acc[r][k]);
    if (cts) cts[7] = globaltimer();   // lane partials reduced

    if (split_panel) {
      // partial B of this segment -> slot (CTA, first|last segment); the last covering CTA
      // to arrive sums all segments in CTA order and runs the epilogue.
      const int which = (panel == first_panel) ? 0 : 1;
      T *bp = static_cast<T *>(p.Bpart) + (((int64_t)blockIdx.x * 2 + which) * kWarps + warp) * C::EP;
      lane0_store_rows<T, C::RT, D, true>(bp, acc, lane);
      const int c_lo = sk_owner((int64_t)panel * p.total_tiles, p.steps, gridDim.x);
      const int c_hi = sk_owner((int64_t)(panel + 1) * p.total_tiles - 1, p.steps, gridDim.x);
      // release/acquire through ONE thread: the CTA barrier orders every consumer's stores
      // before thread 0's (cumulative) fence + arrival; an acquiring fence by thread 0 then the
      // barrier orders the partial reads after it.  (A fence in every thread serialises: ~4 us.)
      named_bar_sync(1, kWarps * 32);
      if (cts) cts[8] = globaltimer();   // partial stored
      if (threadIdx.x == 0) {
        fence_acq_rel_gpu();
        const unsigned prev = atomicAdd(&p.panel_cnt[panel], 1u);
        const int is_last = (prev == (unsigned)(c_hi - c_lo));
        if (is_last) {
          fence_acq_rel_gpu();
          p.panel_cnt[panel] = 0u;   // ready for the next launch
        }
        *flag = is_last;
      }
      named_bar_sync(1, kWarps * 32);
      const int last = *flag;
      if (cts) cts[9] = globaltimer();   // arrival counted
      named_bar_sync(1, kWarps * 32);   // everyone read flag before it is rewritten
      if (!last) continue;
      // Sum the covering CTAs' partials in CTA order.  A covering CTA cb > c_lo starts inside
      // this panel (slot 0); c_lo used slot 1 iff it started in an earlier panel.  Loads are
      // issued 4 CTAs x EPL entries at a time (independent L2 round trips), summed in order.
      const int w2_lo = sk_bound(p.steps, gridDim.x, c_lo) < (int64_t)panel * p.total_tiles ? 1 : 0;
      const T *bpr = static_cast<const T *>(p.Bpart) + (int64_t)warp * C::EP;
      T v[C::EPL];
#pragma unroll
      for (int m = 0; m < C::EPL; ++m) v[m] = T(0);
      for (int cb0 = c_lo; cb0 <= c_hi; cb0 += 4) {
        T part[4][C::EPL];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int cb = cb0 + j;
          const int w2 = cb == c_lo ? w2_lo : 0;
          const T *src = bpr + ((int64_t)cb * 2 + w2) * kWarps * C::EP;
#pragma unroll
          for (int m = 0; m < C::EPL; ++m) {
            const int e = lane + 32 * m;
            part[j][m] = (cb <= c_hi && e < C::E) ? __ldcg(src + e) : T(0);
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
    node_epilogue<T, D, C::NPW, MODE, true>(pt, Xg, lane, node_base, nvalid, sX, sG, sH, sS, sM, g1s, g2s, so, xs,
                                            ns_region, err, xpre);
    commit(split_panel, panel, g1s, g2s, so, xs);
    __syncwarp();
  }

  // ------------------------------------------------------------------ CTA + grid reduction
  if (cts) cts[3] = globaltimer();   // all own segments + epilogues done
  if (err) atomicOr(p.err, err);
  if (MODE == kModeRgs || MODE == kModeGpm) {
    float mx = ns_region;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0 && mx > 0.f) atomicMax(p.ns_region, __float_as_uint(mx));
  }
  s_own = warp_sum(s_own);
  xb = warp_sum(xb);
  if (lane == 0) { red[warp * 2] = s_own; red[warp * 2 + 1] = xb; }
  named_bar_sync(1, kWarps * 32);
  double *cp = part_base + (int64_t)blockIdx.x * C::NPART;
  for (int i = threadIdx.x; i < C::NPART; i += kWarps * 32) {
    double v = 0.0;
    if (i < 2 * C::DD) {
      for (int w = 0; w < kWarps; ++w) v += gram_all[w * 2 * C::DD + i];
    } else {
      for (int w = 0; w < kWarps; ++w) v += red[w * 2 + (i - 2 * C::DD)];
    }
    __stcg(cp + i, v);
  }
  if (!deferred) {
    named_bar_sync(1, kWarps * 32);
    if (threadIdx.x == 0) {
      fence_acq_rel_gpu();
      const int is_last = (atomicAdd(p.done_cnt, 1u) == gridDim.x - 1);
      if (is_last) fence_acq_rel_gpu();
      *flag = is_last;
    }
    named_bar_sync(1, kWarps * 32);
    if (*flag) {
      reduce_slots<C::NPART>(p.cta_part, 2 * (int)gridDim.x, pt.result, warp, lane);
      if (threadIdx.x == 0) *p.done_cnt = 0u;
    }
  }
  if (cts) cts[4] = globaltimer();   // end-of-iteration reduction done
  if (p.iters > 1) {   // grid barrier: this CTA's share of X^{it+1} (and partial slots) is done
    named_bar_sync(1, kWarps * 32);
    if (threadIdx.x == 0) {
      fence_acq_rel_gpu();
      atomicAdd(p.iter_cnt, 1u);
    }
  }
  }  // iterations

  if (p.part_iters != nullptr && p.iters > 1) {
    // deferred objective reduction: once every CTA has arrived after the last iteration, CTA b
    // reduces iterations b, b + G, ... (same fixed slot order as the per-iteration path).
    if (threadIdx.x == 0) {
      const unsigned target = (unsigned)p.iters * gridDim.x;
      unsigned spins = 0;
      while (ld_acquire_gpu(p.iter_cnt) < target) {
        __nanosleep(64);
        if (++spins > (1u << 26)) { atomicOr(p.err, kErrTimeout); break; }
      }
    }
    named_bar_sync(1, kWarps * 32);
    for (int it = blockIdx.x; it < p.iters; it += gridDim.x)
      reduce_slots<C::NPART>(p.part_iters + (int64_t)it * 2 * gridDim.x * C::NPART, 2 * (int)gridDim.x,
                             p.result + (int64_t)it * C::NPART, warp, lane);
  }
}

// ------------------------------------------------------------------ host-side launchers
template <typename T, int D, int MODE>
static cudaError_t launch_impl(const CUtensorMap *tm, const PanelParams &p, int grid, cudaStream_t s) {
  using C = PanelCfg<T, D>;
  auto kern = panel_kernel<T, D, MODE>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
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
  return PanelShape{C::ROWS, C::NODES, C::STAGES, C::SMEM, C::NPART, kThreads};
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
