// sym.cu — symmetric half-storage variant of the A.X pass.
//
// A is symmetric (PAPER.md:227 "A = ZZ^T + sigma W", W_ji = W_ij^T, :63), so B = A X can be
// formed from the upper half only: each stored element A[r][c] of row panel p (rows
// [pR, pR+R)) with c >= pR contributes A[r][c] X[c] to B[r] (row direction) and, for
// c >= pR + R, A[r][c] X[r] to B[c] (column direction, the mirrored element A[c][r]).  Every
// product is counted once: rows of panel p take columns c >= pR from their own row direction
// and columns c < pR from the column direction of the panel that owns row c.  HBM bytes per
// pass halve; FMAs per byte double (d flop/B: still under the FFMA2 roofline for d <= 6).
//
// Kernel 1 (sym_block_kernel): persistent CTAs take blocks (row group I of GP panels x column
// group J of GT tiles) of the upper triangle from an atomic queue (largest first).  A TMA
// producer warp streams (panel, tile) stages exactly like the dense kernel and publishes the
// stage's (I, J, p, t, flags) in smem.  Consumer warp w owns RT rows: the row direction
// accumulates in registers over the block's tiles of a panel and is written once per
// (panel, J) to rowpart[J]; the column direction (4 columns x d per lane, summed over the
// warp's rows in registers) is added into a warp-private smem slice (no atomics), and the 7
// slices are summed once per block into colpart[I].  Every partial has a fixed slot, so the
// result does not depend on which CTA ran which block (bitwise deterministic).
// Kernel 2 (sym_final_kernel): per node, B_i = sum_J rowpart + sum_I colpart in a fixed order,
// then the same per-node epilogue as the dense kernel (epilogue.cuh), fused objective partials.
#include <cuda.h>

#include <type_traits>

#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace nsrgs {

template <int D>
struct SymCfg {
  static_assert(D >= 2 && D <= 6, "symmetric storage: d in [2, 6]");
  static constexpr int RT = (D == 2 ? 12 : D == 3 ? 12 : D == 4 ? 12 : D == 5 ? 10 : 12);  // = dense fp32
  static constexpr int NPW = RT / D;
  static constexpr int ROWS = RT * kWarps;
  static constexpr int NODES = ROWS / D;
  static constexpr int KP = D / 2;                    // component pairs (2kp, 2kp+1)
  static constexpr bool ODD = (D & 1) != 0;          // last component on column pairs
  static constexpr int GT = D >= 6 ? 4 : kSymTilesPerBlock;   // column tiles per block (slices: 7 x GT x d x 128 floats)
  static constexpr int A_BYTES = ROWS * kColTile * 4;
  static constexpr int X_BYTES = D * kColTile * 4;
  static constexpr int STAGE_BYTES = A_BYTES + X_BYTES;
  static constexpr int SLICE_FLOATS = GT * D * kColTile;          // per warp: GT tiles in the X tile layout
  static constexpr int SLICE_BYTES = kWarps * SLICE_FLOATS * 4;
  static constexpr int META_BYTES = 8 * 32;
  static constexpr int BUDGET = 227 * 1024;   // sm_100 max dynamic smem per block
  static constexpr int FIXED = 1024 + 128 + META_BYTES + SLICE_BYTES + 64;
  static constexpr int STAGES_RAW = (BUDGET - FIXED) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : STAGES_RAW;
  static_assert(STAGES >= 2, "need a double-buffered ring");
  static constexpr int SMEM = FIXED + STAGES * STAGE_BYTES;
};

struct SymMeta {
  int I, J, p, t, flags, pad0, pad1, pad2;
};
constexpr int kFirstP = 1, kLastP = 2, kLastBlock = 4;

__device__ __forceinline__ uint64_t ffma2s(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t add2s(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint64_t bcast2(float v) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(v));
  return r;
}
__device__ __forceinline__ void split2(uint64_t v, float &lo, float &hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    sym_block_kernel(const __grid_constant__ CUtensorMap tmA, const SymParams sp) {
  using C = SymCfg<D>;
  extern __shared__ uint8_t smem_raw[];
  // align to 1 KB by offsetting the shared array itself (keeps the shared address space, so
  // every smem access below compiles to LDS/STS rather than generic LD/ST)
  uint8_t *smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t *empty = full + 8;
  SymMeta *meta = reinterpret_cast<SymMeta *>(smem + C::STAGES * C::STAGE_BYTES + 128);
  float *slices = reinterpret_cast<float *>(smem + C::STAGES * C::STAGE_BYTES + 128 + C::META_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const float *Xg = static_cast<const float *>(sp.e.X);
  const int64_t N = sp.N;

  // ------------------------------------------------------------------ producer warp
  if (warp == kWarps) {
    if (lane == 0) {
      prefetch_tmap(&tmA);
      const uint64_t pol_a = sp.e.a_keep > 0.f ? policy_keep_fraction(sp.e.a_keep) : policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (;;) {
        const int idx = (int)atomicAdd(sp.sched_cnt, 1u);
        if (idx >= sp.nblocks) {
          mbar_wait(&empty[stage], phase ^ 1u);
          meta[stage].I = -1;
          mbar_arrive(&full[stage]);
          break;
        }
        const int4 b = sp.blocks[idx];   // (I, J, p_first, p_last)
        for (int pp = b.z; pp <= b.w; ++pp) {
          const int t0p = (int)(((int64_t)pp * C::ROWS) / kColTile);
          const int tlo = max(b.y * C::GT, t0p), thi = min((b.y + 1) * C::GT, sp.nt);
          for (int t = tlo; t < thi; ++t) {
            mbar_wait(&empty[stage], phase ^ 1u);
            SymMeta &m = meta[stage];
            m.I = b.x;
            m.J = b.y;
            m.p = pp;
            m.t = t;
            m.flags = (t == tlo ? kFirstP : 0) | (t == thi - 1 ? kLastP : 0) |
                      (pp == b.w && t == thi - 1 ? kLastBlock : 0);
            uint8_t *sb = smem + stage * C::STAGE_BYTES;
            mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_3d(sb, &tmA, &full[stage], t * kColTile, 0, pp * C::ROWS, pol_a);
            bulk_load(sb + C::A_BYTES, Xg + (int64_t)t * D * kColTile, C::X_BYTES, &full[stage], pol_x);
            if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }
          }
        }
      }
    }
    return;
  }

  // ------------------------------------------------------------------ consumer warps
  // Slice = GT column tiles in the X tile layout (pairs interleaved, odd d's last component
  // contiguous); this warp only touches its own slice until the end-of-block reduction.
  float *myslice = slices + warp * C::SLICE_FLOATS;
  auto zero_slice = [&]() {
#pragma unroll
    for (int g = 0; g < C::GT; ++g) {
#pragma unroll
      for (int kp = 0; kp < C::KP; ++kp) {
        float *b = myslice + (g * D + 2 * kp) * kColTile;
        *reinterpret_cast<float4 *>(b + 4 * lane) = make_float4(0.f, 0.f, 0.f, 0.f);
        *reinterpret_cast<float4 *>(b + kColTile + 4 * lane) = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      if constexpr (C::ODD) *reinterpret_cast<float4 *>(myslice + (g * D + D - 1) * kColTile + 4 * lane) =
          make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncwarp();   // the last component's entries are zeroed by other lanes than their owners
  };
  zero_slice();

  constexpr int KL = C::ODD ? 1 : 0;
  uint64_t acc2[C::RT][C::KP + KL];   // row direction: pairs (+ last component's column pair)
  uint64_t xr[C::RT][C::KP];          // X of this warp's rows, component pairs (column direction)
  float xl[C::RT];                    // ... and the last component for odd d
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    mbar_wait(&full[stage], phase);
    const SymMeta m = meta[stage];
    if (m.I < 0) break;
    const int64_t row_lo = (int64_t)m.p * C::ROWS;        // panel start row
    const int64_t wrow0 = row_lo + warp * C::RT;          // this warp's first row
    if (m.flags & kFirstP) {
      // X rows of this warp (column direction) from the tile layout, 32-bit index arithmetic
      // (N d < 2^31 at every supported size); bounds only in the last panel (uniform branch)
      const int wr0 = (int)wrow0;
      auto load_rows = [&](auto guarded) {
        constexpr bool G = decltype(guarded)::value;
#pragma unroll
        for (int r = 0; r < C::RT; ++r) {
          const int row = wr0 + r;
          const bool ok = !G || row < (int)N;
          const int tb = (row >> 7) * (D * kColTile), o = row & 127;
          const unsigned long long *xp2 = reinterpret_cast<const unsigned long long *>(Xg + tb) + o;
#pragma unroll
          for (int kp = 0; kp < C::KP + KL; ++kp) acc2[r][kp] = 0ull;
#pragma unroll
          for (int kp = 0; kp < C::KP; ++kp) xr[r][kp] = ok ? __ldg(xp2 + kp * kColTile) : 0ull;
          if constexpr (C::ODD) xl[r] = ok ? __ldg(Xg + tb + (D - 1) * kColTile + o) : 0.f;
        }
      };
      if (wr0 + C::RT <= (int)N) load_rows(std::integral_constant<bool, false>{});
      else load_rows(std::integral_constant<bool, true>{});
    }
    const int64_t col0 = (int64_t)m.t * kColTile;
    const float *As = reinterpret_cast<const float *>(smem + stage * C::STAGE_BYTES) + (warp * C::RT) * kColTile + 2 * lane;
    const float *Xt = reinterpret_cast<const float *>(smem + stage * C::STAGE_BYTES + C::A_BYTES);
    const float *Xs = Xt + 4 * lane;
    uint64_t xp[C::KP + KL][4];
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
    uint64_t colc[4][C::KP];
    uint64_t colL[2] = {0ull, 0ull};   // odd d: last component, column pairs (2l, 2l+1), (64+2l, 65+2l)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int kp = 0; kp < C::KP; ++kp) colc[j][kp] = 0ull;
    // Tiles that start past this panel's row block need no masks (all but 1-2 per panel); near
    // the diagonal the row direction keeps c >= row_lo and the column direction c >= row_lo + ROWS.
    auto tile_pass = [&](auto masked) {
      constexpr bool MASK = decltype(masked)::value;
      float mr[4], mc[4];
      if constexpr (MASK) {
        const int64_t cj[4] = {col0 + 2 * lane, col0 + 2 * lane + 1, col0 + 64 + 2 * lane, col0 + 65 + 2 * lane};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          mr[j] = cj[j] >= row_lo ? 1.f : 0.f;
          mc[j] = cj[j] >= row_lo + C::ROWS ? 1.f : 0.f;
        }
      }
#pragma unroll
      for (int r = 0; r < C::RT; ++r) {
        const float2 a0 = *reinterpret_cast<const float2 *>(As + r * kColTile);
        const float2 a1 = *reinterpret_cast<const float2 *>(As + r * kColTile + 64);
        float ar[4] = {a0.x, a0.y, a1.x, a1.y};
        float ac[4] = {a0.x, a0.y, a1.x, a1.y};
        if constexpr (MASK) {
#pragma unroll
          for (int j = 0; j < 4; ++j) { ar[j] *= mr[j]; ac[j] *= mc[j]; }
        }
        // interleave independent chains: consecutive FFMA2s update different accumulators
#pragma unroll
        for (int j = 0; j < 4; ++j) {
#pragma unroll
          for (int kp = 0; kp < C::KP; ++kp) {
            acc2[r][kp] = ffma2s(xp[kp][j], bcast2(ar[j]), acc2[r][kp]);
            colc[j][kp] = ffma2s(xr[r][kp], bcast2(ac[j]), colc[j][kp]);
          }
        }
        if constexpr (C::ODD) {
          uint64_t ra0, ra1, ca0, ca1;
          asm("mov.b64 %0, {%1, %2};" : "=l"(ra0) : "f"(ar[0]), "f"(ar[1]));
          asm("mov.b64 %0, {%1, %2};" : "=l"(ra1) : "f"(ar[2]), "f"(ar[3]));
          asm("mov.b64 %0, {%1, %2};" : "=l"(ca0) : "f"(ac[0]), "f"(ac[1]));
          asm("mov.b64 %0, {%1, %2};" : "=l"(ca1) : "f"(ac[2]), "f"(ac[3]));
          acc2[r][C::KP] = ffma2s(ra0, xp[C::KP][0], acc2[r][C::KP]);
          acc2[r][C::KP] = ffma2s(ra1, xp[C::KP][1], acc2[r][C::KP]);
          colL[0] = ffma2s(ca0, bcast2(xl[r]), colL[0]);
          colL[1] = ffma2s(ca1, bcast2(xl[r]), colL[1]);
        }
      }
    };
    if (col0 >= row_lo + C::ROWS) tile_pass(std::integral_constant<bool, false>{});
    else tile_pass(std::integral_constant<bool, true>{});
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == C::STAGES) { stage = 0; phase ^= 1u; }

    // column direction -> this warp's slice (thread-exclusive entries, no atomics)
    {
      const int g = m.t - m.J * C::GT;
      const uint32_t tb = smem_u32(myslice) + (uint32_t)(g * D * kColTile * 4);
#pragma unroll
      for (int kp = 0; kp < C::KP; ++kp) {
        const uint32_t a0 = tb + (uint32_t)((2 * kp * kColTile + 4 * lane) * 4), a1 = a0 + kColTile * 4;
        uint64_t v0, v1, v2, v3;
        asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(v0), "=l"(v1) : "r"(a0) : "memory");
        asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(v2), "=l"(v3) : "r"(a1) : "memory");
        v0 = add2s(v0, colc[0][kp]);
        v1 = add2s(v1, colc[1][kp]);
        v2 = add2s(v2, colc[2][kp]);
        v3 = add2s(v3, colc[3][kp]);
        asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(a0), "l"(v0), "l"(v1) : "memory");
        asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(a1), "l"(v2), "l"(v3) : "memory");
      }
      if constexpr (C::ODD) {
        const uint32_t l0 = tb + (uint32_t)(((D - 1) * kColTile + 2 * lane) * 4), l1 = l0 + 64 * 4;
        uint64_t v0, v1;
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v0) : "r"(l0) : "memory");
        asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v1) : "r"(l1) : "memory");
        v0 = add2s(v0, colL[0]);
        v1 = add2s(v1, colL[1]);
        asm volatile("st.shared.b64 [%0], %1;" ::"r"(l0), "l"(v0) : "memory");
        asm volatile("st.shared.b64 [%0], %1;" ::"r"(l1), "l"(v1) : "memory");
      }
    }

    if (m.flags & kLastP) {   // row partials of (panel, J) -> rowpart[J][row][k]
      // reduce-scatter butterfly over the warp: value i = r*D + k; after 5 rounds lane l holds
      // the full sums of values [l*VP/32, (l+1)*VP/32) (VP = RT*D padded to a power of two).
      constexpr int V = C::RT * D;
      constexpr int VP = V <= 32 ? 32 : V <= 64 ? 64 : V <= 128 ? 128 : 256;
      float v[VP];
#pragma unroll
      for (int r = 0; r < C::RT; ++r) {
#pragma unroll
        for (int kp = 0; kp < C::KP; ++kp) split2(acc2[r][kp], v[r * D + 2 * kp], v[r * D + 2 * kp + 1]);
        if constexpr (C::ODD) {
          float lo, hi;
          split2(acc2[r][C::KP], lo, hi);
          v[r * D + D - 1] = lo + hi;
        }
      }
#pragma unroll
      for (int i = V; i < VP; ++i) v[i] = 0.f;
#pragma unroll
      for (int round = 0; round < 5; ++round) {
        const int off = 16 >> round;
        const int cnt = VP >> (round + 1);
        const bool upper = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < cnt; ++i) {
          const float send = upper ? v[i] : v[i + cnt];
          const float keep = upper ? v[i + cnt] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
      }
      float *rp = sp.rowpart + ((int64_t)m.J * N) * D;
#pragma unroll
      for (int j = 0; j < VP / 32; ++j) {
        const int i = lane * (VP / 32) + j;
        const int r = i / D, k = i % D;
        const int64_t row = wrow0 + r;
        if (i < V && row < N) rp[row * D + k] = v[j];
      }
    }
    if (m.flags & kLastBlock) {   // sum the 7 slices (fixed warp order) -> colpart[I][col][k]
      named_bar_sync(1, kWarps * 32);
      float *cp = sp.colpart + ((int64_t)m.I * N) * D;
      const int64_t cbase = (int64_t)m.J * C::GT * kColTile;
      for (int idx = threadIdx.x; idx < C::SLICE_FLOATS; idx += kWarps * 32) {
        const int gg = idx / (D * kColTile), rem = idx - gg * D * kColTile;
        int k, col;
        if (C::ODD && rem >= (D - 1) * kColTile) {
          k = D - 1;
          col = rem - (D - 1) * kColTile;
        } else {
          const int kp = rem / (2 * kColTile), w2 = rem - kp * 2 * kColTile;
          col = w2 >> 1;
          k = 2 * kp + (w2 & 1);
        }
        const int64_t c = cbase + (int64_t)gg * kColTile + col;
        if (c < N) {
          float v = 0.f;
          for (int w = 0; w < kWarps; ++w) v += slices[w * C::SLICE_FLOATS + idx];
          cp[c * D + k] = v;
        }
      }
      named_bar_sync(1, kWarps * 32);
      zero_slice();
    }
  }
}

// B_i from the partial slots (fixed order), then the per-node epilogue.  One warp = NPW nodes.
template <int D, int MODE>
__global__ void __launch_bounds__(256)
    sym_final_kernel(const SymParams sp) {
  using C = SymCfg<D>;
  constexpr int DD = D * D, E = C::NPW * DD, EPL = (E + 31) / 32, DDL = (DD + 31) / 32;
  constexpr int NPART = 2 * DD + 2, W = 8;
  __shared__ float scr[W][5 * E];
  __shared__ double gram[W][2 * DD];
  __shared__ double red[W][2];
  __shared__ int flag;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t N = sp.N;
  const int64_t node_base = ((int64_t)blockIdx.x * W + warp) * C::NPW;
  const int64_t rem = sp.e.n_local - node_base;
  const int nvalid = rem <= 0 ? 0 : (rem < C::NPW ? (int)rem : C::NPW);
  float *sX = scr[warp], *sG = sX + E, *sH = sG + E, *sS = sH + E, *sM = sS + E;
#pragma unroll
  for (int m = 0; m < EPL; ++m) {
    const int e = lane + 32 * m;
    if (e < E) {
      const int q = e / DD, a = (e / D) % D, k = e % D;
      float v = 0.f;
      if (q < nvalid) {
        const int64_t row = (node_base + q) * D + a;
        const int pnl = (int)(row / C::ROWS);
        const int J0 = (int)((((int64_t)pnl * C::ROWS) / kColTile) / C::GT);
        for (int J = J0; J < sp.nJ; ++J) v += __ldcg(sp.rowpart + ((int64_t)J * N + row) * D + k);
        const int Ic = pnl / sp.gp;
        for (int I = 0; I <= Ic; ++I) v += __ldcg(sp.colpart + ((int64_t)I * N + row) * D + k);
      }
      sG[e] = v;
    }
  }
  __syncwarp();
  double g1s[DDL], g2s[DDL], so = 0.0, xs = 0.0;
  float ns_region = 0.f;
  int err = 0;
  node_epilogue<float, D, C::NPW, MODE>(sp.e, static_cast<const float *>(sp.e.X), sp.e.Xout, lane, node_base, nvalid, sX, sG,
                                        sH, sS, sM, g1s, g2s, so, xs, ns_region, err);
  if (err) atomicOr(sp.e.err, err);
  {
    float mx = ns_region;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0 && mx > 0.f) atomicMax(sp.e.ns_region, __float_as_uint(mx));
  }
  so = warp_sum(so);
  xs = warp_sum(xs);
#pragma unroll
  for (int m = 0; m < DDL; ++m) {
    const int e2 = lane + 32 * m;
    if (e2 < DD) { gram[warp][e2] = g1s[m]; gram[warp][DD + e2] = g2s[m]; }
  }
  if (lane == 0) { red[warp][0] = so; red[warp][1] = xs; }
  __syncthreads();
  for (int i = threadIdx.x; i < NPART; i += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < W; ++w) v += i < 2 * DD ? gram[w][i] : red[w][i - 2 * DD];
    __stcg(sp.e.cta_part + (int64_t)blockIdx.x * NPART + i, v);
  }
  __syncthreads();
  if (threadIdx.x == 0) {   // one fence per CTA (bar.sync + cumulative fence), see panel.cu
    fence_acq_rel_gpu();
    const int is_last = (atomicAdd(sp.e.done_cnt, 1u) == gridDim.x - 1);
    if (is_last) fence_acq_rel_gpu();
    flag = is_last;
  }
  __syncthreads();
  if (flag) {
    for (int i = warp; i < NPART; i += W) {
      double v = 0.0;
      for (int b = lane; b < (int)gridDim.x; b += 32) v += __ldcg(sp.e.cta_part + (int64_t)b * NPART + i);
      v = warp_sum(v);
      if (lane == 0) sp.e.result[i] = v;
    }
    if (threadIdx.x == 0) {
      *sp.e.done_cnt = 0u;
      *sp.sched_cnt = 0u;   // block queue of the next sym_block_kernel launch (stream-ordered)
    }
  }
}

// ------------------------------------------------------------------ host side
template <int D>
static SymShape sym_shape_impl() {
  using C = SymCfg<D>;
  return SymShape{C::ROWS, C::NODES, C::STAGES, C::SMEM, C::GT, C::NPW, 8 * C::NPW};
}

template <int D>
static cudaError_t sym_launch_impl(const CUtensorMap *tm, const SymParams &sp, int grid, int mode, cudaStream_t s) {
  using C = SymCfg<D>;
  static bool attr[64] = {};
  {
    const cudaError_t e = set_smem_attr_once(reinterpret_cast<const void *>(sym_block_kernel<D>), C::SMEM, attr);
    if (e != cudaSuccess) return e;
  }
  sym_block_kernel<D><<<grid, kThreads, C::SMEM, s>>>(*tm, sp);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const unsigned fgrid = (unsigned)((sp.e.n_local + 8 * C::NPW - 1) / (8 * C::NPW));
  switch (mode) {
    case kModeRgs: sym_final_kernel<D, kModeRgs><<<fgrid, 256, 0, s>>>(sp); break;
    case kModeObjective: sym_final_kernel<D, kModeObjective><<<fgrid, 256, 0, s>>>(sp); break;
    case kModeProduct: sym_final_kernel<D, kModeProduct><<<fgrid, 256, 0, s>>>(sp); break;
    default: sym_final_kernel<D, kModeGpm><<<fgrid, 256, 0, s>>>(sp); break;
  }
  return cudaGetLastError();
}

cudaError_t sym_dispatch(int d, int mode, bool shape_only, SymShape *shape, const CUtensorMap *tm, const SymParams *sp,
                         int grid, cudaStream_t s) {
  switch (d) {
#define NSRGS_SYM_CASE(DV)                                              \
  case DV:                                                             \
    if (shape_only) { *shape = sym_shape_impl<DV>(); return cudaSuccess; } \
    return sym_launch_impl<DV>(tm, *sp, grid, mode, s);
    NSRGS_SYM_CASE(2)
    NSRGS_SYM_CASE(3)
    NSRGS_SYM_CASE(4)
    NSRGS_SYM_CASE(5)
    NSRGS_SYM_CASE(6)
#undef NSRGS_SYM_CASE
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace nsrgs
