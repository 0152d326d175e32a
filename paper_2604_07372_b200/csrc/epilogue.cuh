// epilogue.cuh — the per-node epilogue of one warp (NPW nodes), shared by the dense panel
// kernel (panel.cu) and the symmetric-storage finaliser (sym.cu).
//
// On entry sG holds B_i = sum_j A_ij X_j for the warp's nodes (entry e = (q*D + a)*D + b).
// Modes: RGS — G = (n-1)X - B, P = (G - X G^T X)/2, F = X - eta P, K Newton-Schulz steps
// (Algorithm 1 :172-182), X^{t+1} -> Xout; OBJECTIVE — partials only;
// GPM — X^{t+1} = sgn(B) by scaled NS; PRODUCT — W = B -> Xout and the Gram
// partials W^T W, Y^T W of the subspace sweep.  Objective / Gram partial
// contributions of the warp's nodes are returned per lane in g1s/g2s/so/xs.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace nsrgs {

template <typename T> __device__ __forceinline__ T tfma(T a, T b, T c) { return fma(a, b, c); }

template <typename T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// X_i entries of the warp's NPW nodes, entry e = lane + 32 m = (q, a, b) -> X_{node_base+q}[a][b],
// into registers (zero past nvalid).  Loaded from L2 (written by other CTAs).  The panel kernel
// issues this when a segment starts so the latency hides under the A stream.
template <typename T, int D, int NPW>
__device__ __forceinline__ void epi_load_x(const PanelParams &p, const T *Xg, int lane, int64_t node_base, int nvalid,
                                           T (&xv)[(NPW * D * D + 31) / 32]) {
  constexpr int DD = D * D, E = NPW * DD, EPL = (E + 31) / 32;
#pragma unroll
  for (int m = 0; m < EPL; ++m) {
    const int e = lane + 32 * m;
    const int q = e / DD, a = (e / D) % D, b = e % D;
    xv[m] = T(0);
    if (e < E && q < nvalid) {
      const int64_t c = (p.node0 + node_base + q) * D + a;
      xv[m] = __ldcg(Xg + tile_index(c, b, D, p.rows_local, p.tiles_per_rank));
    }
  }
}

// XPRE: the caller passes the epi_load_x registers in xpre (else they are loaded here).
// Xout: where X^{t+1} (RGS / GPM) or W (PRODUCT) goes (explicit: the panel kernel alternates
// buffers per iteration without copying its parameter block).
template <typename T, int D, int NPW, int MODE, bool XPRE = false>
__device__ __forceinline__ void node_epilogue(const PanelParams &p, const T *Xg, void *Xout, int lane, int64_t node_base,
                                              int nvalid, T *sX, T *sG, T *sH, T *sS, T *sM,
                                              double (&g1s)[(D * D + 31) / 32], double (&g2s)[(D * D + 31) / 32],
                                              double &so, double &xs, float &ns_region, int &err,
                                              const T *xpre = nullptr) {
  constexpr int DD = D * D;
  constexpr int E = NPW * DD;
  constexpr int EPL = (E + 31) / 32;
  constexpr int DDL = (DD + 31) / 32;
  const T coef = (T)p.coef, eta = (T)p.eta;
  {
    T xv[EPL];
    if constexpr (XPRE) {
#pragma unroll
      for (int m = 0; m < EPL; ++m) xv[m] = xpre[m];
    } else {
      epi_load_x<T, D, NPW>(p, Xg, lane, node_base, nvalid, xv);
    }
#pragma unroll
    for (int m = 0; m < EPL; ++m)
      if (lane + 32 * m < E) sX[lane + 32 * m] = xv[m];
  }
  __syncwarp();

  if constexpr (MODE == kModeProduct) {
    // W = A Y rows -> Xout; Gram partials W^T W and Y^T W (Cholesky-QR of the sweep).
    T *Wout = static_cast<T *>(Xout);
#pragma unroll
    for (int m = 0; m < EPL; ++m) {
      const int e = lane + 32 * m;
      if (e < E) {
        const int q = e / DD, a = (e / D) % D, b = e % D;
        if (q < nvalid) {
          const int64_t c = (p.node0 + node_base + q) * D + a;
          Wout[tile_index(c, b, D, p.rows_local, p.tiles_per_rank)] = sG[e];
        }
      }
    }
#pragma unroll
    for (int m = 0; m < DDL; ++m) {
      const int e2 = lane + 32 * m;
      double g1 = 0.0, g2 = 0.0;
      if (e2 < DD) {
        const int a = e2 / D, b = e2 % D;
        for (int q = 0; q < nvalid; ++q)
#pragma unroll
          for (int k = 0; k < D; ++k) {
            const double w_ka = (double)sG[(q * D + k) * D + a], w_kb = (double)sG[(q * D + k) * D + b];
            g1 += w_ka * w_kb;
            g2 += (double)sX[(q * D + k) * D + a] * w_kb;
          }
      }
      g1s[m] = g1;
      g2s[m] = g2;
    }
    so = 0.0;
    xs = 0.0;
    __syncwarp();
    return;
  } else {
    // <X, B> and the X Gram terms of the objective expansion.
    xs = 0.0;
    so = 0.0;
#pragma unroll
    for (int m = 0; m < EPL; ++m) {
      const int e = lane + 32 * m;
      if (e < E && e / DD < nvalid) xs += (double)sX[e] * (double)sG[e];
    }
#pragma unroll
    for (int m = 0; m < DDL; ++m) {
      const int e2 = lane + 32 * m;
      double g1 = 0.0;
      if (e2 < DD) {
        const int a = e2 / D, b = e2 % D;
        for (int q = 0; q < nvalid; ++q) {
          double v = 0.0;
#pragma unroll
          for (int k = 0; k < D; ++k)
            v += (double)sX[(q * D + k) * D + a] * (double)sX[(q * D + k) * D + b];
          g1 += v;
          so += v * v;
        }
      }
      g1s[m] = g1;
      g2s[m] = 0.0;
    }
    if constexpr (MODE == kModeObjective) {
      __syncwarp();
      return;
    }
    if constexpr (MODE == kModeGpm) {
      // GPM (comparison method): X_i <- sgn(B_i), B_i = sum_{j!=i} A_ij X_j, by
      // Newton-Schulz from S_0 = B_i / ||B_i||_F (singular values in (0, 1]) to convergence.
      T *inv = sM + E - NPW;   // scratch: per-node scale (sM is rewritten below)
      if constexpr (NPW == 1) {   // one node per warp (wide blocks): the d^2 sum over the lanes
        T f2 = T(0);
        for (int e2 = lane; e2 < DD; e2 += 32) f2 += sG[e2] * sG[e2];
        f2 = warp_sum(f2);
        if (lane == 0) inv[0] = f2 > T(0) ? T(1) / sqrt(f2) : T(0);
      } else if (lane < NPW) {
        T f2 = T(0);
        for (int e2 = 0; e2 < DD; ++e2) f2 += sG[lane * DD + e2] * sG[lane * DD + e2];
        inv[lane] = f2 > T(0) ? T(1) / sqrt(f2) : T(0);
      }
      __syncwarp();
#pragma unroll
      for (int m = 0; m < EPL; ++m) {
        const int e = lane + 32 * m;
        if (e < E) sS[e] = sG[e] * inv[e / DD];
      }
      __syncwarp();
      const T tol = sizeof(T) == 4 ? T(2e-5) * (D > 3 ? T(D) / T(3) : T(1)) : T(1e-13) * T(D);   // fp32 floor grows ~ d
      int polish = 2;
      bool conv = false;
      for (int it = 0; it < 100; ++it) {
#pragma unroll
        for (int m = 0; m < EPL; ++m) {
          const int e = lane + 32 * m;
          if (e < E) {
            const int q = e / DD, a = (e / D) % D, b = e % D;
            const T *Sq = sS + q * DD;
            T v = T(0);
#pragma unroll
            for (int k = 0; k < D; ++k) v = tfma(Sq[k * D + a], Sq[k * D + b], v);
            sM[e] = v;
          }
        }
        __syncwarp();
        bool ok = true;
        if constexpr (NPW == 1) {
          T dev = T(0);
          for (int e2 = lane; e2 < DD; e2 += 32) {
            const T dv = (e2 / D == e2 % D ? T(1) : T(0)) - sM[e2];
            dev += dv * dv;
          }
          dev = warp_sum(dev);
          ok = nvalid == 0 || sqrt(dev) <= tol;
        } else if (lane < nvalid) {
          T dev = T(0);
          for (int e2 = 0; e2 < DD; ++e2) {
            const T dv = (e2 / D == e2 % D ? T(1) : T(0)) - sM[lane * DD + e2];
            dev += dv * dv;
          }
          ok = sqrt(dev) <= tol;
        }
        if (__all_sync(0xffffffffu, ok)) {
          conv = true;
          if (polish-- == 0) break;
        }
        T snew[EPL];
#pragma unroll
        for (int m = 0; m < EPL; ++m) {
          const int e = lane + 32 * m;
          snew[m] = T(0);
          if (e < E) {
            const int q = e / DD, a = (e / D) % D, b = e % D;
            const T *Sq = sS + q * DD, *Mq = sM + q * DD;
            T v = T(0);
#pragma unroll
            for (int k = 0; k < D; ++k) v = tfma(Sq[a * D + k], Mq[k * D + b], v);
            snew[m] = T(1.5) * sS[e] - T(0.5) * v;
          }
        }
        __syncwarp();
#pragma unroll
        for (int m = 0; m < EPL; ++m) {
          const int e = lane + 32 * m;
          if (e < E) sS[e] = snew[m];
        }
        __syncwarp();
      }
      if (!conv && nvalid > 0) err |= kErrSingular;
    } else {
    // G = (n-1) X - B   (in place in sG)
#pragma unroll
    for (int m = 0; m < EPL; ++m) {
      const int e = lane + 32 * m;
      if (e < E) sG[e] = coef * sX[e] - sG[e];
    }
    __syncwarp();
    // H = G^T X
#pragma unroll
    for (int m = 0; m < EPL; ++m) {
      const int e = lane + 32 * m;
      if (e < E) {
        const int q = e / DD, a = (e / D) % D, b = e % D;
        const T *Gq = sG + q * DD, *Xq = sX + q * DD;
        T h = T(0);
#pragma unroll
        for (int k = 0; k < D; ++k) h = tfma(Gq[k * D + a], Xq[k * D + b], h);
        sH[e] = h;
      }
    }
    __syncwarp();
    // P = (G - X H)/2,  F = X - eta P
#pragma unroll
    for (int m = 0; m < EPL; ++m) {
      const int e = lane + 32 * m;
      if (e < E) {
        const int q = e / DD, a = (e / D) % D, b = e % D;
        const T *Hq = sH + q * DD, *Xq = sX + q * DD;
        T xh = T(0);
#pragma unroll
        for (int k = 0; k < D; ++k) xh = tfma(Xq[a * D + k], Hq[k * D + b], xh);
        const T P = T(0.5) * (sG[e] - xh);
        sS[e] = sX[e] - eta * P;
      }
    }
    __syncwarp();
    // Algorithm 1: K Newton-Schulz steps S <- 1/2 S (3I - S^T S) = 1.5 S - 0.5 S (S^T S)
    for (int it = 0; it < p.K; ++it) {
#pragma unroll
      for (int m = 0; m < EPL; ++m) {
        const int e = lane + 32 * m;
        if (e < E) {
          const int q = e / DD, a = (e / D) % D, b = e % D;
          const T *Sq = sS + q * DD;
          T v = T(0);
#pragma unroll
          for (int k = 0; k < D; ++k) v = tfma(Sq[k * D + a], Sq[k * D + b], v);
          sM[e] = v;
        }
      }
      __syncwarp();
      if constexpr (NPW == 1) {   // ||I - F^T F||_F of the warp's node (PAPER.md:465 eq:conclusion:sigma)
        if (it == 0) {
          float acc2 = 0.f;
          for (int e2 = lane; e2 < DD; e2 += 32) {
            const float dv = (float)((e2 / D == e2 % D ? T(1) : T(0)) - sM[e2]);
            acc2 += dv * dv;
          }
          acc2 = warp_sum(acc2);
          if (lane < nvalid) ns_region = fmaxf(ns_region, sqrtf(acc2));
        }
      } else if (it == 0 && lane < nvalid) {   // ... of node `lane`
        const T *Mq = sM + lane * DD;
        float acc2 = 0.f;
        for (int e2 = 0; e2 < DD; ++e2) {
          const float dv = (float)((e2 / D == e2 % D ? T(1) : T(0)) - Mq[e2]);
          acc2 += dv * dv;
        }
        ns_region = fmaxf(ns_region, sqrtf(acc2));
      }
      T snew[EPL];
#pragma unroll
      for (int m = 0; m < EPL; ++m) {
        const int e = lane + 32 * m;
        snew[m] = T(0);
        if (e < E) {
          const int q = e / DD, a = (e / D) % D, b = e % D;
          const T *Sq = sS + q * DD, *Mq = sM + q * DD;
          T v = T(0);
#pragma unroll
          for (int k = 0; k < D; ++k) v = tfma(Sq[a * D + k], Mq[k * D + b], v);
          snew[m] = T(1.5) * sS[e] - T(0.5) * v;
        }
      }
      __syncwarp();
#pragma unroll
      for (int m = 0; m < EPL; ++m) {
        const int e = lane + 32 * m;
        if (e < E) sS[e] = snew[m];
      }
      __syncwarp();
    }
    }  // MODE == kModeRgs
    // divergence guard: non-finite or ||S||_F > 10 sqrt(d)
    if constexpr (NPW == 1) {
      float f2 = 0.f;   // a threshold test at ||S||_F^2 = 100 d: fp32 lane sums suffice (NaN / Inf propagate)
      for (int e2 = lane; e2 < DD; e2 += 32) f2 += (float)sS[e2] * (float)sS[e2];
      f2 = warp_sum(f2);
      if (nvalid > 0 && !(f2 <= 100.f * D)) err |= kErrDivergence;
    } else if (lane < nvalid) {
      const T *Sq = sS + lane * DD;
      double f2 = 0.0;
      for (int e2 = 0; e2 < DD; ++e2) f2 += (double)Sq[e2] * (double)Sq[e2];
      if (!(f2 <= 100.0 * D)) err |= kErrDivergence;
    }
    T *Xo = static_cast<T *>(Xout);
#pragma unroll
    for (int m = 0; m < EPL; ++m) {
      const int e = lane + 32 * m;
      if (e < E) {
        const int q = e / DD, a = (e / D) % D, b = e % D;
        if (q < nvalid) {
          const int64_t c = (p.node0 + node_base + q) * D + a;
          const int64_t idx = tile_index(c, b, D, p.rows_local, p.tiles_per_rank);
          Xo[idx] = sS[e];
          if (p.p2p)   // fused exchange: the same rows into every peer's X^{t+1} (NVLink stores)
            for (int g = 0; g < p.world; ++g)
              if (g != p.rank) static_cast<T *>(p.peer_X[g])[idx] = sS[e];
        }
      }
    }
    __syncwarp();
  }
}

}  // namespace nsrgs
