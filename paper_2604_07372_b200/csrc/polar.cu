// polar.cu — X^0_i = sgn(Y_i) for the spectral initialisation (reading R6):
// the GPM branch of the shared per-node epilogue (Frobenius pre-scaling, Newton-Schulz to
// convergence, NSRGS_ERR_SINGULAR flag) applied to B_i := Y_i, warp-parallel in smem.
#include "common.cuh"
#include "epilogue.cuh"
#include "kernels.h"

namespace nsrgs {

template <typename T, int D>
struct PolarCfg {
  static constexpr int NPW = (D * D >= 32) ? 1 : 32 / (D * D);   // nodes per warp
  static constexpr int W = D * D >= 256 ? 2 : 4;                  // static smem <= 48 KB
  static constexpr int E = NPW * D * D;
};

template <typename T, int D>
__global__ void __launch_bounds__(128) polar_warp_kernel(const PanelParams p) {
  using C = PolarCfg<T, D>;
  constexpr int DDL = (D * D + 31) / 32;
  __shared__ T scr[C::W][5 * C::E];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t node_base = ((int64_t)blockIdx.x * C::W + warp) * C::NPW;   // global node = local here
  const int64_t rem = p.n_local - node_base;
  const int nvalid = rem <= 0 ? 0 : (rem < C::NPW ? (int)rem : C::NPW);
  T *sX = scr[warp], *sG = sX + C::E, *sH = sG + C::E, *sS = sH + C::E, *sM = sS + C::E;
  const T *Y = static_cast<const T *>(p.X);
  for (int e = lane; e < C::E; e += 32) {
    const int q = e / (D * D), a = (e / D) % D, b = e % D;
    sG[e] = q < nvalid ? Y[tile_index((node_base + q) * D + a, b, D, p.rows_local, p.tiles_per_rank)] : T(0);
  }
  __syncwarp();
  double g1s[DDL], g2s[DDL], so = 0.0, xs = 0.0;
  float nsr = 0.f;
  int err = 0;
  node_epilogue<T, D, C::NPW, kModeGpm>(p, Y, p.Xout, lane, node_base, nvalid, sX, sG, sH, sS, sM, g1s, g2s, so, xs, nsr, err);
  if (err) atomicOr(p.err, err);
}

template <typename T, int D>
static cudaError_t polar_launch(const PanelParams &p, cudaStream_t s) {
  using C = PolarCfg<T, D>;
  const int64_t per = (int64_t)C::W * C::NPW;
  polar_warp_kernel<T, D><<<(unsigned)((p.n_local + per - 1) / per), 32 * C::W, 0, s>>>(p);
  return cudaGetLastError();
}

// All n nodes on every rank (X is replicated): node0 = 0, n_local = n in the view passed here.
cudaError_t launch_polar(int dtype, int d, int64_t n, const void *Y, void *X, int64_t rows_local, int64_t tpr, int *err,
                         cudaStream_t s) {
  PanelParams p{};
  p.X = Y;
  p.Xout = X;
  p.err = err;
  p.n = n;
  p.n_local = n;
  p.node0 = 0;
  p.rows_local = rows_local;
  p.tiles_per_rank = tpr;
  p.iters = 1;
#define NSRGS_POLAR(DV)                                                                     \
  case DV:                                                                                 \
    return dtype == 0 ? polar_launch<float, DV>(p, s)                                      \
                      : (DV <= 6 ? polar_launch<double, (DV <= 6 ? DV : 2)>(p, s) : cudaErrorInvalidValue);
  switch (d) {
    NSRGS_POLAR(2) NSRGS_POLAR(3) NSRGS_POLAR(4) NSRGS_POLAR(5) NSRGS_POLAR(6) NSRGS_POLAR(7) NSRGS_POLAR(8)
    NSRGS_POLAR(9) NSRGS_POLAR(10) NSRGS_POLAR(11) NSRGS_POLAR(12) NSRGS_POLAR(13) NSRGS_POLAR(14)
    NSRGS_POLAR(15) NSRGS_POLAR(16) NSRGS_POLAR(20) NSRGS_POLAR(24)
    NSRGS_POLAR(25) NSRGS_POLAR(32)
    default: return cudaErrorInvalidValue;
  }
#undef NSRGS_POLAR
}

}  // namespace nsrgs
