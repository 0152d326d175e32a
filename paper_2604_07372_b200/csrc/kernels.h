// kernels.h — host-visible entry points of the device code (internal to libnsrgs.so).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace nsrgs {

enum PanelMode { kModeRgs = 0, kModeObjective = 1, kModeProduct = 2, kModeGpm = 3 };

struct PanelShape {
  int rows, nodes, stages, smem, npart, threads;
  int nw;   // consumer warps (the (panel, warp) epilogue unit count per panel)
};

// panel.cu: shape query (shape_only) or launch of the fused A.X + epilogue kernel.
cudaError_t panel_dispatch(int dtype, int d, int mode, bool shape_only, PanelShape *shape,
                           const CUtensorMap *tm, const PanelParams *p, int grid, cudaStream_t s);

cudaError_t launch_p2p_wait(const unsigned *xcnt, int world, unsigned target, int *err, cudaStream_t s);

// wide.cu: d > 10 (one node per warp, lane = component).
bool wide_supported(int d);
cudaError_t wide_dispatch(int d, int mode, bool shape_only, PanelShape *shape, const CUtensorMap *tm,
                          const PanelParams *p, int grid, cudaStream_t s, bool mma);
// wide_tc.cu: d > 10 on tcgen05 (3xTF32, TMEM accumulators, persistent stream-K grid).
// slot_floats: floats of one CTA's partial-row slot (Bpart = grid slots, ucnt = grid flags).
cudaError_t wide_tc_dispatch(int d, int mode, bool shape_only, PanelShape *shape, int *slot_floats,
                             const CUtensorMap *tm, const PanelParams *p, int grid, cudaStream_t s);

// sym.cu: symmetric half-storage pass (fp32, world == 1, d in [2, 6]).
struct SymShape {
  int rows, nodes, stages, smem, gt, npw, final_nodes_per_cta;
};
cudaError_t sym_dispatch(int d, int mode, bool shape_only, SymShape *shape, const CUtensorMap *tm, const SymParams *sp,
                         int grid, cudaStream_t s);

// bsr.cu: block-sparse storage (fp32, any supported d).
int bsr_xs_stride(int d, bool slab);
int bsr_grid(int d, int64_t n_local);
int bsr_slab_lg2g(int d, double p_eff);
cudaError_t bsr_dispatch(int d, int mode, const BsrParams *bp, int lg2g, const CUtensorMap *tmX, cudaStream_t s);
cudaError_t launch_bsr_pack_x(int d, const void *X, float *Xs, int64_t n, int64_t rows_local, int64_t tpr, bool slab,
                              cudaStream_t s);
cudaError_t launch_bsr_count(int64_t n, int64_t node0, int64_t n_local, uint64_t seed, double p_obs, int64_t *cnt,
                             int64_t *rowptr, cudaStream_t s);
cudaError_t launch_bsr_fill(int d, int64_t n, int64_t node0, int64_t n_local, uint64_t seed, double sigma, double p_obs,
                            const double *Z64, const int64_t *rowptr, int *col, float *vals, double *part,
                            cudaStream_t s);
cudaError_t launch_bsr_validate(const int64_t *rowptr, const int *col, int64_t n_local, int64_t nnzb, int64_t n,
                                int *bad, cudaStream_t s);
cudaError_t launch_bsr_sumsq(const float *vals, int64_t count, double *part, int *nblocks, cudaStream_t s);

// objective64.cu: F(X) with fp64 accumulation of <X, A X> (the nsrgs_solve stopping rule).
struct Obj64Args {
  const float *A;              // dense shard (NULL when block-sparse)
  int64_t lda;
  const int64_t *bsr_rowptr;   // block-sparse shard (NULL when dense)
  const int *bsr_col;
  const float *bsr_vals;
  int64_t n, n_local, node0;
  const float *Xs;             // row-major n d x d stack of X (all nodes)
  double *part_x;              // [grid_x] <X_loc, (A X)_loc> partials
  double *part_g;              // [grid_g][2 d^2 + 2] Gram partials
  int grid_x, grid_g, sm_count;
};
void obj64_grids(int64_t n_local, int d, bool bsr, int sm_count, int *grid_x, int *grid_g);
cudaError_t launch_obj64(int d, const Obj64Args &a, cudaStream_t s);

// aux.cu
cudaError_t launch_gen_Z(int dtype, int d, int64_t n, uint64_t seed, double *Z64, void *Zt, cudaStream_t s);
cudaError_t launch_gen_A(int dtype, int d, int64_t n, int64_t node0, int64_t n_local, uint64_t seed,
                         double sigma, double p_obs, const double *Z64, void *A, int64_t lda, double *part,
                         int *nblocks, cudaStream_t s);
cudaError_t launch_gen_Y0(int dtype, int d, int64_t n, uint64_t seed, void *Y, int64_t rows_local,
                          int64_t tiles_per_rank, cudaStream_t s);
cudaError_t launch_sumsq(int dtype, const void *A, int64_t rows, int64_t cols, int64_t lda, double *part,
                         int *nblocks, cudaStream_t s);
cudaError_t launch_reduce(const double *part, int nblocks, int width, double *out, cudaStream_t s);
cudaError_t launch_pack(int dtype, int d, int64_t n, const void *stack, void *tiled, int64_t rows_local,
                        int64_t tiles_per_rank, int unpack, cudaStream_t s);
cudaError_t launch_chol(int d, const double *res, double *MC, int *err, cudaStream_t s);
cudaError_t launch_scale(int dtype, int d, int64_t node0, int64_t n_local, const double *MC, void *W,
                         const void *Yold, int64_t rows_local, int64_t tiles_per_rank, double *part,
                         int *nblocks, cudaStream_t s);
cudaError_t launch_cheb_combine(int dtype, int d, int64_t node0, int64_t n_local, double alpha, double beta, void *W,
                                const void *Yprev, const void *Ycur, int64_t rows_local, int64_t tpr, double *part,
                                int *nblocks, cudaStream_t s);
cudaError_t launch_cheb_apply(int dtype, int d, int64_t node0, int64_t n_local, const double *MC, const void *Yin,
                              void *Yout, int64_t rows_local, int64_t tpr, cudaStream_t s);
cudaError_t launch_polar(int dtype, int d, int64_t n, const void *Y, void *X, int64_t rows_local,
                         int64_t tiles_per_rank, int *err, cudaStream_t s);
cudaError_t launch_objective_final(int d, int T, const double *res, int npart, const double *a_fro2,
                                   double *F, cudaStream_t s);
int metrics_blocks(int d, int64_t n);
cudaError_t launch_metrics(int dtype, int d, int64_t n, const void *X, const void *Z, int64_t rows_local,
                           int64_t tiles_per_rank, double *part, int *nblocks, cudaStream_t s);
cudaError_t launch_metrics_final(int d, int64_t n, const double *grams, double *out3, cudaStream_t s);

}  // namespace nsrgs
