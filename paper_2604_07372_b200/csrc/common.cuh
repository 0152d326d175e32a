// common.cuh — device helpers shared by the libnsrgs kernels (PTX wrappers for mbarrier,
// TMA / bulk copies, L2 policies; the Philox4x32-10 counter RNG; the X tile layout).
// Nothing here is shared with oracle/ (the oracle re-implements the generator in NumPy).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace nsrgs {

constexpr int kColTile = 128;      // X/A column tile (elements); one float4/double4 per lane
constexpr int kTsSlots = 16;   // debug timestamp slots per CTA per iteration
constexpr int kWarps = 7;          // consumer warps per panel CTA (7 + producer = 8 warps: 2 per SMSP, 255 regs)
constexpr int kThreads = 32 * (kWarps + 1);   // + 1 TMA producer warp
constexpr int kMaxWorld = 8;       // ranks of one NVSwitch box (fused P2P exchange)

// ------------------------------------------------------------------------------------------
// Launch parameters of the panel kernel (panel.cu).  Plain struct, passed by value.
struct PanelParams {
  const void *X;        // tile layout, input iterate X^t (or Y for the subspace sweep)
  void *Xout;           // tile layout, output X^{t+1} (RGS / GPM) or W = A Y (PRODUCT)
  // ---- dense panel kernel (panel.cu): dynamic schedule over a fixed unit list
  const int4 *units;    // [nunits] (panel, t_begin, t_end, slot): column steps [t_begin, t_end) of
                        // a panel; slot >= 0: the split unit's partial-B slot, -1: whole panel
  const int2 *pinfo;    // [panels] (units covering the panel, first slot); a split panel's slots
                        // are contiguous in column order (= the fixed combine order)
  int nunits;
  void *Bpart;          // split-unit partial B rows [slots][kWarps][EP] (EP = RT d padded to 16 B)
  unsigned *ucnt;       // [panels][consumer warps] unit arrivals per (split panel, warp); self-resetting
  unsigned *ctl;        // [0] unit queue head (runs over iters x nunits), [1] (panel, warp)
                        // epilogues completed (X^{t+1} readiness), [2] CTAs exited; self-resetting
  unsigned long long *acc;   // [iters][npart][2] exact 128-bit fixed-point sums (lo, hi); self-zeroing
  // ---- wide / sym kernels: per-CTA fp64 slots + last-CTA reduction
  double *cta_part;     // [grid][npart]
  unsigned *done_cnt;   // CTA arrival counter for the last-CTA reduction
  double *result;       // [iters][npart] doubles: reduced partials (objective / Gram terms)
  int *err;             // device error word (bit flags, see kErr*)
  unsigned *ns_region;  // float bits of max ||I - F^T F||_F (atomicMax on non-negative floats)
  int64_t n;            // total nodes
  int64_t n_local, node0, rows_local;
  int64_t tiles_per_rank;
  int world, rank;
  int panels, total_tiles;   // total_tiles = column tiles per panel (all ranks' slices)
  float a_keep;         // fraction of A accesses tagged L2 evict_last (A shard ~ L2 size), else evict_first
  int keep_panels;      // > 0: panels [0, keep_panels) always evict_last, the rest evict_first (an
                        // address-deterministic resident subset; replaces the random fraction)
  double coef;          // n - 1   (identity term of G_i)
  double eta;           // step size mu
  int K;                // Newton-Schulz steps (Algorithm 1)
  // iterations per launch (panel kernel, world == 1): iteration t reads X (t even) or Xout
  // (t odd) and writes the other; X^t is complete once ctl[1] >= t * panels * kWarps
  int iters;
  unsigned long long *ts;   // optional phase timestamps [iters][grid][kTsSlots] (%globaltimer ns), debug
  // ---- P > 1 fused X exchange over NVLink (dense kernel, RGS / GPM, one iteration per launch):
  // the epilogue also stores its X^{t+1} rows into every rank's Xout (peer_X[g], IPC-mapped);
  // at exit each CTA adds its count of (panel, warp) epilogues to every rank's arrival counter
  // for this rank (peer_cnt[g] + rank) after a system-scope release; the producer reads rank
  // g's slice of X^t only once xcnt[g] >= xtarget (its acquire).  Replaces the all-gather.
  // ---- tcgen05 wide pass (wide_tc.cu): column tiles per accumulator drain; launch epoch of the
  // per-CTA contribution flags (ucnt[cta] == epoch: the CTA's partial rows are in Bpart[cta])
  int drain_tiles;
  unsigned epoch;
  int p2p;
  unsigned xtarget;
  const unsigned *xcnt;
  void *peer_X[kMaxWorld];
  unsigned *peer_cnt[kMaxWorld];
};

// Symmetric half-storage pass (sym.cu): blocks of GP panels x kSymTilesPerBlock column tiles.
constexpr int kSymTilesPerBlock = 6;
constexpr int kSymPanelsPerBlock = 16;
struct SymParams {
  PanelParams e;          // epilogue + partial-reduction fields (X, Xout, n, node0, coef, eta, K, ...)
  float *rowpart;         // [nJ][N][d]  row-direction partials of (panel, column group J)
  float *colpart;         // [nI][N][d]  column-direction partials of (row group I, column)
  const int4 *blocks;     // active upper-triangle blocks (I, J, p_first, p_last), largest first
  unsigned *sched_cnt;    // block queue head (reset by the final kernel)
  int nblocks, nt, nJ, gp;
  int64_t N;
};

// Block-sparse storage of an incompletely observed instance (bsr.cu):
// local node row il owns blocks [rowptr[il], rowptr[il+1]) (a multiple of 4, zero-padded),
// block b = A_{node0+il, col[b]} at vals + b*d*d (row-major d x d).
struct BsrParams {
  PanelParams e;          // epilogue + partial-reduction fields (X, Xout, n_local, coef, eta, K, ...)
  const int64_t *rowptr;  // [n_local + 1]
  const int *col;         // [nnzb] global block column (node) j
  const float *vals;      // [nnzb][d][d]
  const float *Xs;        // d <= 10: padded node-major copy of X^t (bsr_xs_stride(d) floats per node)
};

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: remember it per (kernel, device)
// (a process may drive contexts on several GPUs).  `done` is a kernel-specific static table.
inline cudaError_t set_smem_attr_once(const void *kern, int bytes, bool (&done)[64]) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < 0 || dev >= 64) return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (done[dev]) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done[dev] = true;
  return e;
}

constexpr int kErrDivergence = 1;   // ||S||_F > 10 sqrt(d) or non-finite after NS
constexpr int kErrSingular = 2;     // init polar did not converge / Cholesky failed
constexpr int kErrNonfinite = 4;
constexpr int kErrTimeout = 8;      // multi-iteration grid barrier timed out (should never happen)

// Tile layout of X: the N stack rows of one rank's slice are cut into column
// tiles of 128; tile (g, j) holds d x 128 values: component pairs (2kp, 2kp+1) as pair-blocks
// of 128 x 2 (interleaved, so a lane's two adjacent columns of one pair come in one 128-bit
// load and feed FFMA2 with a broadcast A operand), and for odd d the last component as a plain
// 128-vector (its column pairs feed FFMA2 against A column pairs).  No padding component.
// Wide blocks (d > kMaxNarrowD, §8(f) row 4: the paper's d = 25) use the "wide" kernel
// (wide.cu): 32-column tiles and the X tile as a plain row-major 32 x d slab of the stack.
constexpr int kMaxNarrowD = 10;
constexpr int kWideColTile = 32;
constexpr int kMaxD = 32;
__host__ __device__ constexpr int col_tile(int d) { return d > kMaxNarrowD ? kWideColTile : kColTile; }

__host__ __device__ inline int64_t tile_index(int64_t c, int k, int d, int64_t rows_local,
                                              int64_t tiles_per_rank) {
  if (d > kMaxNarrowD) {   // wide: per-rank stack padded to whole 32-row tiles
    const int64_t g = c / rows_local, cl = c - g * rows_local;
    return ((g * tiles_per_rank * kWideColTile) + cl) * d + k;
  }
  int64_t g = c / rows_local, cl = c - g * rows_local;
  int64_t j = cl / kColTile, o = cl - j * kColTile;
  const int64_t base = (g * tiles_per_rank + j) * d * kColTile;
  if ((d & 1) && k == d - 1) return base + (int64_t)(d - 1) * kColTile + o;   // odd d: last component contiguous
  return base + (int64_t)(k & ~1) * kColTile + 2 * o + (k & 1);
}

// ------------------------------------------------------------------------------------------
// Philox4x32-10 (Salmon et al., SC'11).  Same definition as oracle/instance.py, written
// independently.
struct U4 { uint32_t x, y, z, w; };
__device__ __forceinline__ U4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                            uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
    uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  return {c0, c1, c2, c3};
}
__device__ __forceinline__ double uniform53(uint32_t a, uint32_t b) {
  uint64_t m = (uint64_t)(a >> 5) * 67108864ull + (uint64_t)(b >> 6);
  return ((double)m + 1.0) * 1.1102230246251565404236316680908203125e-16;   // 2^-53
}
// Normals 2q and 2q+1 of the stream (c0, c1, *, tag): Box-Muller on the two uniforms.
__device__ __forceinline__ void normal_pair(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t q,
                                            uint32_t tag, double &z0, double &z1) {
  U4 v = philox4x32_10(c0, c1, q, tag, (uint32_t)(seed & 0xffffffffu), (uint32_t)(seed >> 32));
  double u1 = uniform53(v.x, v.y), u2 = uniform53(v.z, v.w);
  double r = sqrt(-2.0 * log(u1));
  double th = (2.0 * 3.141592653589793) * u2;
  double s, c;
  sincos(th, &s, &c);
  z0 = r * c;
  z1 = r * s;
}

// ------------------------------------------------------------------------------------------
// PTX wrappers (sm_90+/sm_100a): mbarrier, TMA tensor + bulk copies, L2 cache policies.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint: the waiting thread is parked until the phase completes
// (or the hint expires) instead of spinning, so an idle producer does not steal issue slots
// from the consumer warp that shares its scheduler.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr), "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Fraction `f` of accesses evict_last, the rest evict_first (keeps a resident subset of a
// stream that is slightly larger than L2 instead of thrashing all of it).
__device__ __forceinline__ uint64_t policy_keep_fraction(float f) {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;" : "=l"(p) : "f"(f));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_3d(void *smem_dst, const void *tmap, uint64_t *bar, int c0,
                                            int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void *smem_dst, const void *gsrc, uint32_t bytes, uint64_t *bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(smem_dst)),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const void *tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Release/acquire ordering for the last-arriver patterns (data stores -> fence -> relaxed
// atomic; atomic observed -> fence -> data loads).  fence.acq_rel is sufficient under the PTX
// memory model and far cheaper than __threadfence()'s fence.sc (MEMBAR.SC.GPU).
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// generic-proxy writes (other CTAs' X^{t+1} stores, acquired above) before async-proxy reads
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void red_add_sys(unsigned *p, unsigned v) {
  asm volatile("red.relaxed.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// one lane of a converged warp; ptxas then emits the uniform-datapath instructions issued under
// this predicate (UTCHMMA, UTMALDG, UBLKCP, UTCBAR) straight-line — under a `lane == 0` test it
// wraps each of them in an ELECT loop (measured: 50 instead of 17 cycles per N = 32 MMA)
__device__ __forceinline__ bool elect_one() {
  uint32_t e;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(e));
  return e != 0;
}
template <typename T> struct Vec4;
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double4; };

}  // namespace nsrgs
