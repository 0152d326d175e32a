// runtime.cu — libnsrgs.so host runtime and C-ABI (include/nsrgs.h).
//
// One nsrgs_ctx per (process, GPU).  The context owns: the two X buffers in the tile layout
// (double-buffered iterate), fp64 partial / result buffers, the split-K scratch, the device
// error word, the TMA tensor map of the A shard and (world > 1) an NCCL communicator created
// from a caller-broadcast unique id.  NCCL is loaded lazily with dlopen (the already-loaded
// libnccl.so.2 of the process is preferred), so single-GPU use has no NCCL dependency.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/nsrgs.h"
#include "common.cuh"
#include "kernels.h"

using namespace nsrgs;

// ------------------------------------------------------------------------------ NCCL (dlopen)
namespace {
struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

bool load_nccl() {
  if (g_nccl.tried) return g_nccl.ok;
  g_nccl.tried = true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return false;
#define NSRGS_SYM(f, name) g_nccl.f = reinterpret_cast<decltype(g_nccl.f)>(dlsym(h, name))
  NSRGS_SYM(GetUniqueId, "ncclGetUniqueId");
  NSRGS_SYM(CommInitRank, "ncclCommInitRank");
  NSRGS_SYM(AllGather, "ncclAllGather");
  NSRGS_SYM(AllReduce, "ncclAllReduce");
  NSRGS_SYM(CommDestroy, "ncclCommDestroy");
  NSRGS_SYM(GetErrorString, "ncclGetErrorString");
#undef NSRGS_SYM
  g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.AllGather && g_nccl.AllReduce &&
              g_nccl.CommDestroy && g_nccl.GetErrorString;
  return g_nccl.ok;
}

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
// arrival counters [kMaxWorld] (then handshake words [kMaxWorld]) after X0 | X1 in an xblock
unsigned *xcnt_of(void *block, size_t xstride) {
  return reinterpret_cast<unsigned *>(static_cast<char *>(block) + 2 * xstride);
}

int plan_impl(int64_t n, int32_t d, int32_t world, int32_t rank, nsrgs_plan_t *out, std::string *why) {
  auto fail = [&](const char *m) {
    if (why) *why = m;
    return (int)NSRGS_ERR_INVALID_ARG;
  };
  if (!out) return fail("plan: out is NULL");
  if (n < 2) return fail("n must be >= 2");
  if (d < 2 || d > kMaxD) return fail("d must be in [2, 32] (d = 1: O(1) has a trivial tangent space, SPEC.md:295)");
  if (d > kMaxNarrowD && !wide_supported(d)) return fail("d in [11, 32]: supported wide sizes are 11-16, 20, 24, 25, 32");
  if (world < 1 || rank < 0 || rank >= world) return fail("need world >= 1 and 0 <= rank < world");
  if (n % world) return fail("n must be divisible by world (row-block sharding by node)");
  out->n_local = n / world;
  out->node0 = (int64_t)rank * out->n_local;
  out->rows_local = out->n_local * d;
  out->row0 = out->node0 * d;
  out->col_tile = col_tile(d);
  out->tiles_per_rank = ceil_div(out->rows_local, out->col_tile);
  out->x_slice_elems = out->tiles_per_rank * d * out->col_tile;
  out->x_elems = (int64_t)world * out->x_slice_elems;
  return NSRGS_OK;
}

template <typename T>
void pack_host_t(int64_t n, int d, const nsrgs_plan_t &pl, T *stack, T *tiled, bool unpack) {
  const int64_t N = n * d;
  if (!unpack) std::memset(tiled, 0, sizeof(T) * pl.x_elems);
  for (int64_t c = 0; c < N; ++c)
    for (int k = 0; k < d; ++k) {
      const int64_t t = tile_index(c, k, d, pl.rows_local, pl.tiles_per_rank);
      if (unpack) stack[c * d + k] = tiled[t]; else tiled[t] = stack[c * d + k];
    }
}
}  // namespace

// ------------------------------------------------------------------------------ in-process rank group
// nsrgs_debug_group (test-only): `world` emulated rank contexts of ONE process on one GPU, each
// driven by its own host thread, whose collectives exchange real data.  A collective is two
// host barriers: every rank publishes its buffer after its stream has drained; each rank then
// reads all ranks' buffers (all-reduce: one kernel summing them in rank order, so every rank
// gets the same bits; all-gather: device-to-device copies of the other ranks' slices); the
// second barrier keeps every buffer unchanged until all ranks have read it.  No kernel ever
// waits for another rank's kernel (B200_PROFILING.md: such ranks must not share a GPU).
struct RankGroup {
  int world = 0, refs = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;                  // a rank timed out: every later barrier fails at once
  void *ptr[kMaxWorld] = {};
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (broken) return false;
    const unsigned long long g0 = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    const bool ok = cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g0 || broken; });
    if (!ok || broken) {
      broken = true;
      cv.notify_all();
      return false;
    }
    return true;
  }
};
std::mutex g_group_mu;   // RankGroup reference counts

struct GroupPtrs { const double *p[kMaxWorld]; };

__global__ void group_sum_kernel(GroupPtrs g, int world, int64_t count, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int r = 0; r < world; ++r) acc += g.p[r][i];   // rank order: identical on every rank
    out[i] = acc;
  }
}

// ------------------------------------------------------------------------------ context
struct nsrgs_ctx {
  int64_t n = 0, N = 0;
  int d = 0, dtype = 0, rank = 0, world = 1, device = 0;
  size_t esz = 4;
  nsrgs_plan_t plan{};
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // A shard
  void *A = nullptr;
  int64_t lda = 0;
  bool own_A = false, have_A = false;
  CUtensorMap tmA;
  CUtensorMap tmA_sym;   // symmetric pass: same A, its own panel height
  int wide_mma = 0;      // d > 10 pass: 2 (default) 3xTF32 on tcgen05 (wide_tc.cu), 1 3xTF32 on mma.sync,
                         // 0 CUDA cores (NSRGS_WIDE_MMA); 1 and 2 read A through the 128-byte TMA swizzle
  int wide_drain = 1;    // tcgen05 pass: column tiles per accumulator drain (NSRGS_WIDE_DRAIN)
  unsigned wide_epoch = 0;
  int wide_slot = 0;     // floats per CTA partial-row slot (tcgen05 pass)
  // d = 10 on the tcgen05 pass (X stays in the narrow tile layout; wide_tc.cu NL): its own launch
  // shape, tensor map (32-column box, 128-byte swizzle) and partial buffers next to the narrow ones
  bool narrow_tc = false;
  PanelShape tc_shape{};
  int tc_grid = 0, tc_panels = 0;
  CUtensorMap tmA_tc;
  unsigned *tc_flags = nullptr, *tc_cnt = nullptr;
  void *tc_bpart = nullptr;
  double *tc_part = nullptr;
  double a_fro2 = 0.0;
  // iterate
  void *X[2] = {nullptr, nullptr};   // both inside xblock (one IPC-shareable allocation)
  void *xblock = nullptr;            // [X0 | X1 | xcnt[kMaxWorld] | hello[kMaxWorld]]
  size_t xstride = 0;                // bytes from X0 to X1 (and X1 to xcnt)
  // fused P2P exchange (world > 1): peers' xblock mapped into this process
  bool p2p = false;
  void *peer_block[kMaxWorld] = {};
  bool peer_opened[kMaxWorld] = {};
  unsigned p2p_epoch = 0;            // P2P iterations completed on this context (all ranks in lockstep)
  int cur = 0;
  bool have_X = false;
  void *stage = nullptr;   // n*d*d elements (host<->device staging for set/get/Z)
  // panel launch shape
  PanelShape shape{};
  int sm_count = 0, grid = 0, panels = 0, total_tiles = 0;
  float a_keep = 0.f;   // L2 evict_last fraction for A (only when the shard is within ~4x of L2)
  int keep_panels = 0;  // dense pass: panels [0, keep_panels) evict_last (deterministic resident subset)
  // symmetric half-storage pass (sym.cu)
  bool sym = false;
  SymShape symshape{};
  float *rowpart = nullptr, *colpart = nullptr;
  int4 *blocks = nullptr;
  unsigned *sym_cnt = nullptr;   // [0] block queue head, [1] final-kernel done counter
  double *sym_part = nullptr;
  int nblocks = 0, nJ = 0, nI = 0, sym_grid = 0;
  int64_t a_bytes_pass = 0;
  // block-sparse storage (bsr.cu)
  bool bsr = false, own_bsr = false;
  bool bsr_sorted = false;        // every row's columns non-decreasing (generator layout): slab pass
  int bsr_lg2g = -1;              // slab pass column-group size (log2), -1: per-block gather pass
  bool bsr_g4 = false;            // per-block gather by TMA tile::gather4 (tmXs over the padded X copy)
  CUtensorMap tmXs;
  int64_t *bsr_rowptr = nullptr;
  int *bsr_col = nullptr;
  float *bsr_vals = nullptr;
  int64_t bsr_nnzb = 0;
  float *bsr_xs = nullptr;        // padded node-major X copy (d <= 10)
  double *bsr_part = nullptr;     // [bsr grid][npart]
  void *yprev = nullptr;          // Chebyshev-filtered init: previous iterate (tile layout, x_elems)
  unsigned *bsr_cnt = nullptr;    // [0] last-CTA counter
  // scratch
  double *cta_part = nullptr;   // grid * npart
  unsigned *counters = nullptr; // [0] done_cnt (wide kernel)
  bool coop = false;            // multi-iteration launches available (world == 1)
  // dense panel kernel: dynamic schedule (panel.cu)
  int4 *units = nullptr;        // [nunits] (panel, t_begin, t_end, slot)
  int2 *pinfo = nullptr;        // [panels] (units covering the panel, first slot)
  int nunits = 0, nslots = 0, split_panels = 0;
  unsigned *ucnt = nullptr;     // [panels][consumer warps]
  unsigned *ctl = nullptr;      // [4] queue head, epilogues done, CTAs exited
  unsigned long long *acc = nullptr;   // [acc_cap][npart][2] fixed-point sums
  int acc_cap = 0;
  void *Bpart = nullptr;
  double *res = nullptr;        // res_cap * npart
  int res_cap = 0;
  double *red_part = nullptr;   // generic reduction partials
  int64_t red_cap = 0;
  double *small = nullptr;      // [0] a_fro2 | [1] chg2 | [8..8+2DD) MC | [kSmallOut..) F trace / metrics
  int64_t small_cap = 0;
  int *err = nullptr;
  unsigned *ns_region = nullptr;
  // NCCL
  ncclComm_t comm = nullptr;
  bool emulated = false;   // test-only: world > 1 without a communicator (collectives are no-ops)
  bool forced_nccl = false; // test-only: world == 1 with a 1-rank NCCL communicator
  RankGroup *group = nullptr;   // test-only: in-process rank group (nsrgs_debug_group)
  double *group_tmp = nullptr;  // all-reduce result before it replaces the caller's buffer
  int64_t group_cap = 0;
  unsigned long long *ts = nullptr;   // debug phase timestamps (nsrgs_debug_timestamps)
  // stats / timing
  bool timing = false;
  std::vector<cudaEvent_t> ev;
  int ev_used = 0;
  double panel_ms = 0.0;
  int64_t panel_launches = 0, kernel_launches = 0;
  double ns_region_max = 0.0;
  std::string msg;
};

namespace {
int set_err(nsrgs_ctx *c, int code, const char *fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->msg = buf;
  }
  return code;
}

#define CUDA_TRY(c, expr)                                                                        \
  do {                                                                                           \
    cudaError_t e_ = (expr);                                                                     \
    if (e_ != cudaSuccess)                                                                       \
      return set_err((c), e_ == cudaErrorMemoryAllocation ? NSRGS_ERR_OOM : NSRGS_ERR_CUDA,      \
                     "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__);      \
  } while (0)

#define NCCL_TRY(c, expr)                                                                        \
  do {                                                                                           \
    ncclResult_t r_ = (expr);                                                                    \
    if (r_ != ncclSuccess)                                                                       \
      return set_err((c), NSRGS_ERR_NCCL, "%s: %s", #expr, g_nccl.GetErrorString(r_));           \
  } while (0)

#define NSRGS_TRY(expr)              \
  do {                               \
    int s_ = (expr);                 \
    if (s_ != NSRGS_OK) return s_;   \
  } while (0)

ncclDataType_t nccl_type(const nsrgs_ctx *c) { return c->dtype == NSRGS_F32 ? ncclFloat32 : ncclFloat64; }

int enter(nsrgs_ctx *c) {
  if (!c) return NSRGS_ERR_INVALID_ARG;
  c->msg.clear();
  CUDA_TRY(c, cudaSetDevice(c->device));
  return NSRGS_OK;
}

int sync_and_check(nsrgs_ctx *c, int *flags_out = nullptr) {
  int flags = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&flags, c->err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  if (flags) {
    CUDA_TRY(c, cudaMemsetAsync(c->err, 0, sizeof(int), c->stream));
    if (flags & kErrTimeout) {   // a timed-out launch may leave the dense kernel's counters dirty
      if (c->ctl) CUDA_TRY(c, cudaMemsetAsync(c->ctl, 0, sizeof(unsigned) * 4, c->stream));
      if (c->ucnt && c->d <= kMaxNarrowD) CUDA_TRY(c, cudaMemsetAsync(c->ucnt, 0, sizeof(unsigned) * (size_t)c->panels * c->shape.nw, c->stream));
      if (c->acc) CUDA_TRY(c, cudaMemsetAsync(c->acc, 0, sizeof(unsigned long long) * 2 * (size_t)c->acc_cap * c->shape.npart, c->stream));
      CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
  }
  if (flags_out) *flags_out = flags;
  if (c->timing && c->ev_used) {
    for (int i = 0; i + 1 < c->ev_used; i += 2) {
      float ms = 0.f;
      CUDA_TRY(c, cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]));
      c->panel_ms += ms;
    }
    c->ev_used = 0;
  }
  // a caller that does not inspect the flags still must not return a result built from a
  // non-finite partial (the fixed-point sums would hide it)
  if (!flags_out && (flags & kErrNonfinite)) return set_err(c, NSRGS_ERR_NONFINITE, "non-finite partial sum");
  return NSRGS_OK;
}

int group_barrier(nsrgs_ctx *c) {
  if (!c->group->barrier())
    return set_err(c, NSRGS_ERR_NCCL, "rank group: a rank did not reach the collective within 120 s");
  return NSRGS_OK;
}

// In-process rank group: sum of every rank's `buf` in rank order (see RankGroup).
int group_allreduce(nsrgs_ctx *c, double *buf, size_t count) {
  if ((int64_t)count > c->group_cap) {
    if (c->group_tmp) cudaFree(c->group_tmp);
    c->group_tmp = nullptr;
    c->group_cap = 0;
    CUDA_TRY(c, cudaMalloc(&c->group_tmp, sizeof(double) * count));
    c->group_cap = (int64_t)count;
  }
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->group->ptr[c->rank] = buf;
  NSRGS_TRY(group_barrier(c));
  GroupPtrs g{};
  for (int r = 0; r < c->world; ++r) g.p[r] = static_cast<const double *>(c->group->ptr[r]);
  const int blocks = (int)std::min<int64_t>(1024, ((int64_t)count + 255) / 256);
  group_sum_kernel<<<blocks, 256, 0, c->stream>>>(g, c->world, (int64_t)count, c->group_tmp);
  CUDA_TRY(c, cudaGetLastError());
  c->kernel_launches++;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  NSRGS_TRY(group_barrier(c));
  CUDA_TRY(c, cudaMemcpyAsync(buf, c->group_tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, c->stream));
  return NSRGS_OK;
}

// In-process rank group: copy every other rank's slice of its X buffer into ours.
int group_allgather(nsrgs_ctx *c, void *buf) {
  const size_t bytes = (size_t)c->plan.x_slice_elems * c->esz;
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->group->ptr[c->rank] = buf;
  NSRGS_TRY(group_barrier(c));
  for (int r = 0; r < c->world; ++r)
    if (r != c->rank)
      CUDA_TRY(c, cudaMemcpyAsync(static_cast<char *>(buf) + r * bytes, static_cast<const char *>(c->group->ptr[r]) + r * bytes,
                                  bytes, cudaMemcpyDeviceToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  return group_barrier(c);
}

int allreduce_sum(nsrgs_ctx *c, double *buf, size_t count) {
  if (count == 0) return NSRGS_OK;
  if (c->group) return group_allreduce(c, buf, count);
  if ((c->world == 1 && !c->forced_nccl) || c->emulated) return NSRGS_OK;
  NCCL_TRY(c, g_nccl.AllReduce(buf, buf, count, ncclFloat64, ncclSum, c->comm, c->stream));
  return NSRGS_OK;
}

int allgather_X(nsrgs_ctx *c, void *buf) {
  if (c->group) return group_allgather(c, buf);
  if ((c->world == 1 && !c->forced_nccl) || c->emulated) return NSRGS_OK;
  const size_t cnt = (size_t)c->plan.x_slice_elems;
  char *base = static_cast<char *>(buf);
  NCCL_TRY(c, g_nccl.AllGather(base + (size_t)c->rank * cnt * c->esz, base, cnt, nccl_type(c), c->comm, c->stream));
  return NSRGS_OK;
}

int ensure_red(nsrgs_ctx *c, int64_t count) {
  if (count <= c->red_cap) return NSRGS_OK;
  if (c->red_part) cudaFree(c->red_part);
  c->red_part = nullptr;
  CUDA_TRY(c, cudaMalloc(&c->red_part, sizeof(double) * count));
  c->red_cap = count;
  return NSRGS_OK;
}

int ensure_res(nsrgs_ctx *c, int slots) {
  if (slots <= c->res_cap) return NSRGS_OK;
  if (c->res) cudaFree(c->res);
  c->res = nullptr;
  const int cap = std::max(slots, 2 * c->res_cap);
  CUDA_TRY(c, cudaMalloc(&c->res, sizeof(double) * (size_t)cap * c->shape.npart));
  c->res_cap = cap;
  return NSRGS_OK;
}

// Fixed-point accumulators of the dense kernel for `iters` iterations per launch (zeroed; the
// kernel re-zeroes what it used).
int ensure_acc(nsrgs_ctx *c, int iters) {
  if (iters <= c->acc_cap) return NSRGS_OK;
  const int cap = std::max(iters, 2 * c->acc_cap);   // geometric growth: one realloc per doubling
  if (c->acc) cudaFree(c->acc);
  c->acc = nullptr;
  c->acc_cap = 0;
  const size_t bytes = sizeof(unsigned long long) * 2 * (size_t)cap * c->shape.npart;
  CUDA_TRY(c, cudaMalloc(&c->acc, bytes));
  CUDA_TRY(c, cudaMemsetAsync(c->acc, 0, bytes, c->stream));
  c->acc_cap = cap;
  return NSRGS_OK;
}

// Work-unit list of the dense kernel (fixed per context, so results are reproducible).  Whole
// panels while more than two panels per CTA remain, then the remaining panels cut into equal
// column ranges of >= 24 tiles (~1/64 of a CTA's share), so the dynamic queue ends with small
// units and every SM finishes within about half a unit of the others.
static void build_units(nsrgs_ctx *c, std::vector<int4> &units, std::vector<int2> &pinfo) {
  const int P = c->panels, TT = c->total_tiles, G = c->sm_count;
  double tail_panels = 2.0, unit_div = 64.0;
  int unit_min = 24;
  if (const char *e = std::getenv("NSRGS_UNITS")) std::sscanf(e, "%lf,%lf,%d", &tail_panels, &unit_div, &unit_min);   // tuning
  const int whole = std::max(0, P - (int)(tail_panels * G));
  const double per_cta = (double)P * TT / G;
  const int unit = std::min(TT, std::max(unit_min, (int)(per_cta / unit_div)));
  const int S = std::max(1, (TT + unit / 2) / unit);   // units per split panel
  units.clear();
  pinfo.assign(P, make_int2(1, -1));
  int slot = 0;
  for (int pnl = 0; pnl < P; ++pnl) {
    if (pnl < whole || S == 1) {
      units.push_back(make_int4(pnl, 0, TT, -1));
      continue;
    }
    pinfo[pnl] = make_int2(S, slot);
    for (int u = 0; u < S; ++u)
      units.push_back(make_int4(pnl, (int)((int64_t)TT * u / S), (int)((int64_t)TT * (u + 1) / S), slot++));
  }
  c->nunits = (int)units.size();
  c->nslots = slot;
  c->split_panels = S == 1 ? 0 : P - whole;
}

int ensure_small(nsrgs_ctx *c, int64_t count) {
  if (count <= c->small_cap) return NSRGS_OK;
  double *nb = nullptr;
  CUDA_TRY(c, cudaMalloc(&nb, sizeof(double) * count));
  CUDA_TRY(c, cudaMemsetAsync(nb, 0, sizeof(double) * count, c->stream));
  if (c->small) {
    CUDA_TRY(c, cudaMemcpyAsync(nb, c->small, sizeof(double) * c->small_cap, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    cudaFree(c->small);
  }
  c->small = nb;
  c->small_cap = count;
  return NSRGS_OK;
}
constexpr int kSmallFro = 0, kSmallChg = 1, kSmallMC = 8, kSmallOut = 8 + 2 * kMaxD * kMaxD;   // MC holds 2 d^2

int build_tmap(nsrgs_ctx *c, CUtensorMap *out = nullptr, int rows = 0) {
  if (!out) out = &c->tmA;
  if (rows <= 0) rows = c->shape.rows;
  static EncodeTiledFn encode = nullptr;
  if (!encode) {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CUDA_TRY(c, cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      return set_err(c, NSRGS_ERR_CUDA, "cuTensorMapEncodeTiled not available from the driver");
    encode = reinterpret_cast<EncodeTiledFn>(fn);
  }
  const cuuint64_t Nr = (cuuint64_t)c->plan.rows_local;
  cuuint64_t dims[3] = {c->world == 1 ? (cuuint64_t)c->N : Nr, (cuuint64_t)c->world, (cuuint64_t)c->plan.rows_local};
  cuuint64_t strides[2] = {c->world == 1 ? (cuuint64_t)(c->lda * c->esz) : (cuuint64_t)(Nr * c->esz),
                           (cuuint64_t)(c->lda * c->esz)};
  const bool tcmap = out == &c->tmA_tc;   // d = 10 on the tcgen05 pass: 32-column swizzled boxes
  cuuint32_t box[3] = {(cuuint32_t)(tcmap ? kWideColTile : col_tile(c->d)), 1u, (cuuint32_t)rows};
  cuuint32_t estr[3] = {1u, 1u, 1u};
  const bool swz = tcmap || (out == &c->tmA && c->wide_mma != 0);   // the tensor-core passes read swizzled tiles
  CUresult r = encode(out, c->dtype == NSRGS_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                      3, c->A, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(c, NSRGS_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
  return NSRGS_OK;
}

// One panel-kernel launch: X[src] -> out (mode), partials into res slot.
int launch_panel(nsrgs_ctx *c, int mode, const void *Xin, void *Xout, double *result, double eta, int K,
                 int iters = 1, bool p2p = false) {
  PanelParams p{};
  p.iters = iters;
  if (p2p) {   // fused exchange (one iteration per launch): see PanelParams
    const size_t off = static_cast<char *>(Xout) - static_cast<char *>(c->xblock);
    p.p2p = 1;
    p.xtarget = c->p2p_epoch * (unsigned)c->panels * (unsigned)c->shape.nw;
    p.xcnt = xcnt_of(c->xblock, c->xstride);
    for (int g = 0; g < c->world; ++g) {
      p.peer_X[g] = static_cast<char *>(c->peer_block[g]) + off;
      p.peer_cnt[g] = xcnt_of(c->peer_block[g], c->xstride);
    }
  }
  p.ts = c->ts;
  if (c->d <= kMaxNarrowD && !c->sym && !c->bsr) NSRGS_TRY(ensure_acc(c, iters));
  p.X = Xin;
  p.Xout = Xout;
  p.units = c->units;
  p.pinfo = c->pinfo;
  p.nunits = c->nunits;
  p.Bpart = c->Bpart;
  p.ucnt = c->ucnt;
  p.ctl = c->ctl;
  p.acc = c->acc;
  p.cta_part = c->cta_part;
  p.done_cnt = c->counters;
  p.result = result;
  p.err = c->err;
  p.ns_region = c->ns_region;
  p.n = c->n;
  p.n_local = c->plan.n_local;
  p.node0 = c->plan.node0;
  p.rows_local = c->plan.rows_local;
  p.tiles_per_rank = c->plan.tiles_per_rank;
  p.world = c->world;
  p.rank = c->rank;
  p.panels = c->panels;
  p.total_tiles = c->total_tiles;
  p.a_keep = c->a_keep;
  p.keep_panels = c->keep_panels;
  p.coef = (double)(c->n - 1);
  p.eta = eta;
  p.K = K;
  if (c->timing) {
    while ((int)c->ev.size() < c->ev_used + 2) {
      cudaEvent_t e;
      CUDA_TRY(c, cudaEventCreate(&e));
      c->ev.push_back(e);
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[c->ev_used], c->stream));
  }
  if (c->bsr) {
    BsrParams bp{};
    bp.e = p;
    bp.e.cta_part = c->bsr_part;
    bp.e.done_cnt = c->bsr_cnt;
    bp.rowptr = c->bsr_rowptr;
    bp.col = c->bsr_col;
    bp.vals = c->bsr_vals;
    if (c->d <= kMaxNarrowD) {   // X^t -> padded node-major records for the per-lane gathers
      CUDA_TRY(c, launch_bsr_pack_x(c->d, Xin, c->bsr_xs, c->n, c->plan.rows_local, c->plan.tiles_per_rank,
                                    c->bsr_lg2g >= 0 || c->bsr_g4, c->stream));
      c->kernel_launches++;
      bp.Xs = c->bsr_xs;
    }
    CUDA_TRY(c, bsr_dispatch(c->d, mode, &bp, c->bsr_lg2g, c->bsr_g4 ? &c->tmXs : nullptr, c->stream));
  } else if (c->sym) {
    SymParams sp{};
    sp.e = p;
    sp.e.cta_part = c->sym_part;
    sp.e.done_cnt = c->sym_cnt + 1;
    sp.rowpart = c->rowpart;
    sp.colpart = c->colpart;
    sp.blocks = c->blocks;
    sp.sched_cnt = c->sym_cnt;
    sp.nblocks = c->nblocks;
    sp.nt = (int)c->plan.tiles_per_rank;
    sp.nJ = c->nJ;
    sp.gp = kSymPanelsPerBlock;
    sp.N = c->N;
    CUDA_TRY(c, sym_dispatch(c->d, mode, false, nullptr, &c->tmA_sym, &sp, c->sym_grid, c->stream));
    c->kernel_launches++;
  } else if (c->narrow_tc && iters == 1 && !p2p) {
    p.drain_tiles = c->wide_drain;
    p.epoch = ++c->wide_epoch;
    p.panels = c->tc_panels;
    p.ucnt = c->tc_flags;
    p.Bpart = c->tc_bpart;
    p.cta_part = c->tc_part;
    p.done_cnt = c->tc_cnt;
    if (c->tc_grid > c->grid) p.ts = nullptr;   // the timestamp buffer is sized for the CUDA-core grid
    CUDA_TRY(c, wide_tc_dispatch(c->d, mode, false, nullptr, nullptr, &c->tmA_tc, &p, c->tc_grid, c->stream));
  } else if (c->d > kMaxNarrowD) {
    if (c->wide_mma == 2) {
      p.drain_tiles = c->wide_drain;
      p.epoch = ++c->wide_epoch;
      CUDA_TRY(c, wide_tc_dispatch(c->d, mode, false, nullptr, nullptr, &c->tmA, &p, c->grid, c->stream));
    } else {
      CUDA_TRY(c, wide_dispatch(c->d, mode, false, nullptr, &c->tmA, &p, c->grid, c->stream, c->wide_mma == 1));
    }
  } else {
    CUDA_TRY(c, panel_dispatch(c->dtype, c->d, mode, false, nullptr, &c->tmA, &p, c->grid, c->stream));
  }
  if (c->timing) {
    CUDA_TRY(c, cudaEventRecord(c->ev[c->ev_used + 1], c->stream));
    c->ev_used += 2;
  }
  c->panel_launches += iters;   // per-pass statistics: one launch may run several iterations
  c->kernel_launches++;
  return NSRGS_OK;
}

int objective_from_res(nsrgs_ctx *c, int T, double *host_out) {
  NSRGS_TRY(ensure_small(c, kSmallOut + std::max(T, 8)));
  CUDA_TRY(c, launch_objective_final(c->d, T, c->res, c->shape.npart, c->small + kSmallFro, c->small + kSmallOut,
                                     c->stream));
  c->kernel_launches++;
  if (host_out)
    CUDA_TRY(c, cudaMemcpyAsync(host_out, c->small + kSmallOut, sizeof(double) * T, cudaMemcpyDeviceToHost, c->stream));
  return NSRGS_OK;
}

// F(X[cur]) with fp64 accumulation of <X, A X> (objective64.cu) into small[kSmallOut + slot]:
// X unpacked to the row-major stack in `stage`, xs and Gram partials reduced in fixed order into
// res_slot (the fused kernels' npart layout), all-reduced, then the shared finaliser.
int objective_fp64(nsrgs_ctx *c, double *res_slot, int out_slot) {
  if (c->dtype != NSRGS_F32) return set_err(c, NSRGS_ERR_INVALID_ARG, "objective_fp64: F32 contexts only");
  const int np = c->shape.npart;
  CUDA_TRY(c, launch_pack(c->dtype, c->d, c->n, c->stage, c->X[c->cur], c->plan.rows_local, c->plan.tiles_per_rank, 1,
                          c->stream));
  Obj64Args a{};
  obj64_grids(c->plan.n_local, c->d, c->bsr, c->sm_count, &a.grid_x, &a.grid_g);
  NSRGS_TRY(ensure_red(c, (int64_t)a.grid_x + (int64_t)a.grid_g * 8 * np));
  a.part_x = c->red_part;
  a.part_g = c->red_part + a.grid_x;
  if (c->bsr) {
    a.bsr_rowptr = c->bsr_rowptr;
    a.bsr_col = c->bsr_col;
    a.bsr_vals = c->bsr_vals;
  } else {
    a.A = static_cast<const float *>(c->A);
    a.lda = c->lda;
  }
  a.n = c->n;
  a.n_local = c->plan.n_local;
  a.node0 = c->plan.node0;
  a.Xs = static_cast<const float *>(c->stage);
  a.sm_count = c->sm_count;
  CUDA_TRY(c, launch_obj64(c->d, a, c->stream));
  CUDA_TRY(c, launch_reduce(a.part_g, a.grid_g * 8, np, res_slot, c->stream));
  CUDA_TRY(c, launch_reduce(a.part_x, a.grid_x, 1, res_slot + np - 1, c->stream));
  c->kernel_launches += 5;
  NSRGS_TRY(allreduce_sum(c, res_slot, np));
  NSRGS_TRY(ensure_small(c, kSmallOut + out_slot + 1));
  CUDA_TRY(c, launch_objective_final(c->d, 1, res_slot, np, c->small + kSmallFro, c->small + kSmallOut + out_slot,
                                     c->stream));
  c->kernel_launches++;
  return NSRGS_OK;
}

int fro2_finish(nsrgs_ctx *c, int nblocks) {
  CUDA_TRY(c, launch_reduce(c->red_part, nblocks, 1, c->small + kSmallFro, c->stream));
  c->kernel_launches++;
  NSRGS_TRY(allreduce_sum(c, c->small + kSmallFro, 1));
  CUDA_TRY(c, cudaMemcpyAsync(&c->a_fro2, c->small + kSmallFro, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  NSRGS_TRY(sync_and_check(c));
  return NSRGS_OK;
}

// Leave block-sparse storage (a dense A is being attached / generated).
void drop_bsr(nsrgs_ctx *c) {
  if (c->own_bsr) {
    cudaFree(c->bsr_rowptr);
    cudaFree(c->bsr_col);
    cudaFree(c->bsr_vals);
  }
  c->bsr_rowptr = nullptr;
  c->bsr_col = nullptr;
  c->bsr_vals = nullptr;
  c->own_bsr = false;
  c->bsr = false;
  c->bsr_sorted = false;
  c->bsr_nnzb = 0;
}

// Scratch of the block-sparse pass: padded X copy (d <= 10), per-CTA partial slots, counter.
int bsr_scratch(nsrgs_ctx *c) {
  if (c->d <= kMaxNarrowD && !c->bsr_xs)
    CUDA_TRY(c, cudaMalloc(&c->bsr_xs, sizeof(float) * (size_t)c->n * bsr_xs_stride(c->d, true)));
  if (!c->bsr_part)
    CUDA_TRY(c, cudaMalloc(&c->bsr_part, sizeof(double) * (size_t)bsr_grid(c->d, c->plan.n_local) * c->shape.npart));
  if (!c->bsr_cnt) {
    CUDA_TRY(c, cudaMalloc(&c->bsr_cnt, 4 * sizeof(unsigned)));
    CUDA_TRY(c, cudaMemsetAsync(c->bsr_cnt, 0, 4 * sizeof(unsigned), c->stream));
  }
  c->a_bytes_pass = c->bsr_nnzb * (int64_t)(c->d * c->d * 4 + 4) + 8 * (c->plan.n_local + 1);
  const char *env = std::getenv("NSRGS_BSR_SLAB");
  const double p_eff = (double)c->bsr_nnzb / ((double)c->plan.n_local * (double)c->n);
  c->bsr_lg2g = (c->bsr_sorted && !(env && env[0] == '0')) ? bsr_slab_lg2g(c->d, p_eff) : -1;
  const char *env4 = std::getenv("NSRGS_BSR_G4");
  // opt-in (measured slower than the LSU gather at n 20000: d 5 p 0.5 4.40 vs 4.14 ms, d 3 2.39 vs
  // 1.86 ms; p 0.1 1.18 vs 1.23 ms — the TMA unit's per-operation cost dominates 4-row gathers)
  c->bsr_g4 = c->bsr_lg2g < 0 && c->d <= 6 && env4 && env4[0] == '1';
  if (c->bsr_g4) {   // the padded X copy as an n x DSS tensor, one row (record) per gathered box row
    static EncodeTiledFn encode = nullptr;
    if (!encode) {
      void *fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      CUDA_TRY(c, cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
      if (!fn || q != cudaDriverEntryPointSuccess)
        return set_err(c, NSRGS_ERR_CUDA, "cuTensorMapEncodeTiled not available from the driver");
      encode = reinterpret_cast<EncodeTiledFn>(fn);
    }
    const int dss = bsr_xs_stride(c->d, true);
    cuuint64_t dims[2] = {(cuuint64_t)dss, (cuuint64_t)c->n};
    cuuint64_t strides[1] = {(cuuint64_t)dss * 4};
    cuuint32_t box[2] = {(cuuint32_t)dss, 1u};
    cuuint32_t estr[2] = {1u, 1u};
    CUresult r = encode(&c->tmXs, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, c->bsr_xs, dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) c->bsr_g4 = false;   // fall back to the LSU gather
  }
  return NSRGS_OK;
}

int require_ready(nsrgs_ctx *c, bool need_X) {
  if (!c->have_A) return set_err(c, NSRGS_ERR_STATE, "no A: call nsrgs_generate or nsrgs_attach_A first");
  if (need_X && !c->have_X) return set_err(c, NSRGS_ERR_STATE, "no iterate: call nsrgs_init_spectral or nsrgs_set_X");
  return NSRGS_OK;
}
}  // namespace

// ------------------------------------------------------------------------------ C-ABI
extern "C" {

int nsrgs_version(void) { return NSRGS_VERSION; }

int nsrgs_plan(int64_t n, int32_t d, int32_t world, int32_t rank, nsrgs_plan_t *out) {
  return plan_impl(n, d, world, rank, out, nullptr);
}

int nsrgs_pack_host(int64_t n, int32_t d, int32_t world, int32_t dtype, const void *stack, void *tiled) {
  nsrgs_plan_t pl;
  int s = plan_impl(n, d, world, 0, &pl, nullptr);
  if (s) return s;
  if (!stack || !tiled) return NSRGS_ERR_INVALID_ARG;
  if (dtype == NSRGS_F32) pack_host_t<float>(n, d, pl, (float *)stack, (float *)tiled, false);
  else if (dtype == NSRGS_F64) pack_host_t<double>(n, d, pl, (double *)stack, (double *)tiled, false);
  else return NSRGS_ERR_INVALID_ARG;
  return NSRGS_OK;
}

int nsrgs_unpack_host(int64_t n, int32_t d, int32_t world, int32_t dtype, const void *tiled, void *stack) {
  nsrgs_plan_t pl;
  int s = plan_impl(n, d, world, 0, &pl, nullptr);
  if (s) return s;
  if (!stack || !tiled) return NSRGS_ERR_INVALID_ARG;
  if (dtype == NSRGS_F32) pack_host_t<float>(n, d, pl, (float *)stack, (float *)tiled, true);
  else if (dtype == NSRGS_F64) pack_host_t<double>(n, d, pl, (double *)stack, (double *)tiled, true);
  else return NSRGS_ERR_INVALID_ARG;
  return NSRGS_OK;
}

int nsrgs_get_nccl_unique_id(void *out128) {
  if (!out128) return NSRGS_ERR_INVALID_ARG;
  if (!load_nccl()) return NSRGS_ERR_NCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return NSRGS_ERR_NCCL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out128, &id, 128);
  return NSRGS_OK;
}

static thread_local std::string g_create_msg;

const char *nsrgs_last_error(const nsrgs_ctx *ctx) { return ctx ? ctx->msg.c_str() : g_create_msg.c_str(); }

// Fused-exchange setup, collective over the communicator (world > 1, not emulated): map every
// peer's xblock with CUDA IPC and prove each mapping with a write handshake.  Any failure on any
// rank leaves every rank on the NCCL all-gather path (same decision everywhere).
static int setup_p2p(nsrgs_ctx *c) {
  const char *env = getenv("NSRGS_P2P");
  bool ok = c->world <= kMaxWorld && c->d <= kMaxNarrowD && !(env && env[0] == '0');
  constexpr int kH = (int)sizeof(cudaIpcMemHandle_t);   // 64 bytes
  char *dh = nullptr;   // [world][kH] handles, then one double for the agreement sums
  CUDA_TRY(c, cudaMalloc(&dh, (size_t)kH * c->world + 16));
  cudaIpcMemHandle_t mine{};
  if (ok) ok = cudaIpcGetMemHandle(&mine, c->xblock) == cudaSuccess;
  cudaGetLastError();
  std::vector<cudaIpcMemHandle_t> all(c->world);
  double *flag = reinterpret_cast<double *>(dh + (size_t)kH * c->world);
  int rc = NSRGS_OK;
  auto agree = [&](bool mine_ok, bool *all_ok) -> int {   // all ranks ok?
    const double bad = mine_ok ? 0.0 : 1.0;
    CUDA_TRY(c, cudaMemcpyAsync(flag, &bad, sizeof bad, cudaMemcpyHostToDevice, c->stream));
    NCCL_TRY(c, g_nccl.AllReduce(flag, flag, 1, ncclFloat64, ncclSum, c->comm, c->stream));
    double tot = 0.0;
    CUDA_TRY(c, cudaMemcpyAsync(&tot, flag, sizeof tot, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    *all_ok = tot == 0.0;
    return NSRGS_OK;
  };
  do {
    CUDA_TRY(c, cudaMemcpyAsync(dh + (size_t)kH * c->rank, &mine, kH, cudaMemcpyHostToDevice, c->stream));
    NCCL_TRY(c, g_nccl.AllGather(dh + (size_t)kH * c->rank, dh, kH, ncclInt8, c->comm, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(all.data(), dh, (size_t)kH * c->world, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    bool all_ok = false;
    if ((rc = agree(ok, &all_ok)) != NSRGS_OK) break;
    if (!all_ok) { ok = false; break; }
    for (int g = 0; g < c->world && ok; ++g) {
      if (g == c->rank) { c->peer_block[g] = c->xblock; continue; }
      ok = cudaIpcOpenMemHandle(&c->peer_block[g], all[g], cudaIpcMemLazyEnablePeerAccess) == cudaSuccess;
      c->peer_opened[g] = ok;
    }
    cudaGetLastError();
    // handshake: write a token into every peer's hello[rank], barrier, check our hello[]
    const unsigned token = 0x5EED0000u;
    for (int g = 0; g < c->world && ok; ++g) {
      if (g == c->rank) continue;
      const unsigned v = token + (unsigned)c->rank;
      unsigned *hello = xcnt_of(c->peer_block[g], c->xstride) + kMaxWorld;
      ok = cudaMemcpy(hello + c->rank, &v, sizeof v, cudaMemcpyHostToDevice) == cudaSuccess;
    }
    cudaGetLastError();
    if ((rc = agree(ok, &all_ok)) != NSRGS_OK) break;   // also the barrier after the writes
    if (!all_ok) { ok = false; break; }
    unsigned hello[kMaxWorld] = {};
    CUDA_TRY(c, cudaMemcpy(hello, xcnt_of(c->xblock, c->xstride) + kMaxWorld, sizeof(unsigned) * c->world,
                           cudaMemcpyDeviceToHost));
    for (int g = 0; g < c->world; ++g)
      if (g != c->rank && hello[g] != token + (unsigned)g) ok = false;
    if ((rc = agree(ok, &all_ok)) != NSRGS_OK) break;
    ok = all_ok;
  } while (false);
  cudaFree(dh);
  if (rc != NSRGS_OK) return rc;
  if (!ok) {
    for (int g = 0; g < kMaxWorld; ++g)
      if (c->peer_opened[g]) cudaIpcCloseMemHandle(c->peer_block[g]);
    for (int g = 0; g < kMaxWorld; ++g) { c->peer_opened[g] = false; c->peer_block[g] = nullptr; }
  }
  c->p2p = ok;
  return NSRGS_OK;
}

int nsrgs_destroy(nsrgs_ctx *c) {
  if (!c) return NSRGS_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  for (auto e : c->ev) cudaEventDestroy(e);
  for (int g = 0; g < kMaxWorld; ++g)
    if (c->peer_opened[g]) cudaIpcCloseMemHandle(c->peer_block[g]);
  if (c->group) {
    std::lock_guard<std::mutex> lk(g_group_mu);
    if (--c->group->refs == 0) delete c->group;
    c->group = nullptr;
  }
  if (c->group_tmp) cudaFree(c->group_tmp);
  void *bufs[] = {c->tc_flags, c->tc_cnt, c->tc_bpart, c->tc_part, c->units, c->pinfo, c->ucnt, c->ctl, c->acc, c->ts, c->xblock, c->stage, c->cta_part, c->counters, c->Bpart, c->res, c->red_part, c->small,
                  c->err, c->ns_region, c->rowpart, c->colpart, c->blocks, c->sym_cnt, c->sym_part,
                  c->bsr_xs, c->bsr_part, c->bsr_cnt, c->yprev};
  for (void *b : bufs)
    if (b) cudaFree(b);
  if (c->own_A && c->A) cudaFree(c->A);
  if (c->own_bsr) {
    cudaFree(c->bsr_rowptr);
    cudaFree(c->bsr_col);
    cudaFree(c->bsr_vals);
  }
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return NSRGS_OK;
}

int nsrgs_create(const nsrgs_desc *desc, nsrgs_ctx **out) {
  if (!out) return NSRGS_ERR_INVALID_ARG;
  *out = nullptr;
  if (!desc) return NSRGS_ERR_INVALID_ARG;
  nsrgs_ctx *c = new nsrgs_ctx();
  std::string why;
  // nsrgs_last_error(NULL) reports why a create failed
  auto bail = [&](int code, const char *m = nullptr) {
    g_create_msg = m ? m : (why.empty() ? c->msg : why);
    nsrgs_destroy(c);
    return code;
  };
  g_create_msg.clear();
  if (desc->dtype != NSRGS_F32 && desc->dtype != NSRGS_F64) return bail(NSRGS_ERR_INVALID_ARG, "dtype must be F32 or F64");
  int s = plan_impl(desc->n, desc->d, desc->world, desc->rank, &c->plan, &why);
  if (s) return bail(s);
  if (desc->dtype == NSRGS_F64 && desc->d > 6) return bail(NSRGS_ERR_INVALID_ARG, "F64 supports d in [2, 6]");
  // Test-only rank emulation (NSRGS_EMULATE_RANKS=1): a context for (rank, world > 1) without a
  // communicator, so the sharded kernels can be exercised rank by rank on one GPU (no rank ever
  // waits for another); the caller assembles X across ranks.
  const char *emu = getenv("NSRGS_EMULATE_RANKS");
  c->emulated = desc->world > 1 && desc->nccl_unique_id == nullptr && emu && emu[0] == '1';
  if ((desc->world > 1) != (desc->nccl_unique_id != nullptr) && !c->emulated)
    return bail(NSRGS_ERR_INVALID_ARG, "nccl_unique_id must be given iff world > 1");
  c->n = desc->n;
  c->d = desc->d;
  c->N = desc->n * desc->d;
  c->dtype = desc->dtype;
  c->esz = desc->dtype == NSRGS_F32 ? 4 : 8;
  c->rank = desc->rank;
  c->world = desc->world;
  c->device = desc->device;
  if (c->world > 1 && (c->plan.rows_local * (int64_t)c->esz) % 16)
    return bail(NSRGS_ERR_INVALID_ARG, "world > 1 needs (n/world)*d*sizeof(dtype) % 16 == 0");
  if (cudaSetDevice(c->device) != cudaSuccess) return bail(NSRGS_ERR_CUDA, "cudaSetDevice failed (no GPU?)");
  if (desc->cuda_stream) {
    c->stream = static_cast<cudaStream_t>(desc->cuda_stream);
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) return bail(NSRGS_ERR_CUDA);
    c->own_stream = true;
  }
  cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device);
  if (c->d > kMaxNarrowD) {
    if (c->dtype != NSRGS_F32) return bail(NSRGS_ERR_INVALID_ARG, "d > 10 supports F32 only");
    {
      const char *wm = std::getenv("NSRGS_WIDE_MMA");
      // 3xTF32 tensor-core pass by default (accumulator drained per tile: ≤ 3.1e-7 per step vs
      // 8.4e-7 on CUDA cores, 1.07-1.9x faster; profiles/r01c_wide_variants.txt); =0 CUDA cores
      c->wide_mma = (wm && wm[0] >= '0' && wm[0] <= '2') ? wm[0] - '0' : 2;
      if (const char *wd = std::getenv("NSRGS_WIDE_DRAIN")) c->wide_drain = std::max(1, std::atoi(wd));
    }
    if (c->wide_mma == 2)
      wide_tc_dispatch(c->d, 0, true, &c->shape, &c->wide_slot, nullptr, nullptr, 0, nullptr);
    else
      wide_dispatch(c->d, 0, true, &c->shape, nullptr, nullptr, 0, nullptr, c->wide_mma == 1);
  } else {
    panel_dispatch(c->dtype, c->d, 0, true, &c->shape, nullptr, nullptr, 0, nullptr);
  }
  // launch shape: persistent CTAs (one per SM) over a dynamic queue of work units; wide: CTA per panel
  c->panels = (int)ceil_div(c->plan.rows_local, c->shape.rows);
  c->total_tiles = (int)(c->world * c->plan.tiles_per_rank);
  std::vector<int4> units;
  std::vector<int2> pinfo;
  if (c->d <= kMaxNarrowD) build_units(c, units, pinfo);
  c->grid = c->d > kMaxNarrowD ? c->panels : std::min(c->nunits, c->sm_count);
  if (c->d > kMaxNarrowD && c->wide_mma == 2) {   // persistent stream-K grid: >= 8 column tiles per CTA
    const int64_t U = (int64_t)c->panels * c->total_tiles;
    c->grid = (int)std::max<int64_t>(1, std::min<int64_t>(c->sm_count, U / 8));
  }
  {
    int l2 = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device);
    const double a_bytes = (double)c->esz * (double)c->plan.rows_local * (double)c->N;
    // Part of A stays L2-resident across passes: the first panels (an address-deterministic
    // subset of ~0.45 L2) are loaded evict_last, the rest evict_first.  Measured on B200 (coop
    // per-iteration time, tools/keep_sweep2.sh): n=2000 d=3 (144 MB) 22.1 us vs 23.1 with the
    // earlier random-fraction policy (createpolicy.fractional, best at 0.55 L2) and 31.3 with
    // none; 324 MB 56.3 vs 59.3 us; keeping more than ~0.5 L2 thrashes (0.7: 27.1 us), as the
    // evict_last capacity is about half of the split L2.  None beyond 2.8 L2 (400 MB: keeping
    // anything was 3 % slower).
    const double ratio = a_bytes / std::max(1.0, (double)l2);
    const double panel_bytes = (double)c->esz * (double)c->shape.rows * (double)c->N;
    if (ratio <= 2.8) c->keep_panels = (int)(0.45 * (double)l2 / std::max(1.0, panel_bytes));
    // the symmetric and wide passes keep the random-fraction policy (0.55 / 0.4 L2 of A)
    const double kept = ratio <= 1.5 ? 0.55 * l2 : ratio <= 2.8 ? 0.4 * l2 : 0.0;
    c->a_keep = (float)std::min(1.0, kept / std::max(1.0, a_bytes));
    if (const char *ek = std::getenv("NSRGS_A_KEEP")) {   // experiment: the random-fraction policy
      c->a_keep = (float)std::atof(ek);
      c->keep_panels = 0;
    }
    if (const char *kp = std::getenv("NSRGS_KEEP_L2_FRAC"))   // experiment: kept share of L2
      c->keep_panels = (int)(std::atof(kp) * (double)l2 / std::max(1.0, panel_bytes));
  }
  auto alloc = [&](void **p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes);
    if (e != cudaSuccess) return false;
    return cudaMemsetAsync(*p, 0, bytes, c->stream) == cudaSuccess;
  };
  const size_t xb = c->esz * (size_t)c->plan.x_elems;
  c->xstride = (xb + 255) / 256 * 256;
  bool ok = alloc(&c->xblock, 2 * c->xstride + 2 * sizeof(unsigned) * kMaxWorld);
  if (ok) {
    c->X[0] = c->xblock;
    c->X[1] = static_cast<char *>(c->xblock) + c->xstride;
  }
  ok = ok && alloc(&c->stage, c->esz * (size_t)(c->n * c->d * c->d)) &&
            alloc((void **)&c->cta_part, sizeof(double) * (size_t)c->grid * 2 * c->shape.npart) &&
            alloc((void **)&c->counters, sizeof(unsigned) * 64) &&
            alloc((void **)&c->err, sizeof(int)) && alloc((void **)&c->ns_region, sizeof(unsigned));
  if (ok && c->d <= kMaxNarrowD) {
    ok = alloc((void **)&c->units, sizeof(int4) * units.size()) && alloc((void **)&c->pinfo, sizeof(int2) * pinfo.size()) &&
         alloc((void **)&c->ucnt, sizeof(unsigned) * (size_t)c->panels * c->shape.nw) &&
         alloc((void **)&c->ctl, sizeof(unsigned) * 4) &&
         alloc(&c->Bpart, c->esz * (size_t)std::max(1, c->nslots) * (c->shape.rows * c->d + 4 * 8));   // per-warp rows padded to 16 B
    if (ok) ok = cudaMemcpyAsync(c->units, units.data(), sizeof(int4) * units.size(), cudaMemcpyHostToDevice, c->stream) == cudaSuccess &&
                 cudaMemcpyAsync(c->pinfo, pinfo.data(), sizeof(int2) * pinfo.size(), cudaMemcpyHostToDevice, c->stream) == cudaSuccess &&
                 cudaStreamSynchronize(c->stream) == cudaSuccess;
  }
  if (ok && c->d > kMaxNarrowD && c->wide_mma == 2)
    ok = alloc((void **)&c->ucnt, sizeof(unsigned) * 2 * (size_t)c->grid) &&   // two partial segments per CTA
         alloc(&c->Bpart, sizeof(float) * 2 * (size_t)c->grid * (size_t)c->wide_slot);
  {
    // d = 10 (c4): the CUDA-core pass is FMA co-limited under the power cap; the
    // tcgen05 pass streams it at the rate of d = 16.  World 1, fp32, dense storage; small
    // instances keep the cooperative multi-iteration CUDA-core launch (latency-bound there).
    const char *nt = std::getenv("NSRGS_NARROW_TC");
    const double a_bytes = (double)c->esz * (double)c->plan.rows_local * (double)c->N;
    const bool want = nt ? nt[0] == '1' : a_bytes >= 4e9;
    if (ok && want && c->d == 10 && c->dtype == NSRGS_F32 && c->world == 1 && !c->emulated) {
      int slot = 0;
      wide_tc_dispatch(c->d, 0, true, &c->tc_shape, &slot, nullptr, nullptr, 0, nullptr);
      c->tc_panels = (int)ceil_div(c->plan.rows_local, c->tc_shape.rows);
      const int64_t U = (int64_t)c->tc_panels * 4 * c->total_tiles;
      c->tc_grid = (int)std::max<int64_t>(1, std::min<int64_t>(c->sm_count, U / 8));
      ok = alloc((void **)&c->tc_flags, sizeof(unsigned) * 2 * (size_t)c->tc_grid) &&
           alloc(&c->tc_bpart, sizeof(float) * 2 * (size_t)c->tc_grid * (size_t)slot) &&
           alloc((void **)&c->tc_part, sizeof(double) * 2 * (size_t)c->tc_grid * c->tc_shape.npart) &&
           alloc((void **)&c->tc_cnt, sizeof(unsigned) * 64);
      c->narrow_tc = ok;
    }
  }
  if (!ok) return bail(NSRGS_ERR_OOM, "device allocation failed");
  if (c->d <= kMaxNarrowD && ensure_acc(c, 1)) return bail(NSRGS_ERR_OOM);
  if (ensure_res(c, 128) || ensure_small(c, kSmallOut + 256)) return bail(NSRGS_ERR_OOM);
  // Test-only (NSRGS_FORCE_NCCL=1, world == 1): run every collective through a real 1-rank
  // NCCL communicator so the NCCL plumbing is exercised on a single GPU.
  const char *force = getenv("NSRGS_FORCE_NCCL");
  c->forced_nccl = c->world == 1 && force && force[0] == '1';
  if ((c->world > 1 && !c->emulated) || c->forced_nccl) {
    if (!load_nccl()) return bail(NSRGS_ERR_NCCL, "libnccl.so.2 not loadable");
    ncclUniqueId id;
    if (c->forced_nccl) {
      if (g_nccl.GetUniqueId(&id) != ncclSuccess) return bail(NSRGS_ERR_NCCL, "ncclGetUniqueId failed");
    } else {
      std::memcpy(&id, desc->nccl_unique_id, sizeof id);
    }
    if (g_nccl.CommInitRank(&c->comm, c->world, id, c->rank) != ncclSuccess) return bail(NSRGS_ERR_NCCL, "ncclCommInitRank failed");
    if (c->world > 1) {
      const int r = setup_p2p(c);
      if (r != NSRGS_OK) return bail(r, c->msg.c_str());
    }
  }
  {
    int coop = 0;
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, c->device);
    const char *env = getenv("NSRGS_NO_COOP");
    c->coop = coop && c->world == 1 && !c->forced_nccl && c->d <= kMaxNarrowD && !c->narrow_tc && !(env && env[0] == '1');
  }
  if (cudaStreamSynchronize(c->stream) != cudaSuccess) return bail(NSRGS_ERR_CUDA);
  *out = c;
  return NSRGS_OK;
}

int nsrgs_attach_A(nsrgs_ctx *c, const void *A_shard_dev, int64_t lda) {
  NSRGS_TRY(enter(c));
  if (!A_shard_dev || lda < c->N || (lda * (int64_t)c->esz) % 16 || (reinterpret_cast<uintptr_t>(A_shard_dev) % 16))
    return set_err(c, NSRGS_ERR_INVALID_ARG, "attach_A: need non-NULL 16-byte aligned A, lda >= n d, lda*esz %% 16 == 0");
  drop_bsr(c);
  if (c->own_A && c->A) cudaFree(c->A);
  c->A = const_cast<void *>(A_shard_dev);
  c->lda = lda;
  c->own_A = false;
  NSRGS_TRY(build_tmap(c));
  if (c->sym) NSRGS_TRY(build_tmap(c, &c->tmA_sym, c->symshape.rows));
  if (c->narrow_tc) NSRGS_TRY(build_tmap(c, &c->tmA_tc, c->tc_shape.rows));
  int nb = 0;
  NSRGS_TRY(ensure_red(c, 8 * 4096));
  CUDA_TRY(c, launch_sumsq(c->dtype, c->A, c->plan.rows_local, c->N, c->lda, c->red_part, &nb, c->stream));
  c->kernel_launches++;
  NSRGS_TRY(fro2_finish(c, nb));
  c->have_A = true;
  return NSRGS_OK;
}

int nsrgs_generate(nsrgs_ctx *c, uint64_t seed, double sigma, void *Z_out_host) {
  return nsrgs_generate_observed(c, seed, sigma, 1.0, Z_out_host);
}

int nsrgs_generate_observed(nsrgs_ctx *c, uint64_t seed, double sigma, double p_obs, void *Z_out_host) {
  NSRGS_TRY(enter(c));
  if (!(sigma >= 0.0) || !std::isfinite(sigma)) return set_err(c, NSRGS_ERR_INVALID_ARG, "sigma must be finite, >= 0");
  if (!(p_obs > 0.0 && p_obs <= 1.0)) return set_err(c, NSRGS_ERR_INVALID_ARG, "p must be in (0, 1]");
  drop_bsr(c);
  const int64_t align = 16 / (int64_t)c->esz;
  const int64_t lda = ceil_div(c->N, align) * align;
  if (!(c->own_A && c->A && c->lda == lda)) {
    if (c->own_A && c->A) cudaFree(c->A);
    c->A = nullptr;
    c->own_A = false;
    CUDA_TRY(c, cudaMalloc(&c->A, c->esz * (size_t)c->plan.rows_local * (size_t)lda));
    c->own_A = true;
    c->lda = lda;
    if (lda != c->N)
      CUDA_TRY(c, cudaMemsetAsync(c->A, 0, c->esz * (size_t)c->plan.rows_local * (size_t)lda, c->stream));
  }
  double *Z64 = nullptr;
  CUDA_TRY(c, cudaMalloc(&Z64, sizeof(double) * (size_t)(c->n * c->d * c->d)));
  CUDA_TRY(c, launch_gen_Z(c->dtype, c->d, c->n, seed, Z64, Z_out_host ? c->stage : nullptr, c->stream));
  c->kernel_launches += Z_out_host ? 2 : 1;
  const int64_t nbx = ceil_div(c->n, 128), nby = std::min<int64_t>(c->plan.n_local, 32768);
  NSRGS_TRY(ensure_red(c, nbx * nby));
  int nb = 0;
  CUDA_TRY(c, launch_gen_A(c->dtype, c->d, c->n, c->plan.node0, c->plan.n_local, seed, sigma, p_obs, Z64, c->A,
                           c->lda, c->red_part, &nb, c->stream));
  c->kernel_launches++;
  if (Z_out_host)
    CUDA_TRY(c, cudaMemcpyAsync(Z_out_host, c->stage, c->esz * (size_t)(c->n * c->d * c->d), cudaMemcpyDeviceToHost,
                                c->stream));
  NSRGS_TRY(build_tmap(c));
  if (c->sym) NSRGS_TRY(build_tmap(c, &c->tmA_sym, c->symshape.rows));
  if (c->narrow_tc) NSRGS_TRY(build_tmap(c, &c->tmA_tc, c->tc_shape.rows));
  int s = fro2_finish(c, nb);
  cudaFree(Z64);
  if (s) return s;
  c->have_A = true;
  return NSRGS_OK;
}

int nsrgs_copy_A_rows(nsrgs_ctx *c, int64_t row0, int64_t nrows, void *out_host) {
  NSRGS_TRY(enter(c));
  if (!c->have_A) return set_err(c, NSRGS_ERR_STATE, "no A");
  if (c->bsr) return set_err(c, NSRGS_ERR_STATE, "copy_A_rows: A is block-sparse (use nsrgs_get_A_bsr)");
  if (!out_host || row0 < 0 || nrows < 0 || row0 + nrows > c->plan.rows_local)
    return set_err(c, NSRGS_ERR_INVALID_ARG, "copy_A_rows: bad range");
  CUDA_TRY(c, cudaMemcpy2DAsync(out_host, c->esz * c->N, static_cast<char *>(c->A) + c->esz * row0 * c->lda,
                                c->esz * c->lda, c->esz * c->N, nrows, cudaMemcpyDeviceToHost, c->stream));
  return sync_and_check(c);
}

int nsrgs_generate_observed_bsr(nsrgs_ctx *c, uint64_t seed, double sigma, double p_obs, void *Z_out_host) {
  NSRGS_TRY(enter(c));
  if (c->dtype != NSRGS_F32) return set_err(c, NSRGS_ERR_INVALID_ARG, "block-sparse storage: F32 only");
  if (!(sigma >= 0.0) || !std::isfinite(sigma)) return set_err(c, NSRGS_ERR_INVALID_ARG, "sigma must be finite, >= 0");
  if (!(p_obs > 0.0 && p_obs <= 1.0)) return set_err(c, NSRGS_ERR_INVALID_ARG, "p must be in (0, 1]");
  drop_bsr(c);
  if (c->own_A && c->A) cudaFree(c->A);   // the dense shard is not needed any more
  c->A = nullptr;
  c->own_A = false;
  c->have_A = false;
  c->sym = false;
  const int64_t nl = c->plan.n_local, DD = (int64_t)c->d * c->d;
  double *Z64 = nullptr;
  int64_t *cnt = nullptr;
  CUDA_TRY(c, cudaMalloc(&Z64, sizeof(double) * (size_t)(c->n * DD)));
  CUDA_TRY(c, cudaMalloc(&cnt, sizeof(int64_t) * (size_t)nl));
  CUDA_TRY(c, cudaMalloc(&c->bsr_rowptr, sizeof(int64_t) * (size_t)(nl + 1)));
  c->own_bsr = true;
  CUDA_TRY(c, launch_gen_Z(c->dtype, c->d, c->n, seed, Z64, Z_out_host ? c->stage : nullptr, c->stream));
  CUDA_TRY(c, launch_bsr_count(c->n, c->plan.node0, nl, seed, p_obs, cnt, c->bsr_rowptr, c->stream));
  c->kernel_launches += (Z_out_host ? 2 : 1) + 2;
  int64_t nnzb = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&nnzb, c->bsr_rowptr + nl, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  NSRGS_TRY(sync_and_check(c));
  cudaError_t e1 = cudaMalloc(&c->bsr_col, sizeof(int) * (size_t)std::max<int64_t>(nnzb, 1));
  cudaError_t e2 = cudaMalloc(&c->bsr_vals, sizeof(float) * (size_t)std::max<int64_t>(nnzb * DD, 1));
  if (e1 != cudaSuccess || e2 != cudaSuccess) {
    cudaFree(Z64);
    cudaFree(cnt);
    drop_bsr(c);
    return set_err(c, NSRGS_ERR_OOM, "block-sparse A: cannot allocate %lld blocks", (long long)nnzb);
  }
  c->bsr_nnzb = nnzb;
  NSRGS_TRY(ensure_red(c, std::max<int64_t>(nl, 1)));
  CUDA_TRY(c, launch_bsr_fill(c->d, c->n, c->plan.node0, nl, seed, sigma, p_obs, Z64, c->bsr_rowptr, c->bsr_col,
                              c->bsr_vals, c->red_part, c->stream));
  c->kernel_launches++;
  if (Z_out_host)
    CUDA_TRY(c, cudaMemcpyAsync(Z_out_host, c->stage, c->esz * (size_t)(c->n * DD), cudaMemcpyDeviceToHost, c->stream));
  int st = fro2_finish(c, (int)nl);
  cudaFree(Z64);
  cudaFree(cnt);
  if (st) return st;
  c->bsr_sorted = true;
  NSRGS_TRY(bsr_scratch(c));
  c->bsr = true;
  c->have_A = true;
  return sync_and_check(c);
}

int nsrgs_attach_A_bsr(nsrgs_ctx *c, const int64_t *rowptr_dev, const int32_t *col_dev, const void *vals_dev,
                       int64_t nnzb) {
  NSRGS_TRY(enter(c));
  if (c->dtype != NSRGS_F32) return set_err(c, NSRGS_ERR_INVALID_ARG, "block-sparse storage: F32 only");
  if (!rowptr_dev || nnzb < 0 || (nnzb > 0 && (!col_dev || !vals_dev)) || (reinterpret_cast<uintptr_t>(vals_dev) % 4))
    return set_err(c, NSRGS_ERR_INVALID_ARG, "attach_A_bsr: need rowptr, col, vals (4-byte aligned), nnzb >= 0");
  {   // structural check before anything is replaced (the passes index X by col[b])
    int *bad = nullptr, hbad = 0;
    CUDA_TRY(c, cudaMalloc(&bad, sizeof(int)));
    CUDA_TRY(c, cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
    CUDA_TRY(c, launch_bsr_validate(rowptr_dev, col_dev, c->plan.n_local, nnzb, c->n, bad, c->stream));
    c->kernel_launches++;
    CUDA_TRY(c, cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    const cudaError_t e = cudaStreamSynchronize(c->stream);
    cudaFree(bad);
    CUDA_TRY(c, e);
    if (hbad & 1) return set_err(c, NSRGS_ERR_INVALID_ARG, "attach_A_bsr: rowptr must start at 0, be non-decreasing and end at nnzb");
    if (hbad & 2) return set_err(c, NSRGS_ERR_INVALID_ARG, "attach_A_bsr: col[] outside [0, n)");
  }
  drop_bsr(c);
  if (c->own_A && c->A) cudaFree(c->A);
  c->A = nullptr;
  c->own_A = false;
  c->sym = false;
  c->bsr_rowptr = const_cast<int64_t *>(rowptr_dev);
  c->bsr_col = const_cast<int *>(col_dev);
  c->bsr_vals = static_cast<float *>(const_cast<void *>(vals_dev));
  c->bsr_nnzb = nnzb;
  int nb = 0;
  NSRGS_TRY(ensure_red(c, 1024));
  CUDA_TRY(c, launch_bsr_sumsq(c->bsr_vals, nnzb * c->d * c->d, c->red_part, &nb, c->stream));
  c->kernel_launches++;
  NSRGS_TRY(fro2_finish(c, nb));
  NSRGS_TRY(bsr_scratch(c));
  c->bsr = true;
  c->have_A = true;
  return sync_and_check(c);
}

int nsrgs_get_A_bsr(nsrgs_ctx *c, int64_t *nnzb_out, int64_t *rowptr_host, int32_t *col_host, void *vals_host) {
  NSRGS_TRY(enter(c));
  if (!c->bsr) return set_err(c, NSRGS_ERR_STATE, "get_A_bsr: A is not block-sparse");
  if (nnzb_out) *nnzb_out = c->bsr_nnzb;
  const int64_t DD = (int64_t)c->d * c->d;
  if (rowptr_host)
    CUDA_TRY(c, cudaMemcpyAsync(rowptr_host, c->bsr_rowptr, sizeof(int64_t) * (size_t)(c->plan.n_local + 1),
                                cudaMemcpyDeviceToHost, c->stream));
  if (col_host && c->bsr_nnzb)
    CUDA_TRY(c, cudaMemcpyAsync(col_host, c->bsr_col, sizeof(int) * (size_t)c->bsr_nnzb, cudaMemcpyDeviceToHost,
                                c->stream));
  if (vals_host && c->bsr_nnzb)
    CUDA_TRY(c, cudaMemcpyAsync(vals_host, c->bsr_vals, sizeof(float) * (size_t)(c->bsr_nnzb * DD),
                                cudaMemcpyDeviceToHost, c->stream));
  return sync_and_check(c);
}

int nsrgs_set_X(nsrgs_ctx *c, const void *X, int on_device) {
  NSRGS_TRY(enter(c));
  if (!X) return set_err(c, NSRGS_ERR_INVALID_ARG, "set_X: NULL");
  const size_t bytes = c->esz * (size_t)(c->n * c->d * c->d);
  const void *src = X;
  if (!on_device) {
    CUDA_TRY(c, cudaMemcpyAsync(c->stage, X, bytes, cudaMemcpyHostToDevice, c->stream));
    src = c->stage;
  }
  CUDA_TRY(c, launch_pack(c->dtype, c->d, c->n, src, c->X[c->cur], c->plan.rows_local, c->plan.tiles_per_rank, 0,
                          c->stream));
  c->kernel_launches++;
  NSRGS_TRY(sync_and_check(c));
  c->have_X = true;
  return NSRGS_OK;
}

int nsrgs_get_X(nsrgs_ctx *c, void *X, int on_device) {
  NSRGS_TRY(enter(c));
  if (!X) return set_err(c, NSRGS_ERR_INVALID_ARG, "get_X: NULL");
  if (!c->have_X) return set_err(c, NSRGS_ERR_STATE, "no iterate");
  const size_t bytes = c->esz * (size_t)(c->n * c->d * c->d);
  void *dst = on_device ? X : c->stage;
  CUDA_TRY(c, launch_pack(c->dtype, c->d, c->n, dst, c->X[c->cur], c->plan.rows_local, c->plan.tiles_per_rank, 1,
                          c->stream));
  c->kernel_launches++;
  if (!on_device) CUDA_TRY(c, cudaMemcpyAsync(X, c->stage, bytes, cudaMemcpyDeviceToHost, c->stream));
  return sync_and_check(c);
}

int nsrgs_init_spectral(nsrgs_ctx *c, uint64_t seed, int max_sweeps, double tol, int *sweeps_used) {
  NSRGS_TRY(enter(c));
  NSRGS_TRY(require_ready(c, false));
  if (max_sweeps < 1 || !(tol > 0.0)) return set_err(c, NSRGS_ERR_INVALID_ARG, "init_spectral: max_sweeps >= 1, tol > 0");
  const int DD = c->d * c->d;
  CUDA_TRY(c, launch_gen_Y0(c->dtype, c->d, c->n, seed, c->X[c->cur], c->plan.rows_local, c->plan.tiles_per_rank,
                            c->stream));
  c->kernel_launches++;
  const int64_t nbs = ceil_div(c->plan.rows_local, 256);
  NSRGS_TRY(ensure_red(c, nbs));
  int sweeps = 0, stalled = 0;
  bool converged = false;
  // Stopping (reading R14): the subspace change chg = ||Y_new - Y_old (Y_old^T Y_new)||_F < tol,
  // the first sweep never counts.  In fp32 the change cannot fall below its rounding floor
  // (Y_new is stored in fp32: ~ sqrt(2 d) eps per sweep, amplified by the filter), so a tol
  // below the floor is replaced by it: chg < max(tol, floor), floor = 50 sqrt(d) eps_dtype
  // (fp32: 6.7e-6 at d = 5, 1.5e-5 at d = 25; measured floors 1e-6 / 1e-5, R14).  A
  // change that has stalled within 10x of the floor (no new minimum for 3 sweeps) is that
  // floor too.  Anything else keeps iterating: a slowly contracting instance (gap ratio near 1)
  // runs until tol or max_sweeps (NSRGS_ERR_EIG_NOT_CONVERGED) instead of stopping early.
  const double eps_t = c->dtype == NSRGS_F32 ? 5.960464477539063e-08 : 1.1102230246251565e-16;
  const double floor_chg = 50.0 * std::sqrt((double)c->d) * eps_t;
  const double tol_eff = std::max(tol, floor_chg);
  double best_chg = 1e300;
  // Convergence is read back every `batch` sweeps: one host synchronisation per sweep costs
  // ~10-20 us of launch gap, which matters only when the A pass itself is short (A shard below
  // ~1 GB: <= 0.15 ms per pass); larger shards read it every sweep (no overshoot).
  const double a_bytes = (double)c->esz * (double)c->plan.rows_local * (double)c->N;
  int batch_max = a_bytes < 1e9 ? 4 : 1;
  if (const char *eb = std::getenv("NSRGS_INIT_BATCH")) batch_max = std::min(4, std::max(1, std::atoi(eb)));   // tests
  // Chebyshev filtering (reading R20): from the second sweep on, each sweep applies
  // the three-term recurrence T_{k+1}(A/b) = 2 (A/b) T_k - T_{k-1} that keeps [-b, b] bounded,
  // b = 2 ||A||_F / sqrt(N) (the Wigner bulk-edge bound: the noise spectrum of the instance lies
  // inside): the wanted directions gain x + sqrt(x^2 - 1), x = lambda_d / b, per sweep over the
  // bulk instead of lambda_d / b.  Orthonormalising Y_k and Y_{k-1} by the same right factor keeps
  // the polynomial recurrence exact (and removes any need for a scaled recurrence).  If the
  // change stalls (no gap above b), it falls back to plain sweeps.  NSRGS_INIT_CHEB=0 keeps plain
  // subspace iteration throughout.
  const char *cheb_env = std::getenv("NSRGS_INIT_CHEB");
  const bool cheb_on = !(cheb_env && cheb_env[0] == '0');
  const double bnd = 2.0 * std::sqrt(std::max(c->a_fro2, 0.0) / (double)c->N);
  bool cheb = false, cheb_failed = false;
  double prev_chg = 1e300;
  int cheb_steps = 0, cheb_stall = 0;
  if (cheb_on && !c->yprev) CUDA_TRY(c, cudaMalloc(&c->yprev, c->esz * (size_t)c->plan.x_elems));
  const int64_t ncs = ceil_div(c->plan.rows_local, 64);   // combine partial slots (per 64-row CTA)
  NSRGS_TRY(ensure_red(c, std::max<int64_t>(nbs, ncs * 2 * DD)));
  NSRGS_TRY(ensure_res(c, 1));
  const bool dbg = std::getenv("NSRGS_DEBUG_INIT") != nullptr;
  while (sweeps < max_sweeps && !converged) {
    // sweep 1 alone (its result decides whether the filter starts); then batches
    const int kb = sweeps == 0 ? 1 : std::min(batch_max, max_sweeps - sweeps);
    for (int j = 0; j < kb; ++j) {
      void *Y = c->X[c->cur], *W = c->X[1 - c->cur];
      NSRGS_TRY(launch_panel(c, kModeProduct, Y, W, c->res, 0.0, 0));
      if (!cheb) {
        NSRGS_TRY(allreduce_sum(c, c->res, 2 * DD));
      } else {
        // Y_new = alpha W - beta Y_prev (W = A Y_cur; c = 0 for the symmetric interval), Grams
        const double alpha = (cheb_steps == 0 ? 1.0 : 2.0) / bnd, beta = cheb_steps == 0 ? 0.0 : 1.0;
        int nsl = 0;
        CUDA_TRY(c, launch_cheb_combine(c->dtype, c->d, c->plan.node0, c->plan.n_local, alpha, beta, W, c->yprev, Y,
                                        c->plan.rows_local, c->plan.tiles_per_rank, c->red_part, &nsl, c->stream));
        CUDA_TRY(c, launch_reduce(c->red_part, nsl, 2 * DD, c->res, c->stream));
        c->kernel_launches += 2;
        NSRGS_TRY(allreduce_sum(c, c->res, 2 * DD));
        ++cheb_steps;
      }
      CUDA_TRY(c, launch_chol(c->d, c->res, c->small + kSmallMC, c->err, c->stream));
      int nb = 0;
      CUDA_TRY(c, launch_scale(c->dtype, c->d, c->plan.node0, c->plan.n_local, c->small + kSmallMC, W, Y,
                               c->plan.rows_local, c->plan.tiles_per_rank, c->red_part, &nb, c->stream));
      CUDA_TRY(c, launch_reduce(c->red_part, nb, 1, c->small + kSmallChg + j, c->stream));
      c->kernel_launches += 3;
      if (cheb) {   // the previous iterate in the new basis: Y_prev <- Y_cur M
        CUDA_TRY(c, launch_cheb_apply(c->dtype, c->d, c->plan.node0, c->plan.n_local, c->small + kSmallMC, Y, c->yprev,
                                      c->plan.rows_local, c->plan.tiles_per_rank, c->stream));
        c->kernel_launches++;
      }
      NSRGS_TRY(allreduce_sum(c, c->small + kSmallChg + j, 1));
      NSRGS_TRY(allgather_X(c, W));
      c->cur = 1 - c->cur;
    }
    double chg2[4] = {0.0, 0.0, 0.0, 0.0};
    CUDA_TRY(c, cudaMemcpyAsync(chg2, c->small + kSmallChg, sizeof(double) * kb, cudaMemcpyDeviceToHost, c->stream));
    int flags = 0;
    NSRGS_TRY(sync_and_check(c, &flags));
    if (flags & kErrSingular) return set_err(c, NSRGS_ERR_SINGULAR, "Cholesky of Y^T Y failed at sweep <= %d", sweeps + kb);
    if (flags & kErrNonfinite) return set_err(c, NSRGS_ERR_NONFINITE, "non-finite Gram partial at sweep <= %d", sweeps + kb);
    for (int j = 0; j < kb; ++j) {
      ++sweeps;
      if (!std::isfinite(chg2[j])) return set_err(c, NSRGS_ERR_NONFINITE, "non-finite subspace change at sweep %d", sweeps);
      const double chg = std::sqrt(chg2[j]);
      if (dbg) std::fprintf(stderr, "init sweep %d cheb %d chg %.3e bnd %.6g\n", sweeps, (int)cheb, chg, bnd);
      if (converged) continue;   // later sweeps of the batch only refine the converged subspace
      if (sweeps >= 2 && chg < tol_eff) { converged = true; continue; }
      if (sweeps >= 2) {   // stalled at the rounding floor (within 10x of it, no new minimum)
        if (chg < 10.0 * floor_chg && chg >= best_chg) {
          if (++stalled >= 3) { converged = true; continue; }
        } else if (chg < best_chg) {
          stalled = 0;
        }
        best_chg = std::min(best_chg, chg);
      }
      if (cheb) {   // stall guard: no decrease over 4 filtered sweeps while far from converged
        cheb_stall = (chg > 0.9 * prev_chg && chg > 1e-3) ? cheb_stall + 1 : 0;
        if (cheb_stall >= 4) {
          cheb = false;
          cheb_failed = true;
        }
      } else if (cheb_on && !cheb_failed && sweeps == 1 && bnd > 0.0 && std::isfinite(bnd)) {
        cheb = true;   // Y_1 is orthonormal: start the recurrence from it
      }
      prev_chg = chg;
    }
  }
  if (sweeps > max_sweeps) sweeps = max_sweeps;
  CUDA_TRY(c, launch_polar(c->dtype, c->d, c->n, c->X[c->cur], c->X[1 - c->cur], c->plan.rows_local,
                           c->plan.tiles_per_rank, c->err, c->stream));
  c->kernel_launches++;
  c->cur = 1 - c->cur;
  c->have_X = true;
  int flags = 0;
  NSRGS_TRY(sync_and_check(c, &flags));
  if (sweeps_used) *sweeps_used = sweeps;
  if (flags & kErrSingular) return set_err(c, NSRGS_ERR_SINGULAR, "init polar: Newton-Schulz did not converge (singular Y_i)");
  if (!converged)
    return set_err(c, NSRGS_ERR_EIG_NOT_CONVERGED, "subspace iteration: tol %.3g not reached in %d sweeps", tol, max_sweeps);
  return NSRGS_OK;
}

static int check_run_flags(nsrgs_ctx *c, int flags) {
  if (flags & kErrTimeout) return set_err(c, NSRGS_ERR_CUDA, "multi-iteration grid barrier timed out");
  if (flags & kErrDivergence)
    return set_err(c, NSRGS_ERR_DIVERGENCE, "Newton-Schulz retraction diverged (||S||_F > 10 sqrt(d) or non-finite)");
  if (flags & kErrSingular)
    return set_err(c, NSRGS_ERR_SINGULAR, "GPM: Newton-Schulz sign of B_i did not converge (rank-deficient block)");
  if (flags & kErrNonfinite) return set_err(c, NSRGS_ERR_NONFINITE, "non-finite objective / Gram partial");
  return NSRGS_OK;
}

static int run_impl(nsrgs_ctx *c, int mode, int T, double eta, int K, double *trace) {
  NSRGS_TRY(require_ready(c, true));
  if (T < 0 || K < 0 || (mode == kModeRgs && (!(eta > 0.0) || !std::isfinite(eta))))
    return set_err(c, NSRGS_ERR_INVALID_ARG, "run: need T >= 0, K >= 0, eta > 0");
  if (T == 0) return NSRGS_OK;
  NSRGS_TRY(ensure_res(c, T));
  if (c->p2p && !c->sym && !c->bsr) {
    // fused exchange: peers' X^{t+1} rows arrive by NVLink stores from their epilogues; no
    // all-gather.  Barrier first: every rank has finished its earlier work on its X buffers.
    if (!c->emulated) NSRGS_TRY(allreduce_sum(c, c->small + kSmallChg, 1));
    for (int t = 0; t < T; ++t) {
      NSRGS_TRY(launch_panel(c, mode, c->X[c->cur], c->X[1 - c->cur], c->res + (size_t)t * c->shape.npart, eta, K,
                             1, true));
      c->p2p_epoch++;
      c->cur = 1 - c->cur;
    }
    // every peer's stores into this rank's buffers have landed before the call returns
    if (!c->emulated) {
      CUDA_TRY(c, launch_p2p_wait(xcnt_of(c->xblock, c->xstride), c->world,
                                  c->p2p_epoch * (unsigned)c->panels * (unsigned)c->shape.nw, c->err, c->stream));
      c->kernel_launches++;
    }
  } else if (c->coop && !c->sym && !c->bsr && T > 1) {
    // one persistent cooperative launch for all T iterations (grid barrier between them, A
    // prefetched across the boundary) — removes launch gaps and pipeline drains
    NSRGS_TRY(launch_panel(c, mode, c->X[c->cur], c->X[1 - c->cur], c->res, eta, K, T));
    if (T & 1) c->cur = 1 - c->cur;
  } else {
    for (int t = 0; t < T; ++t) {
      NSRGS_TRY(launch_panel(c, mode, c->X[c->cur], c->X[1 - c->cur], c->res + (size_t)t * c->shape.npart, eta, K));
      NSRGS_TRY(allgather_X(c, c->X[1 - c->cur]));
      c->cur = 1 - c->cur;
    }
  }
  if (trace) {
    NSRGS_TRY(allreduce_sum(c, c->res, (size_t)T * c->shape.npart));
    NSRGS_TRY(objective_from_res(c, T, trace));
  }
  unsigned nr = 0;
  CUDA_TRY(c, cudaMemcpyAsync(&nr, c->ns_region, sizeof(unsigned), cudaMemcpyDeviceToHost, c->stream));
  int flags = 0;
  NSRGS_TRY(sync_and_check(c, &flags));
  float nrf;
  std::memcpy(&nrf, &nr, 4);
  c->ns_region_max = std::max(c->ns_region_max, (double)nrf);
  NSRGS_TRY(check_run_flags(c, flags));
  if (trace)
    for (int t = 0; t < T; ++t)
      if (!std::isfinite(trace[t])) return set_err(c, NSRGS_ERR_NONFINITE, "objective non-finite at t = %d", t);
  return NSRGS_OK;
}

int nsrgs_step(nsrgs_ctx *c, double eta, int K, double *objective_before) {
  NSRGS_TRY(enter(c));
  return run_impl(c, kModeRgs, 1, eta, K, objective_before);
}

int nsrgs_run(nsrgs_ctx *c, int T, double eta, int K, double *objective_trace) {
  NSRGS_TRY(enter(c));
  return run_impl(c, kModeRgs, T, eta, K, objective_trace);
}

int nsrgs_gpm_run(nsrgs_ctx *c, int T, double *objective_trace) {
  NSRGS_TRY(enter(c));
  return run_impl(c, kModeGpm, T, 0.0, 0, objective_trace);
}

int nsrgs_solve(nsrgs_ctx *c, int algorithm, int max_iter, double eta, int K, double stop_tol, int *iters_used,
                double *trace) {
  NSRGS_TRY(enter(c));
  NSRGS_TRY(require_ready(c, true));
  const int mode = algorithm == NSRGS_ALG_GPM ? kModeGpm : kModeRgs;
  if ((algorithm != NSRGS_ALG_NSRGS && algorithm != NSRGS_ALG_GPM) || max_iter < 1 || K < 0 || !(stop_tol >= 0.0) ||
      (mode == kModeRgs && !(eta > 0.0)))
    return set_err(c, NSRGS_ERR_INVALID_ARG, "solve: bad algorithm / max_iter / eta / K / stop_tol");
  NSRGS_TRY(ensure_res(c, max_iter + 1));
  NSRGS_TRY(ensure_small(c, kSmallOut + max_iter + 8));
  const int np = c->shape.npart;
  std::vector<double> F(max_iter + 1, 0.0);
  int it = 0, stopped = 0;
  if (c->dtype == NSRGS_F32) {
    // fp32 storage: F(X^t) for the stopping rule from the fp64-accumulated pass (objective64.cu).
    // The fused fp32 objective's absolute error (~0.1-1 at the paper's Table 1 size) exceeds the
    // rule's threshold 1e-8 F, so the stop would be decided by rounding.
    // Same order as the paper / oracle: F(X^0); then X^{t+1}, F(X^{t+1}), R^t.
    NSRGS_TRY(objective_fp64(c, c->res, 0));
    CUDA_TRY(c, cudaMemcpyAsync(&F[0], c->small + kSmallOut, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    NSRGS_TRY(sync_and_check(c));
    if (!std::isfinite(F[0])) return set_err(c, NSRGS_ERR_NONFINITE, "objective non-finite at t = 0");
    for (; it < max_iter;) {
      NSRGS_TRY(launch_panel(c, mode, c->X[c->cur], c->X[1 - c->cur], c->res + (size_t)(it + 1) * np, eta, K));
      NSRGS_TRY(allgather_X(c, c->X[1 - c->cur]));
      c->cur = 1 - c->cur;
      ++it;
      NSRGS_TRY(objective_fp64(c, c->res + (size_t)it * np, it));
      CUDA_TRY(c, cudaMemcpyAsync(&F[it], c->small + kSmallOut + it, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      int flags = 0;
      NSRGS_TRY(sync_and_check(c, &flags));
      NSRGS_TRY(check_run_flags(c, flags));
      if (!std::isfinite(F[it])) return set_err(c, NSRGS_ERR_NONFINITE, "objective non-finite at t = %d", it);
      if ((F[it - 1] - F[it]) / F[it] < stop_tol) break;   // R^{it-1} < tol: X = X^it
    }
    if (iters_used) *iters_used = it;
    if (trace) std::memcpy(trace, F.data(), sizeof(double) * (it + 1));
    return NSRGS_OK;
  }
  for (; it < max_iter; ++it) {
    // fp64 storage: the fused fp64 partials are exact enough.  X^it -> X^{it+1}; the same pass
    // yields the partials of F(X^it)
    NSRGS_TRY(launch_panel(c, mode, c->X[c->cur], c->X[1 - c->cur], c->res + (size_t)it * np, eta, K));
    NSRGS_TRY(allgather_X(c, c->X[1 - c->cur]));
    c->cur = 1 - c->cur;
    NSRGS_TRY(allreduce_sum(c, c->res + (size_t)it * np, np));
    CUDA_TRY(c, launch_objective_final(c->d, 1, c->res + (size_t)it * np, np, c->small + kSmallFro,
                                       c->small + kSmallOut + it, c->stream));
    c->kernel_launches++;
    CUDA_TRY(c, cudaMemcpyAsync(&F[it], c->small + kSmallOut + it, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    int flags = 0;
    NSRGS_TRY(sync_and_check(c, &flags));
    NSRGS_TRY(check_run_flags(c, flags));
    if (!std::isfinite(F[it])) return set_err(c, NSRGS_ERR_NONFINITE, "objective non-finite at t = %d", it);
    // R^{it-1} = (F(X^{it-1}) - F(X^it)) / F(X^it) < tol: X^it is the answer and
    // the speculative X^{it+1} is dropped (its pass was needed to evaluate F(X^it) anyway).
    if (it >= 1 && (F[it - 1] - F[it]) / F[it] < stop_tol) {
      c->cur = 1 - c->cur;
      stopped = 1;
      break;
    }
  }
  if (!stopped) {   // MaxIter reached: X = X^{max_iter}; evaluate F(X^{max_iter}) for the trace
    NSRGS_TRY(launch_panel(c, kModeObjective, c->X[c->cur], nullptr, c->res + (size_t)max_iter * np, 0.0, 0));
    NSRGS_TRY(allreduce_sum(c, c->res + (size_t)max_iter * np, np));
    CUDA_TRY(c, launch_objective_final(c->d, 1, c->res + (size_t)max_iter * np, np, c->small + kSmallFro,
                                       c->small + kSmallOut + max_iter, c->stream));
    c->kernel_launches++;
    CUDA_TRY(c, cudaMemcpyAsync(&F[max_iter], c->small + kSmallOut + max_iter, sizeof(double), cudaMemcpyDeviceToHost,
                                c->stream));
    NSRGS_TRY(sync_and_check(c));
    it = max_iter;
  }
  if (iters_used) *iters_used = it;
  if (trace) std::memcpy(trace, F.data(), sizeof(double) * (it + 1));
  return NSRGS_OK;
}

int nsrgs_objective_fp64(nsrgs_ctx *c, double *F_out) {
  NSRGS_TRY(enter(c));
  NSRGS_TRY(require_ready(c, true));
  if (!F_out) return set_err(c, NSRGS_ERR_INVALID_ARG, "objective_fp64: NULL out");
  NSRGS_TRY(objective_fp64(c, c->res, 0));
  CUDA_TRY(c, cudaMemcpyAsync(F_out, c->small + kSmallOut, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  NSRGS_TRY(sync_and_check(c));
  if (!std::isfinite(*F_out)) return set_err(c, NSRGS_ERR_NONFINITE, "objective non-finite");
  return NSRGS_OK;
}

int nsrgs_objective(nsrgs_ctx *c, double *F_out) {
  NSRGS_TRY(enter(c));
  NSRGS_TRY(require_ready(c, true));
  if (!F_out) return set_err(c, NSRGS_ERR_INVALID_ARG, "objective: NULL out");
  NSRGS_TRY(launch_panel(c, kModeObjective, c->X[c->cur], nullptr, c->res, 0.0, 0));
  NSRGS_TRY(allreduce_sum(c, c->res, c->shape.npart));
  NSRGS_TRY(objective_from_res(c, 1, F_out));
  NSRGS_TRY(sync_and_check(c));
  if (!std::isfinite(*F_out)) return set_err(c, NSRGS_ERR_NONFINITE, "objective non-finite");
  return NSRGS_OK;
}

int nsrgs_alignment_error(nsrgs_ctx *c, const void *Z, int Z_on_device, double out[3]) {
  NSRGS_TRY(enter(c));
  if (!c->have_X) return set_err(c, NSRGS_ERR_STATE, "no iterate");
  if (!Z || !out) return set_err(c, NSRGS_ERR_INVALID_ARG, "alignment_error: NULL argument");
  const void *Zd = Z;
  if (!Z_on_device) {
    CUDA_TRY(c, cudaMemcpyAsync(c->stage, Z, c->esz * (size_t)(c->n * c->d * c->d), cudaMemcpyHostToDevice, c->stream));
    Zd = c->stage;
  }
  const int w = 3 * c->d * c->d;
  NSRGS_TRY(ensure_red(c, ((int64_t)metrics_blocks(c->d, c->n) + 1) * w));
  NSRGS_TRY(ensure_small(c, kSmallOut + w + 8));
  int nb = 0;
  CUDA_TRY(c, launch_metrics(c->dtype, c->d, c->n, c->X[c->cur], Zd, c->plan.rows_local, c->plan.tiles_per_rank,
                             c->red_part, &nb, c->stream));
  CUDA_TRY(c, launch_reduce(c->red_part, nb, w, c->small + kSmallOut + 8, c->stream));
  CUDA_TRY(c, launch_metrics_final(c->d, c->n, c->small + kSmallOut + 8, c->small + kSmallOut, c->stream));
  c->kernel_launches += 3;
  CUDA_TRY(c, cudaMemcpyAsync(out, c->small + kSmallOut, 3 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  NSRGS_TRY(sync_and_check(c));
  if (!std::isfinite(out[0]) || !std::isfinite(out[1])) return set_err(c, NSRGS_ERR_NONFINITE, "non-finite metrics");
  return NSRGS_OK;
}

int nsrgs_set_symmetric(nsrgs_ctx *c, int enable) {
  NSRGS_TRY(enter(c));
  if (!enable) {
    c->sym = false;
    return NSRGS_OK;
  }
  if (c->world != 1 || c->dtype != NSRGS_F32 || c->d > 6)
    return set_err(c, NSRGS_ERR_INVALID_ARG, "symmetric storage: world == 1, F32, d in [2, 6] only");
  if (c->bsr) return set_err(c, NSRGS_ERR_STATE, "symmetric storage needs the dense A (block-sparse A is active)");
  if (c->sym) return NSRGS_OK;
  CUDA_TRY(c, sym_dispatch(c->d, 0, true, &c->symshape, nullptr, nullptr, 0, nullptr));
  NSRGS_TRY(build_tmap(c, &c->tmA_sym, c->symshape.rows));
  const int64_t R = c->symshape.rows, N = c->N, nt = c->plan.tiles_per_rank;
  const int GT = c->symshape.gt, GP = kSymPanelsPerBlock;
  const int np = (int)ceil_div(c->plan.rows_local, R);   // symmetric panels (its own height)
  c->nJ = (int)ceil_div(nt, GT);
  c->nI = (int)ceil_div(np, GP);
  struct Blk { int I, J, p0, p1; int64_t cost; };
  std::vector<Blk> blks;
  int64_t bytes = 0;
  for (int p = 0; p < np; ++p) {
    const int64_t rows = std::min<int64_t>(R, N - (int64_t)p * R);
    const int64_t t0 = (int64_t)p * R / kColTile;
    bytes += rows * (N - t0 * kColTile) * 4;
  }
  for (int I = 0; I < c->nI; ++I) {
    const int p0 = I * GP, p1 = std::min(np, (I + 1) * GP) - 1;
    for (int J = 0; J < c->nJ; ++J) {
      const int64_t tlo = (int64_t)J * GT, thi = std::min<int64_t>(nt, (int64_t)(J + 1) * GT);
      int plast = -1;
      int64_t cost = 0;
      for (int p = p0; p <= p1; ++p) {
        const int64_t t0 = (int64_t)p * R / kColTile;
        if (t0 >= thi) break;
        plast = p;
        cost += thi - std::max(tlo, t0);
      }
      if (plast >= p0) blks.push_back({I, J, p0, plast, cost});
    }
  }
  std::stable_sort(blks.begin(), blks.end(), [](const Blk &a, const Blk &b) { return a.cost > b.cost; });
  std::vector<int4> hb(blks.size());
  for (size_t i = 0; i < blks.size(); ++i) hb[i] = make_int4(blks[i].I, blks[i].J, blks[i].p0, blks[i].p1);
  c->nblocks = (int)hb.size();
  c->sym_grid = std::min(c->nblocks, c->sm_count);
  c->a_bytes_pass = bytes;
  const int fgrid = (int)ceil_div(c->plan.n_local, c->symshape.final_nodes_per_cta);
  auto alloc0 = [&](void **p, size_t b) -> int {
    CUDA_TRY(c, cudaMalloc(p, b));
    CUDA_TRY(c, cudaMemsetAsync(*p, 0, b, c->stream));
    return NSRGS_OK;
  };
  NSRGS_TRY(alloc0((void **)&c->rowpart, sizeof(float) * (size_t)c->nJ * N * c->d));
  NSRGS_TRY(alloc0((void **)&c->colpart, sizeof(float) * (size_t)c->nI * N * c->d));
  NSRGS_TRY(alloc0((void **)&c->blocks, sizeof(int4) * hb.size()));
  NSRGS_TRY(alloc0((void **)&c->sym_cnt, 2 * sizeof(unsigned)));
  NSRGS_TRY(alloc0((void **)&c->sym_part, sizeof(double) * (size_t)fgrid * c->shape.npart));
  CUDA_TRY(c, cudaMemcpyAsync(c->blocks, hb.data(), sizeof(int4) * hb.size(), cudaMemcpyHostToDevice, c->stream));
  CUDA_TRY(c, cudaStreamSynchronize(c->stream));
  c->sym = true;
  return NSRGS_OK;
}

int nsrgs_debug_timestamps(nsrgs_ctx *c, int max_iters, unsigned long long *out_host) {
  // max_iters > 0: (re)arm a device buffer of [max_iters][grid][8] phase stamps for the next
  // panel launches; max_iters == 0 with out_host: copy the stamps out and disarm.
  NSRGS_TRY(enter(c));
  const size_t per = (size_t)c->grid * nsrgs::kTsSlots;
  static thread_local int armed_iters = 0;
  if (max_iters > 0) {
    if (c->ts) cudaFree(c->ts);
    c->ts = nullptr;
    CUDA_TRY(c, cudaMalloc(&c->ts, sizeof(unsigned long long) * per * max_iters));
    CUDA_TRY(c, cudaMemsetAsync(c->ts, 0, sizeof(unsigned long long) * per * max_iters, c->stream));
    armed_iters = max_iters;
    return sync_and_check(c);
  }
  if (!c->ts) return set_err(c, NSRGS_ERR_STATE, "timestamps not armed");
  if (out_host)
    CUDA_TRY(c, cudaMemcpyAsync(out_host, c->ts, sizeof(unsigned long long) * per * armed_iters, cudaMemcpyDeviceToHost,
                                c->stream));
  NSRGS_TRY(sync_and_check(c));
  cudaFree(c->ts);
  c->ts = nullptr;
  return NSRGS_OK;
}

int nsrgs_debug_link_peers(nsrgs_ctx **ctxs, int world) {
  if (!ctxs || world < 2 || world > kMaxWorld) return NSRGS_ERR_INVALID_ARG;
  for (int r = 0; r < world; ++r) {
    nsrgs_ctx *c = ctxs[r];
    if (!c || !c->emulated || c->group || c->world != world || c->rank != r || c->n != ctxs[0]->n ||
        c->d != ctxs[0]->d || c->dtype != ctxs[0]->dtype || c->d > kMaxNarrowD || c->device != ctxs[0]->device)
      return c ? set_err(c, NSRGS_ERR_INVALID_ARG,
                         "link_peers: need emulated, ungrouped ranks 0..world-1 of one instance, d <= 10")
               : NSRGS_ERR_INVALID_ARG;
  }
  for (int r = 0; r < world; ++r) {
    nsrgs_ctx *c = ctxs[r];
    NSRGS_TRY(enter(c));
    NSRGS_TRY(sync_and_check(c));
    for (int g = 0; g < world; ++g) c->peer_block[g] = ctxs[g]->xblock;
    CUDA_TRY(c, cudaMemset(xcnt_of(c->xblock, c->xstride), 0, sizeof(unsigned) * kMaxWorld));
    c->p2p = true;
    c->p2p_epoch = 0;
  }
  return NSRGS_OK;
}

int nsrgs_debug_group(nsrgs_ctx **ctxs, int world) {
  if (!ctxs || world < 2 || world > kMaxWorld) return NSRGS_ERR_INVALID_ARG;
  for (int r = 0; r < world; ++r) {
    nsrgs_ctx *c = ctxs[r];
    if (!c || !c->emulated || c->group || c->p2p || c->world != world || c->rank != r || c->n != ctxs[0]->n ||
        c->d != ctxs[0]->d || c->dtype != ctxs[0]->dtype || c->device != ctxs[0]->device)
      return c ? set_err(c, NSRGS_ERR_INVALID_ARG,
                         "debug_group: need emulated, unlinked ranks 0..world-1 of one instance on one device")
               : NSRGS_ERR_INVALID_ARG;
  }
  RankGroup *g = new RankGroup();
  g->world = world;
  g->refs = world;
  for (int r = 0; r < world; ++r) {
    NSRGS_TRY(enter(ctxs[r]));
    NSRGS_TRY(sync_and_check(ctxs[r]));
    ctxs[r]->group = g;
  }
  return NSRGS_OK;
}

int nsrgs_get_stats(nsrgs_ctx *c, nsrgs_stats_t *o) {
  if (!c || !o) return NSRGS_ERR_INVALID_ARG;
  o->grid = c->grid;
  o->threads = c->shape.threads;
  o->stages = c->shape.stages;
  o->rows_per_panel = c->shape.rows;
  o->cut_panels = c->split_panels;
  o->panels = c->panels;
  o->smem_bytes = c->shape.smem;
  o->panel_ms_total = c->panel_ms;
  o->panel_launches = c->panel_launches;
  o->kernel_launches = c->kernel_launches;
  o->ns_region_max = c->ns_region_max;
  o->a_fro2 = c->a_fro2;
  o->symmetric = c->sym ? 1 : 0;
  o->a_bytes_per_pass = (c->sym || c->bsr) ? c->a_bytes_pass : (int64_t)c->esz * c->plan.rows_local * c->N;
  o->bsr = c->bsr ? 1 : 0;
  o->bsr_nnzb = c->bsr ? c->bsr_nnzb : 0;
  o->bsr_slab = (c->bsr && c->bsr_lg2g >= 0) ? 1 : 0;
  o->bsr_g4 = (c->bsr && c->bsr_g4) ? 1 : 0;
  o->wide_tc = (c->d > kMaxNarrowD && !c->bsr) ? c->wide_mma : (c->narrow_tc && !c->bsr && !c->sym) ? 2 : 0;
  o->p2p = c->p2p ? 1 : 0;
  return NSRGS_OK;
}

int nsrgs_reset_stats(nsrgs_ctx *c, int enable_panel_timing) {
  NSRGS_TRY(enter(c));
  NSRGS_TRY(sync_and_check(c));
  c->timing = enable_panel_timing != 0;
  c->panel_ms = 0.0;
  c->panel_launches = 0;
  c->kernel_launches = 0;
  c->ns_region_max = 0.0;
  c->ev_used = 0;
  CUDA_TRY(c, cudaMemsetAsync(c->ns_region, 0, sizeof(unsigned), c->stream));
  return sync_and_check(c);
}

}  // extern "C"
