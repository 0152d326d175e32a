// Standalone probe (not part of the library): one CTA runs tcgen05.mma kind::tf32, M = 128,
// N = 32, K = 32 (4 MMAs of K = 8), A K-major and B MN-major, both in 128-byte-swizzled smem,
// accumulator in TMEM, read back with tcgen05.ld 32x32b.  It pins the hand-written descriptor
// encodings a tcgen05 wide pass would use, checks whether the tensor core
// truncates or rounds fp32 operands to tf32, and evaluates the 3xTF32 split
// A·X ≈ A·X_hi + A_lo·X_hi + A·X_lo (A passed raw if the hardware truncates).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_tf32 umma_tf32.cu && ./umma_tf32
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>

constexpr int M = 128, N = 32, K = 32;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// byte offset of element (row, col) of a 128-byte-row tile under the 128-byte swizzle
__host__ __device__ inline uint32_t sw128(int row, int col) {
  return row * 128 + ((((col >> 2) ^ (row & 7)) & 7) << 4) + (col & 3) * 4;
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;        // version 1 (sm_100)
  d |= (uint64_t)2 << 61;        // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ float tf32_lo(float v) {   // v - trunc_tf32(v), exact
  const float hi = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
  return v - hi;
}

// variant 0: D = A X (raw operands); 1: 3xTF32 split; 2: TMEM st/ld round trip (no MMA);
// 3: D preloaded with 7 then accumulate; 4: B K-major (X^T tile); 5: B K-major, 3xTF32.
// Measured on B200: 4 matches the TRUNCATED-tf32 product (2e-7), i.e. kind::tf32 ignores the low
// 13 mantissa bits of fp32 operands; MN-major B (0, 1, 3) leaves D untouched with this encoding.
__global__ void __launch_bounds__(128, 1) umma_probe(const float *A, const float *X, float *D, int variant) {
  __shared__ __align__(1024) uint8_t sA[M * 128];
  __shared__ __align__(1024) uint8_t sAl[M * 128];
  __shared__ __align__(1024) uint8_t sX[K * 128];
  __shared__ __align__(1024) uint8_t sXt[N * 128];   // X^T: component n rows, K contiguous (K-major B)
  __shared__ __align__(1024) uint8_t sXlt[N * 128];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < M * K; i += 128) {
    const int r = i / K, c = i % K;
    const float v = A[i];
    *reinterpret_cast<float *>(sA + sw128(r, c)) = v;
    *reinterpret_cast<float *>(sAl + sw128(r, c)) = tf32_lo(v);
  }
  for (int i = tid; i < K * N; i += 128) {   // X tile row k (A's column) x component n
    const int k = i / N, n = i % N;
    const float v = X[i];
    *reinterpret_cast<float *>(sX + sw128(k, n)) = v;
    *reinterpret_cast<float *>(sXt + sw128(n, k)) = v;
    *reinterpret_cast<float *>(sXlt + sw128(n, k)) = tf32_lo(v);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "n"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  // idesc: D f32, A/B tf32, A K-major, B MN-major, N = 32, M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
                         ((uint32_t)(M >> 4) << 24);
  if (variant == 2 || variant == 3) {   // each thread writes its row's 32 columns, the ld below must return them
    uint32_t w[32];
    for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(variant == 3 ? 7.f : (float)(warp * 32 + lane) + j * 0.001f);
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
                 "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 ::"r"(ta), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
                 "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]),
                 "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]),
                 "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    if (variant == 2 && tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  if (variant == 6) {   // A_lo row `warp*32+lane` -> TMEM lanes, columns 32..63 (A operand from TMEM)
    uint32_t w[32];
    const int row = warp * 32 + lane;
    for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(tf32_lo(A[row * K + j]));
    const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + 32u;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
                 "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
                 ::"r"(ta), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]),
                 "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]),
                 "r"(w[16]), "r"(w[17]), "r"(w[18]), "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]),
                 "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]), "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) {
      const uint32_t idk = idesc & ~(1u << 16);
      for (int t = 0; t < 3; ++t)
        for (int ks = 0; ks < K / 8; ++ks) {
          const uint64_t da = sdesc(smem_u32(sA) + ks * 32, 16, 1024);
          const uint64_t db = sdesc(smem_u32(t == 2 ? sXlt : sXt) + ks * 32, 16, 1024);
          const uint32_t acc = (t | ks) ? 1u : 0u;
          if (t == 1)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
                         ::"r"(tmem), "r"(tmem + 32u + (uint32_t)ks * 8u), "l"(db), "r"(idk), "r"(acc));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                         ::"r"(tmem), "l"(da), "l"(db), "r"(idk), "r"(acc));
        }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
  }
  if (variant != 2 && variant != 6 && tid == 0) {
    const int nterms = (variant == 1 || variant == 5) ? 3 : 1;
    int first = variant == 3 ? 0 : 1;
    const bool kmajor_b = variant >= 4;
    const uint32_t idesc_use = kmajor_b ? (idesc & ~(1u << 16)) : idesc;
    for (int t = 0; t < nterms; ++t) {
      const uint8_t *a = t == 1 ? sAl : sA;
      const uint8_t *x = sX;   // (MN-major B is a no-op anyway: no lo tile for it)
      for (int ks = 0; ks < K / 8; ++ks) {
        const uint64_t da = sdesc(smem_u32(a) + ks * 32, 16, 1024);       // K-major: +32 B per K = 8
        const uint64_t db = kmajor_b ? sdesc(smem_u32(t == 2 ? sXlt : sXt) + ks * 32, 16, 1024)   // K-major X^T
                                     : sdesc(smem_u32(x) + ks * 1024, 16, 1024);  // MN-major: +8 rows of 128 B
        const uint32_t acc = first ? 0u : 1u;
        first = 0;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(da), "l"(db), "r"(idesc_use), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  // wait for the MMAs
  asm volatile("{\n\t.reg .pred P;\n\tWAIT:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t"
               "@!P bra WAIT;\n\t}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t v[32];
  const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "
               "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                 "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                 "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                 "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  const int row = warp * 32 + lane;
  for (int j = 0; j < 32; ++j) D[row * N + j] = __uint_as_float(v[j]);
  if (tid == 0) printf("  [dev] variant %d tmem_base 0x%08x idesc 0x%08x D[0][0..3] %g %g %g %g\n", variant, tmem,
                       (1u << 4) | (2u << 7) | (2u << 10) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24),
                       __uint_as_float(v[0]), __uint_as_float(v[1]), __uint_as_float(v[2]), __uint_as_float(v[3]));
  if (tid == 33) printf("  [dev] row 33 D[33][0..1] %g %g\n", __uint_as_float(v[0]), __uint_as_float(v[1]));
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(64));
}

static float trunc_tf32(float v) { uint32_t u; memcpy(&u, &v, 4); u &= 0xFFFFE000u; memcpy(&v, &u, 4); return v; }
static float rne_tf32(float v) {
  uint32_t u; memcpy(&u, &v, 4);
  u += 0xFFFu + ((u >> 13) & 1u); u &= 0xFFFFE000u; memcpy(&v, &u, 4); return v;
}

int main() {
  float *A, *X, *D;
  cudaMallocManaged(&A, M * K * 4); cudaMallocManaged(&X, K * N * 4); cudaMallocManaged(&D, M * N * 4);
  uint64_t s = 12345;
  auto rnd = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (float)((s >> 11) * 0x1.0p-53) - 0.5f; };
  for (int i = 0; i < M * K; ++i) A[i] = rnd();
  for (int i = 0; i < K * N; ++i) X[i] = rnd();
  {
    double ex0 = 0; for (int k = 0; k < K; ++k) ex0 += (double)A[k] * X[k * N];
    printf("host D[0][0] exact %g\n", ex0);
  }
  for (int variant = 0; variant < 7; ++variant) {
    memset(D, 0, M * N * 4);
    umma_probe<<<1, 128>>>(A, X, D, variant);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("variant %d: CUDA error %s\n", variant, cudaGetErrorString(e)); return 1; }
    double e_exact = 0, e_tr = 0, e_rn = 0, ref = 0;
    for (int r = 0; r < M; ++r)
      for (int n = 0; n < N; ++n) {
        double ex = 0, tr = 0, rn = 0;
        for (int k = 0; k < K; ++k) {
          const float a = A[r * K + k], x = X[k * N + n];
          ex += (double)a * x;
          tr += (double)trunc_tf32(a) * trunc_tf32(x);
          rn += (double)rne_tf32(a) * rne_tf32(x);
        }
        const double g = D[r * N + n];
        e_exact = fmax(e_exact, fabs(g - ex)); e_tr = fmax(e_tr, fabs(g - tr)); e_rn = fmax(e_rn, fabs(g - rn));
        ref = fmax(ref, fabs(ex));
      }
    printf("variant %d (%s): max|D| %.3f  max err vs exact %.3e  vs trunc-tf32 %.3e  vs rne-tf32 %.3e\n", variant,
           variant == 0 ? "raw operands" : variant == 1 ? "3xTF32 split" : variant == 2 ? "tmem roundtrip" : variant == 3 ? "preload 7, accumulate" : variant == 4 ? "K-major B" : variant == 5 ? "K-major B, 3xTF32" : "3xTF32, A_lo operand in TMEM", ref, e_exact, e_tr, e_rn);
  }
  return 0;
}
