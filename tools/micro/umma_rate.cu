// Standalone probe (not part of the library): issue rate of small-N tcgen05.mma kind::tf32
// (M = 128, K = 8) from one thread — same vs alternating accumulators, A from smem (SS) vs TMEM
// (TS), N = 32 / 64 / 128 / 256 — to find what bounds the wide pass's MMA warp (wide_tc.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_rate umma_rate.cu && ./umma_rate
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
__device__ __forceinline__ uint32_t idesc(int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}

extern __shared__ uint8_t dyn[];

__global__ void __launch_bounds__(128, 1) rate(int pattern, int reps, long long *out) {
  uint8_t *sm = dyn + (((smem_u32(dyn) + 1023u) & ~1023u) - smem_u32(dyn));
  uint8_t *sA = sm;                 // 256 rows x 128 B
  uint8_t *sB = sm + 32768;         // 256 rows x 128 B
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 65536 / 4; i += 128) reinterpret_cast<float *>(sm)[i] = 0.001f * (float)(i % 97);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tmem_base;
  // patterns >= 13: pattern - 13 issued by warp 0 while warps 1..3 keep TMEM busy with the split /
  // drain traffic of wide_tc.cu (per rep and warp: 4 x STTM.x16 + 1 x LDTM.x32 + waits)
  const int traffic = pattern >= 13;
  if (traffic) pattern -= 2;   // 13 -> 11 (all-TS sequence), 14 -> 12 (all-TS stacked)
  if (traffic && warp > 0) {
    uint32_t w[16], v[32];
    for (int j = 0; j < 16; ++j) w[j] = tid * 16 + j;
    const uint32_t la = tm + ((uint32_t)(warp * 32) << 16);
    for (int r = 0; r < reps; ++r) {
      for (int q = 0; q < 4; ++q)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     ::"r"(la + 384u + 16u * q), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]),
                       "r"(w[7]), "r"(w[8]), "r"(w[9]), "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]) : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 "
                   "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                     "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
                     "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
                     "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                   : "r"(la + 448u) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      w[r & 15] += v[r & 31];
    }
    if (w[3] == 0x12345678u) out[8] = w[5];
  }
  uint32_t elected = 0;
  if (warp == 0)
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(elected));
  if (warp == 0 && elected) {
    const uint32_t a0 = smem_u32(sA), b0 = smem_u32(sB);
    int count = 0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      switch (pattern) {
        case 0: for (int k = 0; k < 4; ++k) { mma_ss(tm, sdesc(a0 + k * 32), sdesc(b0 + k * 32), idesc(32), 1); ++count; } break;
        case 1: for (int k = 0; k < 4; ++k) { mma_ss(tm + 32 * k, sdesc(a0 + k * 32), sdesc(b0 + k * 32), idesc(32), 1); ++count; } break;
        case 2: for (int k = 0; k < 4; ++k) { mma_ts(tm, tm + 256 + k * 8, sdesc(b0 + k * 32), idesc(32), 1); ++count; } break;
        case 3: for (int k = 0; k < 4; ++k) { mma_ts(tm + 32 * k, tm + 256 + k * 8, sdesc(b0 + k * 32), idesc(32), 1); ++count; } break;
        case 4: for (int k = 0; k < 4; ++k) { mma_ss(tm, sdesc(a0 + k * 32), sdesc(b0 + k * 32), idesc(64), 1); ++count; } break;
        case 5: for (int k = 0; k < 4; ++k) { mma_ss(tm + 64 * (k & 1), sdesc(a0 + k * 32), sdesc(b0 + k * 32), idesc(64), 1); ++count; } break;
        case 6: for (int k = 0; k < 4; ++k) { mma_ss(tm, sdesc(a0 + k * 32), sdesc(b0 + k * 32), idesc(128), 1); ++count; } break;
        case 7: for (int k = 0; k < 4; ++k) { mma_ss(tm, sdesc(a0 + k * 32), sdesc(b0 + k * 32), idesc(256), 1); ++count; } break;
        case 8:   // wide_tc.cu's per-stage sequence: 2 halves x 4 K-steps x (TS main, SS main, SS hilo), N = 32
          for (int h = 0; h < 2; ++h)
            for (int k = 0; k < 4; ++k) {
              mma_ts(tm + 64 * h, tm + 256 + 32 * h + k * 8, sdesc(b0 + k * 32), idesc(32), 1);
              mma_ss(tm + 64 * h, sdesc(a0 + h * 16384 + k * 32), sdesc(b0 + k * 32), idesc(32), 1);
              mma_ss(tm + 128 + 32 * h, sdesc(a0 + h * 16384 + k * 32), sdesc(b0 + 4096 + k * 32), idesc(32), 1);
              count += 3;
            }
          break;
        case 9:   // stacked: SS N = 64 over [X_hi | X_lo] + TS N = 32, per half and K-step
          for (int h = 0; h < 2; ++h)
            for (int k = 0; k < 4; ++k) {
              mma_ss(tm + 64 * h, sdesc(a0 + h * 16384 + k * 32), sdesc(b0 + k * 32), idesc(64), 1);
              mma_ts(tm + 64 * h, tm + 256 + 32 * h + k * 8, sdesc(b0 + k * 32), idesc(32), 1);
              count += 2;
            }
          break;
        case 10:  // K-step outer, halves inner (alternating accumulators), unstacked
          for (int k = 0; k < 4; ++k)
            for (int h = 0; h < 2; ++h) {
              mma_ts(tm + 64 * h, tm + 256 + 32 * h + k * 8, sdesc(b0 + k * 32), idesc(32), 1);
              mma_ss(tm + 128 + 32 * h, sdesc(a0 + h * 16384 + k * 32), sdesc(b0 + 4096 + k * 32), idesc(32), 1);
              mma_ss(tm + 64 * h, sdesc(a0 + h * 16384 + k * 32), sdesc(b0 + k * 32), idesc(32), 1);
              count += 3;
            }
          break;
        case 11:  // all-TS: A_hi and A_lo both from TMEM (three N = 32 TS MMAs per half and K-step)
          for (int h = 0; h < 2; ++h)
            for (int k = 0; k < 4; ++k) {
              mma_ts(tm + 64 * h, tm + 256 + 32 * h + k * 8, sdesc(b0 + k * 32), idesc(32), 1);
              mma_ts(tm + 64 * h, tm + 320 + 32 * h + k * 8, sdesc(b0 + k * 32), idesc(32), 1);
              mma_ts(tm + 128 + 32 * h, tm + 320 + 32 * h + k * 8, sdesc(b0 + 4096 + k * 32), idesc(32), 1);
              count += 3;
            }
          break;
        case 12:  // all-TS stacked: TS N = 64 (A_hi) + TS N = 32 (A_lo)
          for (int h = 0; h < 2; ++h)
            for (int k = 0; k < 4; ++k) {
              mma_ts(tm + 64 * h, tm + 320 + 32 * h + k * 8, sdesc(b0 + k * 32), idesc(64), 1);
              mma_ts(tm + 64 * h, tm + 256 + 32 * h + k * 8, sdesc(b0 + k * 32), idesc(32), 1);
              count += 2;
            }
          break;
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    const long long t1 = clock64();
    asm volatile("{\n\t.reg .pred P;\n\tWAIT:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n\t@!P bra WAIT;\n\t}" ::"r"(smem_u32(&bar)));
    const long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; out[2] = count; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long *out;
  cudaMallocManaged(&out, 64);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 68 * 1024);
  const char *names[] = {"SS N=32 one accumulator", "SS N=32 four accumulators", "TS N=32 one accumulator",
                         "TS N=32 four accumulators", "SS N=64 one accumulator", "SS N=64 two accumulators",
                         "SS N=128", "SS N=256", "wide_tc stage sequence (24 MMAs)", "stacked stage sequence (16 MMAs)",
                         "K-outer interleaved sequence (24)", "all-TS sequence (24)", "all-TS stacked sequence (16)",
                         "all-TS (24) + STTM/LDTM traffic x3 warps", "all-TS stacked (16) + traffic"};
  for (int grid : {1, 148})
    for (int pat = 0; pat < 15; ++pat) {
      const int reps = 256;
      rate<<<grid, 128, 68 * 1024>>>(pat, reps, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("pattern %d: %s\n", pat, cudaGetErrorString(e)); return 1; }
      const double per_stage = (double)out[1] / reps;
      printf("grid %3d  %-36s issue %7.1f cyc/MMA  complete %7.1f cyc/MMA  (%.0f cyc per rep)\n", grid, names[pat],
             (double)out[0] / out[2], (double)out[1] / out[2], per_stage);
    }
  return 0;
}
