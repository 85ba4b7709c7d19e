// Micro-probe of tcgen05.mma.kind::tf32 issue throughput vs the N dimension
// (M = 128, K = 8, cta_group::1, operands: stale shared memory).  One CTA per
// SM, one elected thread issues `iters` MMAs into one or more TMEM
// accumulators; prints executed TF32 TFLOP/s per N.  Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe tools/mma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int N, int NACC, int ROT, int COMMIT>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, dummy;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&dummy)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  const uint32_t base = s32(sm);
  auto desc = [](uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(512 >> 4) << 32) | (1ull << 46) | (4ull << 61);
  };
  const uint64_t desc0a = desc(base), desc0b = desc(base + 16384);
  unsigned long long t0 = clock64();
  if (COMMIT < 0 && (warp == 1 || warp == 2)) {
    // two issuer threads alternate groups of -COMMIT MMAs, each committing its own group;
    // issue order is kept by a shared counter (group g by warp 1 + (g & 1))
    __shared__ volatile int issued;
    if (threadIdx.x == 32) issued = 0;
    __syncwarp();
    const int G = -COMMIT;
    const int me = warp - 1;
    if ((threadIdx.x & 31) == 0) {
      for (int g = me; g * G < iters; g += 2) {
        while (issued < g) {
        }
        for (int j = 0; j < G; ++j) {
          const int i = g * G + j;
          const uint32_t d = tmem + (uint32_t)((i % NACC) * N);
          const uint32_t acc = i >= NACC ? 1u : 0u;
          const uint64_t da = desc(base + (uint32_t)(i % 6) * 8192u);
          const uint64_t db = desc(base + 49152u + (uint32_t)(i % 2) * 9216u);
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        __threadfence_block();
        issued = g + 1;
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            s32(&dummy)));
      }
      if (me == 0) {
        while (issued * G < iters) {
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            s32(&bar)));
      }
    }
    __syncwarp();
    if (me == 0)
      asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
          s32(&bar)));
  } else if (warp == 1) {
    if ((threadIdx.x & 31) == 0) {
      for (int i = 0; i < iters; ++i) {
        const uint32_t d = tmem + (uint32_t)((i % NACC) * N);
        const uint32_t acc = i >= NACC ? 1u : 0u;
        const uint64_t da = ROT ? desc(base + (uint32_t)(i % 6) * 8192u) : desc0a;
        const uint64_t db = ROT ? desc(base + 49152u + (uint32_t)(i % 2) * 9216u) : desc0b;
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
        if (COMMIT > 0 && (i % COMMIT) == COMMIT - 1)  // a commit every COMMIT MMAs (no wait)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              s32(&dummy)));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&bar)));
    }
    __syncwarp();
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
        s32(&bar)));
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, int NACC, int ROT = 0, int COMMIT = 0>
void run(int iters) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, nsm * sizeof(unsigned long long));
  const int smem = 80 * 1024;
  cudaFuncSetAttribute(probe<N, NACC, ROT, COMMIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, NACC, ROT, COMMIT><<<nsm, 128, smem>>>(iters / 10, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<N, NACC, ROT, COMMIT><<<nsm, 128, smem>>>(iters, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c = 0;
  cudaMemcpy(&c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  const double flop = 2.0 * 128 * N * 8 * (double)iters * nsm;
  printf("N=%3d acc=%d rot=%d commit=%d: %.3f ms  %.1f TF32 TFLOP/s  %.1f cycles/MMA  err=%s\n", N, NACC, ROT, COMMIT, ms, flop / ms / 1e9,
         (double)c / iters, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  const int iters = 200000;
  run<96, 3>(iters);
  run<144, 3>(iters);
  run<144, 1>(iters);
  run<192, 2>(iters);
  run<240, 2>(iters);
  run<256, 2>(iters);
  run<256, 1>(iters);
  run<144, 3, 1>(iters);
  run<240, 2, 1>(iters);
  run<144, 3, 1, 18>(iters);
  run<144, 3, 1, 36>(iters);
  run<144, 3, 1, 9>(iters);
  run<144, 3, 1, -18>(iters);
  run<144, 3, 1, -9>(iters);
  return 0;
}
