// Diagnostic probe: does shared-memory write traffic (what TMA adds) slow the
// tcgen05 kind::f16 MMA stream (M=128, N=144, K=16, operands in smem)?
// One CTA per SM; warp 1 lane 0 issues ITERS MMAs into 3 TMEM accumulators,
// committing every 18 (generic address); warps 4.. (NW of them) store 16 B
// per lane per iteration into a separate 64 KB region until the MMAs finish.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_diag/smem_probe tools/smem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NW, int SW>
__global__ void __launch_bounds__(128 + 32 * 8, 1) probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, dummy;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&dummy)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    done = 0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (144u >> 3 << 17) | (8u << 24);  // F32 acc, F16 A/B
  const uint32_t base = s32(sm);
  auto desc = [](uint32_t a) {
    return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
  };
  unsigned long long t0 = clock64();
  unsigned long long stores = 0;
  if (warp == 1) {
    if ((threadIdx.x & 31) == 0) {
      for (int i = 0; i < iters; ++i) {
        const uint32_t d = tmem + (uint32_t)((i % 3) * 144);
        const uint32_t acc = i >= 3 ? 1u : 0u;
        const uint64_t da = desc(base + (uint32_t)(i % 3) * 16384u + (i / 3 % 2) * 32);
        const uint64_t db = desc(base + 49152u + (i / 3 % 2) * 32);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
        if (i % 18 == 17)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"((unsigned long long)&dummy));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(&bar)));
    }
    __syncwarp();
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
        s32(&bar)));
    if ((threadIdx.x & 31) == 0) done = 1;
  } else if (warp >= 4 && warp < 4 + NW) {
    // store stream into [96 KB, 160 KB): SW bytes-per-lane-iteration throttle via a spin
    const uint32_t p = s32(sm + 98304) + (threadIdx.x - 128) * 16;
    int k = 0;
    while (!done) {
#pragma unroll
      for (int u = 0; u < 16; ++u)
        asm volatile("st.shared.v4.u32 [%0], {%1, %1, %1, %1};" ::"r"(p + u * 32 * 8 * 16), "r"(k) : "memory");
      ++k;
      stores += 16;
      for (int s = 0; s < SW; ++s) __nanosleep(0);
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[2 * blockIdx.x] = t1 - t0;
  if (warp == 4 && (threadIdx.x & 31) == 0) out[2 * blockIdx.x + 1] = stores;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int NW, int SW>
void run(int iters) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* o;
  cudaMalloc(&o, 2 * nsm * sizeof(unsigned long long));
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(probe<NW, SW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<NW, SW><<<nsm, 128 + 32 * 8, smem>>>(iters / 10, o);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<NW, SW><<<nsm, 128 + 32 * 8, smem>>>(iters, o);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[2];
  cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  const double flop = 2.0 * 128 * 144 * 16 * (double)iters * nsm;
  const double bytes_per_clk = NW > 0 ? (double)h[1] * 32 * 16 * NW / (double)h[0] : 0.0;  // stores per lane x 512 B per warp-store
  printf("store warps=%d spin=%d: %.3f ms  %.1f f16 TFLOP/s  smem store %.1f B/clk  err=%s\n", NW, SW, ms,
         flop / ms / 1e9, bytes_per_clk, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}

int main() {
  const int iters = 400000;
  run<0, 0>(iters);
  run<1, 8>(iters);
  run<1, 2>(iters);
  run<1, 0>(iters);
  run<2, 0>(iters);
  run<4, 0>(iters);
  return 0;
}
