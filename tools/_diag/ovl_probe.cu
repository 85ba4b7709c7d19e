// Probe (diagnostic only): cost of tcgen05.mma.kind::i8 chains whose accumulators
// partially overlap (the int8 gradient's stacked-digit pattern: D offsets 0/48/96/144,
// N = 192/144/96/48) vs disjoint and identical accumulators.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ovl_probe tools/_diag/ovl_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ uint64_t desc128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id));
}

// MODE 0: overlapping (0/48/96/144 with N 192/144/96/48); 1: disjoint regions (0/192/336/432);
// 2: same four N but every MMA into its own region AND two tiles alternating; 3: all N=192 same D
template <int MODE, bool RANDOM>
__global__ void __launch_bounds__(640, 1) probe(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar, cbar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) done = 0;
  for (int e = threadIdx.x; e < 64 * 1024 / 4; e += blockDim.x) reinterpret_cast<uint32_t*>(sm)[e] = RANDOM ? (uint32_t)(e * 2654435761u) ^ ((uint32_t)e << 13) * 40503u : 0x01010101u * (e & 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&cbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = slot;
  const unsigned long long t0 = clock64();
  if (threadIdx.x == 32) {
    const uint32_t base = s32(sm);
    const uint64_t a0 = desc128(base), a1 = desc128(base + 32), a2 = desc128(base + 64), a3 = desc128(base + 96);
    const uint64_t b = desc128(base + 16384);
    constexpr uint32_t I192 = idesc_i8(192), I144 = idesc_i8(144), I96 = idesc_i8(96), I48 = idesc_i8(48);
    for (int i = 0; i < iters; ++i) {
      if (MODE == 0 || MODE == 5) {
        mma(t, a0, b, I192); mma(t + 48, a1, b, I144); mma(t + 96, a2, b, I96); mma(t + 144, a3, b, I48);
      } else if (MODE == 4) {
        mma(t, a0, b, I192); mma(t + 48, a1, b, I144); mma(t + 96, a2, b, I96); mma(t + 144, a3, b, I48);
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(reinterpret_cast<uint64_t>(&cbar)));
      } else if (MODE == 1) {
        mma(t, a0, b, I192); mma(t + 192, a1, b, I144); mma(t + 336, a2, b, I96); mma(t + 432, a3, b, I48);
      } else if (MODE == 2) {
        mma(t, a0, b, I192); mma(t + 256, a0, b, I192); mma(t + 48, a1, b, I144); mma(t + 304, a1, b, I144);
        mma(t + 96, a2, b, I96); mma(t + 352, a2, b, I96); mma(t + 144, a3, b, I48); mma(t + 400, a3, b, I48);
      } else {
        mma(t, a0, b, I192); mma(t, a1, b, I192); mma(t, a2, b, I192); mma(t, a3, b, I192);
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(reinterpret_cast<uint64_t>(&bar)));
  }
  if (MODE == 5 && warp >= 4) {
    // 16 warps streaming TMEM loads from the other half of TMEM (like an epilogue)
    const uint32_t src = t + ((uint32_t)((warp & 3) * 32) << 16) + 256;
    uint32_t acc = 0;
    while (!done) {
      uint32_t r[8];
      for (int c = 0; c < 192; c += 8) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(src + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        acc += r[0] ^ r[7];
      }
      __syncwarp();
    }
    if (acc == 12345) cyc[200] = acc;
  }
  if (warp < 4) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
      s32(&bar)));
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; done = 1; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "r"(512));
}

template <int MODE, bool RANDOM = false>
void run(const char* name) {
  unsigned long long* cyc;
  cudaMalloc(&cyc, 256 * 8);
  cudaFuncSetAttribute(probe<MODE, RANDOM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  const int iters = 20000;
  const int nt = MODE == 5 ? 640 : 128;
  probe<MODE, RANDOM><<<148, nt, 70 * 1024>>>(iters / 10, cyc);
  probe<MODE, RANDOM><<<148, nt, 70 * 1024>>>(iters, cyc);
  cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const int per = MODE == 2 ? 8 : 4;
  const double ideal = (MODE == 4 || MODE == 5) ? 240.0 : MODE == 3 ? 4 * 96.0 : (MODE == 2 ? 2 * (96 + 72 + 48 + 24.0) : (96 + 72 + 48 + 24.0));
  printf("%-52s %7.1f clk per group of %d MMAs (N/2 sum %.0f)  err=%s\n", name, (double)c / iters, per, ideal,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  run<0>("overlapping D (0/48/96/144, N 192/144/96/48)");
  run<1>("disjoint D regions, same N");
  run<2>("two tiles interleaved, overlapping within a tile");
  run<3>("same D, N = 192 x 4");
  run<4>("overlapping + tcgen05.commit per group of 4");
  run<5>("overlapping + 16 warps streaming tcgen05.ld");
  run<0, true>("RANDOM operands: overlapping");
  run<3, true>("RANDOM operands: same D, N = 192 x 4");
  return 0;
}
