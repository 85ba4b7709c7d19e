// Probe of tcgen05.mma.kind::i8 on sm_100a (diagnostic only):
//  (1) correctness: one 128 x N x 128 int8 GEMM (4 MMAs of K = 32 inside a
//      SWIZZLE_128B K-major tile, signed s8 x s8 -> s32 in TMEM) vs the host;
//  (2) issue throughput vs N (stale operands), as executed int8 TOPS.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o i8_probe tools/_diag/i8_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__host__ __device__ constexpr uint32_t idesc_i8(int n, int m, int sa, int sb) {
  return (2u << 4) | ((uint32_t)sa << 7) | ((uint32_t)sb << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}

// byte offset of (row, k) in a K-major SWIZZLE_128B tile of 128-byte rows
__device__ __forceinline__ int sw128_off(int row, int k) {
  return (row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 4) ^ (row & 7)) & 7) << 4) + (k & 15);
}

template <int N>
__global__ void __launch_bounds__(128, 1) check_kernel(const int8_t* A, const int8_t* B, int* D, int sa, int sb) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* sA = sm;
  uint8_t* sB = sm + 128 * 128;
  for (int e = threadIdx.x; e < 128 * 128; e += 128) sA[sw128_off(e / 128, e % 128)] = (uint8_t)A[e];
  for (int e = threadIdx.x; e < N * 128; e += 128) sB[sw128_off(e / 128, e % 128)] = (uint8_t)B[e];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&slot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (threadIdx.x == 32) {
    const uint32_t id = idesc_i8(N, 128, sa, sb);
    for (int k = 0; k < 4; ++k) {
      const uint64_t da = desc_sw128(s32(sA) + 32 * k), db = desc_sw128(s32(sB) + 32 * k);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                   "l"(da), "l"(db), "r"(id), "r"(k ? 1u : 0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(reinterpret_cast<uint64_t>(&bar)));
  }
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
      s32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = warp * 32 + lane;
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) D[row * N + c + i] = (int)r[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int N, int KIND = 0, int M = 128>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, int nacc, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < 96 * 1024 / 4; e += 128) reinterpret_cast<uint32_t*>(sm)[e] = 0x01010101u * (e & 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(&slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const unsigned long long t0 = clock64();
  if (threadIdx.x == 32) {
    const uint32_t id = KIND == 0 ? idesc_i8(N, M, 1, 1)
                                  : ((1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24));
    const uint32_t base = s32(sm);
    uint64_t da[4], db[4];
    uint32_t dd[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      da[j] = desc_sw128(base + (uint32_t)j * 16384u + 32u * j);
      db[j] = desc_sw128(base + 65536u + 32u * j);
      dd[j] = tmem + (uint32_t)((j % nacc) * N);
    }
    for (int i = 0; i < iters; i += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (KIND == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dd[j]),
                       "l"(da[j]), "l"(db[j]), "r"(id), "r"(1u));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dd[j]),
                       "l"(da[j]), "l"(db[j]), "r"(id), "r"(1u));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(reinterpret_cast<uint64_t>(&bar)));
  }
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
      s32(&bar)));
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N>
int check(int sa, int sb) {
  const int K = 128;
  int8_t *hA = (int8_t*)malloc(128 * K), *hB = (int8_t*)malloc(N * K);
  srand(1234 + N);
  for (int i = 0; i < 128 * K; ++i) hA[i] = (int8_t)((rand() & 255) - 128);
  for (int i = 0; i < N * K; ++i) hB[i] = (int8_t)((rand() & 255) - 128);
  int8_t *dA, *dB;
  int* dD;
  cudaMalloc(&dA, 128 * K);
  cudaMalloc(&dB, N * K);
  cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, hA, 128 * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(check_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  check_kernel<N><<<1, 128, 100 * 1024>>>(dA, dB, dD, sa, sb);
  cudaError_t e = cudaDeviceSynchronize();
  int* hD = (int*)malloc(128 * N * 4);
  cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < N; ++n) {
      long ref = 0;
      for (int k = 0; k < K; ++k) {
        const int a = sa ? (int)hA[m * K + k] : (int)(uint8_t)hA[m * K + k];
        const int b = sb ? (int)hB[n * K + k] : (int)(uint8_t)hB[n * K + k];
        ref += (long)a * b;
      }
      if (ref != hD[m * N + n]) {
        if (bad < 5) printf("  mismatch m=%d n=%d ref=%ld got=%d\n", m, n, ref, hD[m * N + n]);
        ++bad;
      }
    }
  printf("check N=%d sa=%d sb=%d: %s, %ld mismatches of %d\n", N, sa, sb, cudaGetErrorString(e), bad, 128 * N);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  free(hA); free(hB); free(hD);
  return bad != 0 || e != cudaSuccess;
}

template <int N, int KIND = 0, int M = 128>
void rate(int iters, int nacc) {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  cudaMalloc(&cyc, nsm * 8);
  cudaFuncSetAttribute(rate_kernel<N, KIND, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  rate_kernel<N, KIND, M><<<nsm, 128, 100 * 1024>>>(iters / 10, nacc, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  rate_kernel<N, KIND, M><<<nsm, 128, 100 * 1024>>>(iters, nacc, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  const int KK = KIND == 0 ? 32 : 16;
  const double ops = 2.0 * M * N * KK * (double)iters * nsm;
  printf("rate %s M=%d N=%3d nacc=%d: %.3f ms  %.1f TOPS  %.1f cycles/MMA  %.0f MAC/clk/SM  err=%s\n",
         KIND == 0 ? "i8 " : "f16", M, N, nacc, ms,
         ops / ms / 1e9, (double)c / iters, (double)M * N * KK * iters / (double)c, cudaGetErrorString(cudaGetLastError()));
  cudaFree(cyc);
}

int main() {
  int bad = 0;
  bad |= check<48>(1, 1);
  bad |= check<144>(1, 1);
  bad |= check<192>(1, 1);
  bad |= check<256>(1, 1);
  bad |= check<48>(1, 0);
  bad |= check<48>(0, 1);
  const int iters = 200000;
  rate<16>(iters, 4);
  rate<32>(iters, 4);
  rate<48>(iters, 4);
  rate<64>(iters, 4);
  rate<96>(iters, 4);
  rate<128>(iters, 3);
  rate<144>(iters, 3);
  rate<192>(iters, 2);
  rate<256>(iters, 2);
  rate<256>(iters, 1);
  rate<48>(iters, 1);
  rate<48>(iters, 8);
  rate<48, 0, 64>(iters, 4);
  rate<256, 0, 64>(iters, 2);
  rate<48, 1>(iters, 4);
  rate<96, 1>(iters, 4);
  rate<144, 1>(iters, 3);
  rate<256, 1>(iters, 2);
  return bad;
}
