// Probe of tcgen05.mma.kind::i8 with the A operand in TENSOR MEMORY (diagnostic only):
//  (1) layout: A [128 x 32 KS] int8 written to TMEM with tcgen05.st (lane = row, 32-bit
//      column c = bytes 4c..4c+3 of the row's K), B [N x 32 KS] K-major SWIZZLE_32B in
//      shared memory; KS k-steps accumulate (A k-step j at TMEM column ACOL + 8 j); D vs host;
//  (2) issue rate of TS MMAs vs N (stale operands), clocks per MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ts_probe tools/_diag/ts_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ constexpr uint32_t idesc_i8(int n, int m) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ uint64_t desc32(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__device__ __forceinline__ int swz32(int row, int kk, int block_bytes) {
  return (kk >> 5) * block_bytes + (row >> 3) * 256 + (row & 7) * 32 + (((((kk & 31) >> 4) ^ ((row & 7) >> 2)) & 1) << 4) +
         (kk & 15);
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc));
}

constexpr int ACOL = 256;  // A k-steps at TMEM columns 256 + 8 j
template <int N, int KS>
__global__ void __launch_bounds__(128, 1) check_kernel(const int8_t* A, const int8_t* B, int* D) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int K = 32 * KS;
  for (int e = threadIdx.x; e < N * K; e += 128) sm[swz32(e / K, e % K, N * 32)] = (uint8_t)B[e];
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
  const int row = warp * 32 + lane;
  // A row -> TMEM lane `row`, columns ACOL + c: 4 K bytes per 32-bit column (little endian)
  for (int j = 0; j < KS; ++j) {
    uint32_t r[8];
    for (int c = 0; c < 8; ++c) {
      uint32_t v = 0;
      for (int i = 0; i < 4; ++i) v |= (uint32_t)(uint8_t)A[row * K + 32 * j + 4 * c + i] << (8 * i);
      r[c] = v;
    }
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(
                     tmem + ((uint32_t)(warp * 32) << 16) + ACOL + 8 * j),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 32) {
    const uint32_t id = idesc_i8(N, 128);
    for (int j = 0; j < KS; ++j) mma_ts(tmem, tmem + ACOL + 8 * j, desc32(s32(sm) + j * N * 32), id, j ? 1u : 0u);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(reinterpret_cast<uint64_t>(&bar)));
  }
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
      s32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// issue rate: per iteration 4 TS MMAs with N = (4 - p) NB into overlapping accumulators
template <int NB>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < 4 * NB * 32; e += 128) sm[e] = (uint8_t)(e * 7);
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
  if (threadIdx.x == 32) {
    const uint64_t b = desc32(s32(sm));
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int p = 0; p < 4; ++p)
        mma_ts(tmem + p * NB, tmem + 384 + 8 * p, b, idesc_i8((4 - p) * NB, 128), 1u);
      if ((it & 7) == 7)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(
            reinterpret_cast<uint64_t>(&bar)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(reinterpret_cast<uint64_t>(&bar)));
    const unsigned long long t1 = clock64();
    cyc[blockIdx.x * 2] = t1 - t0;
  }
  __syncthreads();
  if (threadIdx.x == 32) {
    // wait for every commit: the barrier counts iters / 8 + 1 phases; poll the last one
    unsigned long long t0 = clock64();
    asm volatile("tcgen05.fence::after_thread_sync;");
    cyc[blockIdx.x * 2 + 1] = t0;
  }
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, int KS>
int run_check() {
  const int K = 32 * KS;
  int8_t *A, *B;
  int* D;
  cudaMallocManaged(&A, 128 * K);
  cudaMallocManaged(&B, N * K);
  cudaMallocManaged(&D, 128 * N * 4);
  srand(1234 + N);
  for (int i = 0; i < 128 * K; ++i) A[i] = (int8_t)(rand() % 256 - 128);
  for (int i = 0; i < N * K; ++i) B[i] = (int8_t)(rand() % 256 - 128);
  cudaFuncSetAttribute(check_kernel<N, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, N * K + 1024);
  check_kernel<N, KS><<<1, 128, N * K + 1024>>>(A, B, D);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("check N=%d KS=%d: %s\n", N, KS, cudaGetErrorString(e));
    return 1;
  }
  long bad = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < N; ++c) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)A[r * K + k] * B[c * K + k];
      if (s != D[r * N + c]) {
        if (bad < 4) printf("  mismatch r=%d c=%d got %d want %ld\n", r, c, D[r * N + c], s);
        ++bad;
      }
    }
  printf("check TS kind::i8 N=%d KS=%d: %s (%ld bad)\n", N, KS, bad ? "FAIL" : "ok", bad);
  cudaFree(A);
  cudaFree(B);
  cudaFree(D);
  return bad != 0;
}

template <int NB>
void run_rate() {
  unsigned long long* c;
  cudaMallocManaged(&c, 2 * 148 * 8);
  const int iters = 4096;
  cudaFuncSetAttribute(rate_kernel<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * NB * 32 + 1024);
  rate_kernel<NB><<<148, 128, 4 * NB * 32 + 1024>>>(iters, c);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  rate_kernel<NB><<<148, 128, 4 * NB * 32 + 1024>>>(iters, c);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double macs = 148.0 * iters * 128.0 * 32.0 * (10.0 * NB);  // (4+3+2+1) NB columns
  printf("rate TS stacked NB=%d: %.3f ms, %.1f int8 TOPS, issue clk/iter %.1f\n", NB, ms, 2.0 * macs / ms / 1e9,
         (double)c[0] / iters);
  cudaFree(c);
}

int main() {
  int bad = 0;
  bad += run_check<64, 1>();
  bad += run_check<64, 4>();
  bad += run_check<128, 2>();
  bad += run_check<32, 3>();
  run_rate<32>();
  run_rate<48>();
  run_rate<64>();
  return bad;
}
