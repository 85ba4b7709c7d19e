#include <cstdio>
#include <cuda_runtime.h>
// DMMA rate with the gradient kernel's per-k-step instruction mix: 6 A fragments
// (LDS.64), NJ B fragments (LDS.32 + F2F + DADD), 6 x NJ DMMA, operands in shared memory.
template <int NJ, int CENTER>
__global__ void __launch_bounds__(512, 1) k(double* out, int iters) {
  extern __shared__ double dsm[];
  double* sA = dsm;
  float* sB = reinterpret_cast<float*>(dsm + 48 * 292);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gq = lane >> 2, tq = lane & 3;
  for (int i = threadIdx.x; i < 48 * 292; i += blockDim.x) sA[i] = i * 1e-6;
  for (int i = threadIdx.x; i < 24 * 776; i += blockDim.x) sB[i] = i * 1e-5f;
  __syncthreads();
  double c[6][NJ][2];
#pragma unroll
  for (int m = 0; m < 6; ++m)
#pragma unroll
    for (int j = 0; j < NJ; ++j) c[m][j][0] = c[m][j][1] = 0.0;
  const double lcg = 0.1;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 6; ++s) {
      const int kk = (it & 7) * 24 + s * 4 + tq;
      double a[6], b[NJ];
#pragma unroll
      for (int m = 0; m < 6; ++m) a[m] = sA[(m * 8 + gq) * 292 + kk];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const float v = sB[((s * 4 + tq) / 3) * 776 + (warp * 8 * NJ + gq) * 3 + (s * 4 + tq) % 3 + j * 24];
        b[j] = CENTER ? (double)v - lcg : (double)v;
      }
#pragma unroll
      for (int m = 0; m < 6; ++m)
#pragma unroll
        for (int j = 0; j < NJ; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                       : "+d"(c[m][j][0]), "+d"(c[m][j][1]) : "d"(a[m]), "d"(b[j]));
    }
  }
  double sum = 0;
#pragma unroll
  for (int m = 0; m < 6; ++m)
#pragma unroll
    for (int j = 0; j < NJ; ++j) sum += c[m][j][0] + c[m][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = sum;
}
template <int NJ, int CENTER>
void run(int threads) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, sizeof(double) * nsm * threads);
  const int iters = 400;
  const int smem = 48 * 292 * 8 + 24 * 776 * 4;
  cudaFuncSetAttribute(k<NJ, CENTER>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<NJ, CENTER><<<nsm, threads, smem>>>(o, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NJ, CENTER><<<nsm, threads, smem>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flop = 2.0 * 256 * 6 * NJ * 6 * iters * (double)(nsm * threads / 32);
  printf("NJ=%d center=%d threads %d: %.1f TFLOP/s  err=%s\n", NJ, CENTER, threads, flop / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}
int main() { run<2, 1>(512); run<2, 0>(512); run<4, 1>(256); run<4, 0>(256); return 0; }
