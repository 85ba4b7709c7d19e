#include <cstdio>
#include <cuda_runtime.h>
// fp64 tensor-core rate with distinct operands per DMMA (6 A x 3 B fragments,
// 18 accumulators: the refine kernel's per-warp tile) vs one shared operand pair
template <int DISTINCT>
__global__ void k(double* out, int iters) {
  double a[6], b[3], c[6][3][2];
#pragma unroll
  for (int i = 0; i < 6; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int j = 0; j < 3; ++j) b[j] = threadIdx.x * 2e-3 + j;
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][j][0]), "+d"(c[i][j][1])
                     : "d"(DISTINCT ? a[i] : a[0]), "d"(DISTINCT ? b[j] : b[0]));
    if (DISTINCT == 3) {  // fresh operands converted from fp32 every step (F2F only)
#pragma unroll
      for (int i = 0; i < 6; ++i) a[i] = (double)__int_as_float(__double2loint(a[i]) ^ it);
#pragma unroll
      for (int j = 0; j < 3; ++j) b[j] = (double)__int_as_float(__double2loint(b[j]) ^ it);
    }
    if (DISTINCT == 2) {  // fresh operands every step (as loaded from shared memory)
#pragma unroll
      for (int i = 0; i < 6; ++i) a[i] = a[i] * 1.0000001 + 1e-9;
#pragma unroll
      for (int j = 0; j < 3; ++j) b[j] = b[j] * 0.9999999 + 1e-9;
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 6; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) s += c[i][j][0] + c[i][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int D>
void run(int threads, int per_sm) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, sizeof(double) * nsm * per_sm * threads);
  const int iters = 2000;
  k<D><<<nsm * per_sm, threads>>>(o, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<D><<<nsm * per_sm, threads>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flop = 2.0 * 256 * 18 * iters * (double)(nsm * per_sm * threads / 32);
  printf("distinct=%d threads %d x %d/SM: %.1f TFLOP/s\n", D, threads, per_sm, flop / ms / 1e9);
  cudaFree(o);
}
int main() { run<1>(256, 2); run<2>(256, 2); run<3>(256, 2); return 0; }
