#include <cstdio>
#include <cuda_runtime.h>
// fp64 tensor-core throughput probe: mma.sync f64 shapes, register operands
template <int SHAPE>
__global__ void k(double* out, int iters) {
  double a[4], b[2], c[8][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 2; ++i) b[i] = threadIdx.x * 2e-3 + i;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) c[j][i] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (SHAPE == 0) {  // m8n8k4: a 1, b 1, c 2
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a[0]), "d"(b[0]));
      } else if (SHAPE == 1) {  // m16n8k4: a 2, b 1, c 4
        asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3]) : "d"(a[0]), "d"(a[1]), "d"(b[0]));
      } else if (SHAPE == 2) {  // m16n8k8: a 4, b 2, c 4
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                     : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) s += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int SHAPE>
void run(int threads, int per_sm = 2) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* o; cudaMalloc(&o, sizeof(double) * nsm * 2 * threads);
  const int iters = 4000;
  k<SHAPE><<<nsm * per_sm, threads>>>(o, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<SHAPE><<<nsm * per_sm, threads>>>(o, iters);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const int mnk[3] = {8 * 8 * 4, 16 * 8 * 4, 16 * 8 * 8};
  double flop = 2.0 * mnk[SHAPE] * 8 * iters * (double)(nsm * per_sm * threads / 32);
  printf("shape %d threads %d x %d/SM: %.1f TFLOP/s fp64  err=%s\n", SHAPE, threads, per_sm, flop / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(o);
}
int main() { run<0>(256); run<0>(256, 1); run<0>(128, 1); run<0>(64, 1); return 0; }
