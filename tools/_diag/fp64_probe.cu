#include <cstdio>
#include <cuda_runtime.h>
template <typename T, int CH>
__global__ void k(T* out, int iters, T a, T b) {
  T x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename T, int CH>
void run(const char* name, int threads) {
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  T* o; cudaMalloc(&o, sizeof(T) * nsm * threads);
  const int iters = 20000;
  k<T, CH><<<nsm, threads>>>(o, 100, (T)0.999, (T)0.001);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<T, CH><<<nsm, threads>>>(o, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma = (double)nsm * threads * iters * CH;
  printf("%s threads/SM=%d chains=%d: %.2f TFMA/s (%.1f TFLOP/s)\n", name, threads, CH, fma / ms / 1e9, 2 * fma / ms / 1e9);
  cudaFree(o);
}
int main() {
  run<double, 8>("f64", 256);
  run<double, 8>("f64", 512);
  run<double, 8>("f64", 1024);
  run<double, 1>("f64", 256);
  run<float, 8>("f32", 1024);
  return 0;
}
