// Probe (diagnostic only): 2-D TMA of a UINT8 tensor with SWIZZLE_64B / 128B boxes
// of 128 rows, checked byte by byte against the swizzle formula the int8 gradient
// kernel uses for its hand-written operand (grad_i8.cu swz64).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_u8_probe tools/_diag/tma_u8_probe.cu -lcuda
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, int c0, int c1, int nbytes, uint8_t* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(&bar)), "r"(nbytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            s32(sm)),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(c1), "r"(s32(&bar))
        : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n\t}" ::"r"(
      s32(&bar)));
  for (int e = threadIdx.x; e < nbytes; e += blockDim.x) out[e] = sm[e];
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int rows = 1024, cols = 768;
  uint8_t* h = (uint8_t*)malloc(rows * cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) h[r * cols + c] = (uint8_t)(r * 7 + c * 13);
  uint8_t *d, *o;
  cudaMalloc(&d, rows * cols);
  cudaMalloc(&o, 1 << 16);
  cudaMemcpy(d, h, rows * cols, cudaMemcpyHostToDevice);
  int bad_total = 0;
  for (int sw : {32, 64, 128}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols};
    cuuint32_t box[2] = {(cuuint32_t)sw, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult cr = enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      sw == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : sw == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int c0 = (3 * 37) & ~15, c1 = 256;  // the K start must be 16-byte aligned (an unaligned one faults)
    const int nbytes = sw * 128;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    probe<<<1, 128, 40000>>>(map, c0, c1, nbytes, o);
    cudaError_t e = cudaDeviceSynchronize();
    uint8_t* got = (uint8_t*)malloc(nbytes);
    cudaMemcpy(got, o, nbytes, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < sw; ++c) {
        int off;
        if (sw == 32)
          off = (r >> 3) * 256 + (r & 7) * 32 + ((((c >> 4) ^ ((r & 7) >> 2)) & 1) << 4) + (c & 15);
        else if (sw == 64)
          off = (r >> 3) * 512 + (r & 7) * 64 + ((((c >> 4) ^ ((r & 7) >> 1)) & 3) << 4) + (c & 15);
        else
          off = (r >> 3) * 1024 + (r & 7) * 128 + ((((c >> 4) ^ (r & 7)) & 7) << 4) + (c & 15);
        const int gc = c0 + c;
        const uint8_t ref = gc < cols ? h[(c1 + r) * cols + gc] : 0;
        if (got[off] != ref) {
          if (bad < 4) printf("  sw%d r=%d c=%d got %d ref %d\n", sw, r, c, got[off], ref);
          ++bad;
        }
      }
    printf("SWIZZLE_%dB encode=%d kernel=%s mismatches=%d of %d\n", sw, (int)cr, cudaGetErrorString(e), bad, nbytes);
    bad_total += bad + (e != cudaSuccess);
    free(got);
  }
  return bad_total != 0;
}
