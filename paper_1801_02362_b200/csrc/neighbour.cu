// Neighbour list update (SPEC neighbourlist.maybe_update):
// for each selected row of a distance matrix, the indices of the M smallest
// distances, ties broken by the lower index, written in ascending index order.
//
// One CTA per row.  Distances are mapped to order-preserving 64-bit keys
// (IEEE bit pattern, sign-folded; NaN sorts last), the M-th smallest key is
// found by an 8-pass radix select over shared-memory histograms, and the
// selection {key < K*} plus the first (M - #less) keys equal to K* in index
// order is compacted in index order with block prefix sums.  Each thread owns
// a contiguous index range so "index order" is thread order.
#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int NNT = 256;

__device__ __forceinline__ uint64_t order_key(double d) {
  if (d != d) return ~0ull;  // NaN last
  const uint64_t b = static_cast<uint64_t>(__double_as_longlong(d));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

// exclusive block prefix sum of v (NNT threads); returns the block total in *total
__device__ __forceinline__ int block_excl_scan(int v, int* sh, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  int base = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < NNT / 32; ++w) {
    const int s = sh[w];
    if (w < warp) base += s;
    tot += s;
  }
  *total = tot;
  return base + x - v;
}
}  // namespace

template <typename T>
__global__ void __launch_bounds__(NNT)
topm_kernel(const T* __restrict__ D, int L, int64_t ldd, const int* __restrict__ rows, int M,
            int* __restrict__ idx_out) {
  __shared__ int hist[256];
  __shared__ int sh[NNT / 32];
  __shared__ uint64_t s_prefix;
  __shared__ int s_rank;
  const int row = rows ? rows[blockIdx.x] : blockIdx.x;
  const T* d = D + (int64_t)row * ldd;
  const int per = (L + NNT - 1) / NNT;
  const int i0 = threadIdx.x * per, i1 = min(L, i0 + per);
  // radix select of the M-th smallest key (rank M - 1, 0-based)
  if (threadIdx.x == 0) { s_prefix = 0; s_rank = M - 1; }
  uint64_t mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += NNT) hist[b] = 0;
    __syncthreads();
    const uint64_t prefix = s_prefix;
    for (int i = i0; i < i1; ++i) {
      const uint64_t k = order_key((double)d[i]);
      if ((k & mask) == prefix) atomicAdd(&hist[(k >> shift) & 0xff], 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int r = s_rank, b = 0;
      while (hist[b] <= r) { r -= hist[b]; ++b; }
      s_rank = r;
      s_prefix = prefix | ((uint64_t)b << shift);
    }
    mask |= 0xffull << shift;
    __syncthreads();
  }
  const uint64_t kstar = s_prefix;
  // counts below / equal to K* in this thread's index range
  int nless = 0, neq = 0;
  for (int i = i0; i < i1; ++i) {
    const uint64_t k = order_key((double)d[i]);
    nless += k < kstar;
    neq += k == kstar;
  }
  int tot_less = 0, tot_eq = 0;
  block_excl_scan(nless, sh, &tot_less);
  const int eq_before = block_excl_scan(neq, sh, &tot_eq);
  const int need_eq = M - tot_less;  // >= 1 by construction of K*
  // selected in this range: all "less" + the equal ones whose global equal-rank < need_eq
  int take_eq = min(neq, max(0, need_eq - eq_before));
  int tot_sel = 0;
  int pos = block_excl_scan(nless + take_eq, sh, &tot_sel);
  int* out = idx_out + (int64_t)blockIdx.x * M;
  for (int i = i0; i < i1; ++i) {
    const uint64_t k = order_key((double)d[i]);
    bool sel = k < kstar;
    if (k == kstar && take_eq > 0) {
      sel = true;
      --take_eq;
    }
    if (sel) out[pos++] = i;
  }
}

cudaError_t launch_topm(const void* D, int dtype, int nrows, int L, int64_t ldd, const int* rows, int M, int* idx,
                        cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
  if (dtype == 0)
    topm_kernel<float><<<nrows, NNT, 0, stream>>>((const float*)D, L, ldd, rows, M, idx);
  else
    topm_kernel<double><<<nrows, NNT, 0, stream>>>((const double*)D, L, ldd, rows, M, idx);
  return cudaGetLastError();
}

}  // namespace mc
