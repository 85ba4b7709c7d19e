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

// Fast path: the row's order keys live in shared memory (32-bit keys for fp32
// input, 64-bit for fp64), histogram updates are warp-aggregated
// (__match_any_sync: one shared atomic per distinct digit per warp, so a
// skewed digit distribution does not serialise), and the index-ordered
// compaction runs in rounds of NNT consecutive indices with ballots.
template <typename T, typename K>
__global__ void __launch_bounds__(NNT)
topm_smem_kernel(const T* __restrict__ D, int L, int64_t ldd, const int* __restrict__ rows, int M,
                 int* __restrict__ idx_out) {
  extern __shared__ __align__(16) unsigned char tsm[];
  K* keys = reinterpret_cast<K*>(tsm);
  __shared__ int hist[256];
  __shared__ int wl[NNT / 32], we[NNT / 32];
  __shared__ K s_prefix;
  __shared__ int s_rank;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int row = rows ? rows[blockIdx.x] : blockIdx.x;
  const T* d = D + (int64_t)row * ldd;
  for (int i = threadIdx.x; i < L; i += NNT) {
    if (sizeof(K) == 4) {
      const float v = (float)d[i];
      const uint32_t b = __float_as_uint(v);
      keys[i] = (K)(v != v ? 0xffffffffu : ((b >> 31) ? ~b : (b | 0x80000000u)));
    } else {
      keys[i] = (K)order_key((double)d[i]);
    }
  }
  if (threadIdx.x == 0) { s_prefix = 0; s_rank = M - 1; }
  K mask = 0;
  for (int shift = 8 * (int)sizeof(K) - 8; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += NNT) hist[b] = 0;
    __syncthreads();
    const K prefix = s_prefix;
    for (int i0 = 0; i0 < L; i0 += NNT) {
      const int i = i0 + threadIdx.x;
      const bool live = i < L && (keys[i] & mask) == prefix;
      const unsigned act = __ballot_sync(0xffffffffu, live);
      if (live) {
        const int dg = (int)((keys[i] >> shift) & 0xff);
        const unsigned grp = __match_any_sync(act, dg);
        if (lane == __ffs(grp) - 1) atomicAdd(&hist[dg], __popc(grp));
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int r = s_rank, b = 0;
      while (hist[b] <= r) { r -= hist[b]; ++b; }
      s_rank = r;
      s_prefix = prefix | ((K)b << shift);
    }
    mask |= (K)0xff << shift;
    __syncthreads();
  }
  const K kstar = s_prefix;
  // #keys < K*: the rank of K* minus the equal keys below it in the final bucket
  int nl = 0;
  for (int i = threadIdx.x; i < L; i += NNT) nl += keys[i] < kstar;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nl += __shfl_xor_sync(0xffffffffu, nl, o);
  if (lane == 0) wl[warp] = nl;
  __syncthreads();
  int tot_less = 0;
#pragma unroll
  for (int w = 0; w < NNT / 32; ++w) tot_less += wl[w];
  const int need_eq = M - tot_less;
  int eq_taken = 0, out_pos = 0;
  int* out = idx_out + (int64_t)blockIdx.x * M;
  for (int i0 = 0; i0 < L; i0 += NNT) {
    const int i = i0 + threadIdx.x;
    const K k = i < L ? keys[i] : (K)~(K)0;
    const bool less = i < L && k < kstar, eq = i < L && k == kstar;
    const unsigned bl = __ballot_sync(0xffffffffu, less), be = __ballot_sync(0xffffffffu, eq);
    __syncthreads();
    if (lane == 0) { wl[warp] = __popc(bl); we[warp] = __popc(be); }
    __syncthreads();
    int lbefore = 0, ebefore = 0, lsum = 0, esum = 0;
#pragma unroll
    for (int w = 0; w < NNT / 32; ++w) {
      if (w < warp) { lbefore += wl[w]; ebefore += we[w]; }
      lsum += wl[w];
      esum += we[w];
    }
    const unsigned below = (1u << lane) - 1u;
    const int erank = eq_taken + ebefore + __popc(be & below);  // equal keys before i (index order)
    const bool take_eq = eq && erank < need_eq;
    const int etaken_before = min(max(need_eq - eq_taken, 0), ebefore + __popc(be & below));
    if (less || take_eq) out[out_pos + lbefore + __popc(bl & below) + etaken_before] = i;
    out_pos += lsum + min(max(need_eq - eq_taken, 0), esum);
    eq_taken += esum;
  }
}

cudaError_t launch_topm(const void* D, int dtype, int nrows, int L, int64_t ldd, const int* rows, int M, int* idx,
                        cudaStream_t stream) {
  if (nrows <= 0) return cudaSuccess;
  const size_t ksz = dtype == 0 ? 4 : 8;
  const size_t smem = ksz * (size_t)L;
  if (smem <= 200 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(topm_smem_kernel<float, uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(topm_smem_kernel<double, uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      attr = true;
    }
    if (dtype == 0)
      topm_smem_kernel<float, uint32_t><<<nrows, NNT, smem, stream>>>((const float*)D, L, ldd, rows, M, idx);
    else
      topm_smem_kernel<double, uint64_t><<<nrows, NNT, smem, stream>>>((const double*)D, L, ldd, rows, M, idx);
    return cudaGetLastError();
  }
  // very long rows: keys re-read from global memory each pass
  if (dtype == 0)
    topm_kernel<float><<<nrows, NNT, 0, stream>>>((const float*)D, L, ldd, rows, M, idx);
  else
    topm_kernel<double><<<nrows, NNT, 0, stream>>>((const double*)D, L, ldd, rows, M, idx);
  return cudaGetLastError();
}

}  // namespace mc
