// Metric pruning of the screening GEMM (fp32-coordinate path, config 4 shape).
//
// The optimally superimposed weighted RMSD d = sqrt(MSD) is a (pseudo)metric
// on centred structures (the same rotation applies to every atom, the w-norm is
// rotation invariant), so for any frame t, landmark l and coarse landmark c
//     d(t, l) >= d(c, l) - d(t, c).
// A one-term screen against a coarse subset C of the landmarks gives
// d(t, c) <= dhi = sqrt(Dc + e_tc) (e_tc: the rigorous one-term error bound),
// and the exact coarse-to-landmark distances give, per 48-landmark tile tau,
// mind[c, tau] = min_{l in tau} d(c, l).  With the K nearest coarse landmarks
//     LB(t, tau) = max_c max(0, mind[c, tau] - dhi(t, c))^2 <= min_{l in tau} D(t, l)
// and Dmin_ub(t) = min_c (Dc + e_tc) >= min_l D(t, l).  A tile with
// LB > Dmin_ub + cutoff / lambda holds no landmark of weight >= e^-cutoff, so
// it is dropped: identical significant sets, truncated mass below the existing
// window bound.  The other side of the triangle, d(t, l) >= d(t, c) - d(c, l),
// with dlo = sqrt(max(0, Dc - e_tc)) and maxd[c, tau] = max_{l in tau} d(c, l)
// over the coarse landmarks within one tile of tau, gives
//     LB2(t, tau) = max_c max(0, dlo(t, c) - maxd[c, tau])^2,
// which prunes the far side of the path for every frame (a frame far from the
// coarse landmarks around a tile is far from the whole tile); config 4: mean
// hull 34.7 -> 3.7 tiles, screened tiles 25% -> 5.7% (tools/_diag/prune2.py).  prune_plan_kernel emits each frame's admissible tile hull
// [lo, hi); frames are then sorted by hull start (wide hulls first), banded
// into 128-frame tiles, and band_tiles_kernel lists the (frame tile, landmark
// tile) pairs the tensor-core kernel computes.
#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int PNT = 256;  // 8 frames (warps) per CTA
constexpr int KNEAR_MAX = 8;
}  // namespace

__global__ void __launch_bounds__(PNT)
prune_plan_kernel(const float* __restrict__ Dc, int T, int C, int64_t lddc, const double* __restrict__ fnorm,
                  const double* __restrict__ cnorm, const double* __restrict__ frnorm,
                  const double* __restrict__ crnorm, double c_unit, const float* __restrict__ mind,
                  const float* __restrict__ maxd, int cstride, int ntl, double thr, int knear, int wide,
                  const double* __restrict__ dub_in, double* __restrict__ dub_out, int* __restrict__ hull_lo,
                  int* __restrict__ hull_hi, int* __restrict__ key) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * (PNT / 32) + (threadIdx.x >> 5);
  if (t >= T) return;
  const float* row = Dc + (int64_t)t * lddc;
  // rigorous one-term error of the pair (t, c): legacy c_unit ||x|| ||c||, or with the
  // rounding-residual norms 5 (r_t |c| + |x| r_c + r_t r_c) + c_unit (|x| + r_t)(|c| + r_c)
  // + 1e-6 |x| |c|  (c_unit = 5 n 2^-27: the fp32 accumulation term)
  const double p1 = fnorm[t], p2 = frnorm ? frnorm[t] : 0.0;
  auto ebound = [&](int c) -> double {
    if (!frnorm) return c_unit * p1 * cnorm[c];
    const double q1 = cnorm[c], q2 = crnorm[c];
    return 5.0 * (p2 * q1 + p1 * q2 + p2 * q2) + c_unit * (p1 + p2) * (q1 + q2) + 1e-6 * p1 * q1;
  };
  // D_min upper bound over all landmarks (the coarse ones are a subset)
  double dub = INFINITY;
  for (int c = lane; c < C; c += 32) dub = fmin(dub, (double)row[c] + ebound(c));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dub = fmin(dub, __shfl_xor_sync(0xffffffffu, dub, o));
  // landmark-sharded evaluation: pass 1 writes this shard's bound (dub_out, no hulls),
  // the host all-reduces the minimum, pass 2 prunes against it (dub_in) -- a shard
  // far from the frame then admits no tile at all
  if (dub_out && lane == 0) dub_out[t] = dub;
  if (!hull_lo) return;
  if (dub_in) dub = fmin(dub, dub_in[t]);
  // the knear nearest coarse landmarks (by estimate), with their distance upper bounds
  int near[KNEAR_MAX];
  double dhi[KNEAR_MAX];
  unsigned taken_lo = 0;  // per lane: which of its coarse entries are already chosen (bit j: c = lane + 32 j)
  for (int k = 0; k < knear; ++k) {
    float best = INFINITY;
    int bc = 0x7fffffff;
    for (int j = 0, c = lane; c < C; ++j, c += 32) {
      if (j < 32 && ((taken_lo >> j) & 1u)) continue;
      const float v = row[c];
      if (v < best || (v == best && c < bc)) { best = v; bc = c; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ob < best || (ob == best && oc < bc)) { best = ob; bc = oc; }
    }
    near[k] = bc;
    dhi[k] = bc < C ? sqrt(fmax(0.0, (double)row[bc] + ebound(bc))) : INFINITY;
    if (bc < C && (bc & 31) == lane && (bc >> 5) < 32) taken_lo |= 1u << (bc >> 5);
  }
  // admissible hull of landmark tiles
  const double lim = dub + thr;
  int lo = ntl, hi = -1;
  for (int tau = lane; tau < ntl; tau += 32) {
    double lb = 0.0;
    for (int k = 0; k < knear; ++k) {
      if (near[k] >= C) continue;
      const double g = fmax(0.0, (double)mind[(int64_t)near[k] * ntl + tau] - dhi[k]);
      lb = fmax(lb, g * g);
    }
    if (maxd) {
      // far side: d(t,l) >= d_lo(t,c) - maxd[c,tau] for the coarse landmarks within one
      // tile of tau (a frame far from them is far from the whole tile)
      const int c0 = max(0, (tau * 48 - 48 + cstride - 1) / cstride);
      const int c1 = min(C - 1, (tau * 48 + 95) / cstride);
      for (int c = c0; c <= c1; ++c) {
        const double dlo = sqrt(fmax(0.0, (double)row[c] - ebound(c)));
        const double g = fmax(0.0, dlo - (double)maxd[(int64_t)c * ntl + tau]);
        lb = fmax(lb, g * g);
      }
    }
    if (lb <= lim) { lo = min(lo, tau); hi = max(hi, tau); }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if (lane == 0) {
    if (hi < lo) {
      if (dub_in) {
        // sharded: no tile of this shard can hold a significant landmark; the empty
        // hull [ntl, 0) neither widens a band's union nor its row range, and sorts last
        hull_lo[t] = ntl;
        hull_hi[t] = 0;
        key[t] = ntl;
        return;
      }
      lo = 0;  // cannot happen unsharded (the nearest coarse tile is admissible); stay safe
      hi = ntl - 1;
    }
    hull_lo[t] = lo;
    hull_hi[t] = hi + 1;
    // sort key: frames whose hull covers >= `wide` tiles first (they need almost
    // everything), the rest by hull start so 128-frame bands share landmark tiles
    key[t] = (hi + 1 - lo >= wide) ? 0 : 1 + lo;
  }
}

// Per 128-frame band of the sorted order: union of the member hulls, the
// band's landmark index range for the candidate scan, and the (tm, tl) list.
// One CTA; bands processed in chunks of blockDim with a running offset.
__global__ void __launch_bounds__(1024)
band_tiles_kernel(const int* __restrict__ perm, int T, const int* __restrict__ hull_lo,
                  const int* __restrict__ hull_hi, int BM, int BL, int L, int* __restrict__ tlist,
                  int* __restrict__ nlist, int* __restrict__ row_lo, int* __restrict__ row_hi) {
  __shared__ int wsum[32];
  __shared__ int s_base;
  const int ntm = (T + BM - 1) / BM;
  if (threadIdx.x == 0) s_base = 0;
  __syncthreads();
  for (int tm0 = 0; tm0 < ntm; tm0 += blockDim.x) {
    const int tm = tm0 + threadIdx.x;
    int lo = 0x7fffffff, hi = -1;
    if (tm < ntm) {
      for (int r = tm * BM; r < min(T, tm * BM + BM); ++r) {
        const int t = perm[r];
        lo = min(lo, hull_lo[t]);
        hi = max(hi, hull_hi[t]);
      }
    }
    const int cnt = tm < ntm ? max(0, hi - lo) : 0;
    // block exclusive scan of cnt
    int x = cnt;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      if (w < warp) before += wsum[w];
      total += wsum[w];
    }
    const int base = s_base;
    const int off = base + before + x - cnt;
    for (int k = 0; k < cnt; ++k) {
      tlist[2 * (off + k)] = tm;
      tlist[2 * (off + k) + 1] = lo + k;
    }
    if (tm < ntm)
      for (int r = tm * BM; r < min(T, tm * BM + BM); ++r) {
        row_lo[r] = cnt ? lo * BL : 0;
        row_hi[r] = cnt ? min(L, hi * BL) : 0;
      }
    __syncthreads();
    if (threadIdx.x == 0) s_base = base + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) *nlist = s_base;
}

template <typename E>
__global__ void gather_rows_kernel(const E* __restrict__ src, int64_t rowlen, const int* __restrict__ idx, int rows,
                                   E* __restrict__ dst) {
  const int r = blockIdx.y;
  for (int64_t rr = r; rr < rows; rr += gridDim.y) {
    const E* s = src + (int64_t)idx[rr] * rowlen;
    E* d = dst + rr * rowlen;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < rowlen; e += (int64_t)gridDim.x * blockDim.x)
      d[e] = s[e];
  }
}

cudaError_t launch_prune_plan(const float* Dc, int T, int C, int64_t lddc, const double* fnorm, const double* cnorm,
                              const double* frnorm, const double* crnorm, double c_unit, const float* mind, const float* maxd, int cstride, int ntl, double thr,
                              int knear, int wide, const double* dub_in, double* dub_out, int* hull_lo, int* hull_hi,
                              int* key, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  if (knear > KNEAR_MAX) knear = KNEAR_MAX;
  prune_plan_kernel<<<(T + PNT / 32 - 1) / (PNT / 32), PNT, 0, stream>>>(
      Dc, T, C, lddc, fnorm, cnorm, frnorm, crnorm, c_unit, mind, maxd, cstride, ntl, thr, knear, wide, dub_in,
      dub_out, hull_lo, hull_hi, key);
  return cudaGetLastError();
}

cudaError_t launch_band_tiles(const int* perm, int T, const int* hull_lo, const int* hull_hi, int BM, int BL, int L,
                              int* tlist, int* nlist, int* row_lo, int* row_hi, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  band_tiles_kernel<<<1, 1024, 0, stream>>>(perm, T, hull_lo, hull_hi, BM, BL, L, tlist, nlist, row_lo, row_hi);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const void* src, int esz, int64_t rowlen, const int* idx, int rows, void* dst,
                               cudaStream_t stream) {
  if (rows <= 0 || rowlen <= 0) return cudaSuccess;
  // whole rows as 16-byte vectors when possible
  if ((rowlen * esz) % 16 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 &&
      (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
    const int64_t vl = rowlen * esz / 16;
    const dim3 grid((unsigned)((vl + 255) / 256 < 64 ? (vl + 255) / 256 : 64), (unsigned)(rows < 65535 ? rows : 65535));
    gather_rows_kernel<float4><<<grid, 256, 0, stream>>>((const float4*)src, vl, idx, rows, (float4*)dst);
  } else if (esz == 4) {
    const dim3 grid((unsigned)((rowlen + 255) / 256 < 64 ? (rowlen + 255) / 256 : 64),
                    (unsigned)(rows < 65535 ? rows : 65535));
    gather_rows_kernel<float><<<grid, 256, 0, stream>>>((const float*)src, rowlen, idx, rows, (float*)dst);
  } else {
    const dim3 grid((unsigned)((rowlen + 255) / 256 < 64 ? (rowlen + 255) / 256 : 64),
                    (unsigned)(rows < 65535 ? rows : 65535));
    gather_rows_kernel<double><<<grid, 256, 0, stream>>>((const double*)src, rowlen, idx, rows, (double*)dst);
  }
  return cudaGetLastError();
}

}  // namespace mc
