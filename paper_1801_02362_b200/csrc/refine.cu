// Exact refinement of the tensor-core MSD estimates (fp32-coordinate path).
//
// The 3xTF32 estimate (tf32_gemm.cu) carries an absolute error of ~1e-7 ..
// 1e-5 (fp32 accumulation over N atoms), too large for the north_star
// tolerance on the pairs that matter.  So:
//   cand_kernel    per frame: D_min of the estimate and the contiguous
//                  landmark window [lo, lo+cnt) holding every landmark with
//                  lam (D_est - D_min) <= thr (thr = cutoff + error margin);
//   sort kernels   counting sort of the frames by window start, so that
//                  groups of 32 consecutive sorted frames share windows;
//   refine_kernel  exact fp64 covariance of (frame group x 32-landmark
//                  sub-tile) on CUDA cores, recentred on the fly from the raw
//                  fp32 coordinates and fp64 centroids, with the Newton +
//                  adjugate fit (mc_math.cuh) fused in its epilogue; writes
//                  exact D (and R) for in-window pairs only.
// With lo = 0, cnt = L and the identity order the same kernel is the dense
// exact all-pairs MSD matrix (config 2).
#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int CNT = 256;
}

__global__ void __launch_bounds__(CNT)
cand_kernel(const float* __restrict__ D, int T, int L, int64_t ldd, double lam, double thr0,
            const double* __restrict__ fnorm, double fcoef, const int* __restrict__ rlo, const int* __restrict__ rhi,
            const float* __restrict__ dref, int cap, int* __restrict__ lo, int* __restrict__ cnt,
            float* __restrict__ dmin_out, uint8_t* __restrict__ flags, const double* __restrict__ dlife) {
  __shared__ double scratch[CNT / 32];
  __shared__ int imin[CNT / 32], imax[CNT / 32];
  const int t = blockIdx.x;
  const double thr = fnorm ? thr0 + fcoef * fnorm[t] : thr0;
  const float* row = D + (int64_t)t * ldd;
  // scan range: the whole row, or the banded range the pruned screen computed
  const int i0 = rlo ? rlo[t] : 0, i1 = rhi ? rhi[t] : L;
  double m = INFINITY;
  for (int i = i0 + threadIdx.x; i < i1; i += CNT) m = fmin(m, (double)row[i]);
  m = block_min<CNT>(m, scratch);
  // landmark-sharded evaluation: the window is taken against the minimum over every
  // shard's estimate (an all-reduce of the per-frame minima), so a shard that holds
  // none of the frame's window returns an empty one
  if (dref) m = fmin(m, (double)dref[t]);
  // close-structure lifetime window (PathCV.close_replay): frame t is
  // a refresh frame y whose later frames x lie within D(x, y) <= delta = dlife[t].  With the
  // RMSD triangle inequality every landmark any of them needs (lam (D~_l(x) - min D~(x))
  // <= thr) has d(y, a_l) <= sqrt(delta) + sqrt((sqrt(delta) + d_min(y))^2 + thr / lam), so
  // the window grows by lam (2 delta + 2 sqrt(delta) (X + dmu)), X^2 = (sqrt(delta) + dmu)^2
  // + thr / lam, dmu = sqrt(m + e_t) >= d_min(y) (e_t = fnorm[t] the estimate error bound)
  double thr_t = thr;
  if (dlife) {
    const double dl = fmax(dlife[t], 0.0), sd = sqrt(dl);
    const double dmu = sqrt(fmax(m + (fnorm ? fnorm[t] : 0.0), 0.0));
    const double X = sqrt((sd + dmu) * (sd + dmu) + thr / lam);
    thr_t = thr + lam * (2.0 * dl + 2.0 * sd * (X + dmu));
  }
  int a = L, b = -1;
  for (int i = i0 + threadIdx.x; i < i1; i += CNT) {
    if (lam * ((double)row[i] - m) <= thr_t) { a = min(a, i); b = max(b, i); }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
    b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
  }
  if ((threadIdx.x & 31) == 0) { imin[threadIdx.x >> 5] = a; imax[threadIdx.x >> 5] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < CNT / 32; ++w) { a = min(a, imin[w]); b = max(b, imax[w]); }
    a = min(imin[0], a);
    b = max(imax[0], b);
    int c = b - a + 1;
    if (c <= 0) { a = 0; c = 0; }
    uint8_t f = 0;
    if (!isfinite(m)) f |= kFlagNonFinite;
    if (c > cap) { f |= kFlagSigOverflow; c = cap; }
    lo[t] = a;
    cnt[t] = c;
    if (dmin_out) dmin_out[t] = (float)m;
    if (flags) flags[t] = f;
  }
}

cudaError_t launch_candidates(const float* D, int T, int L, int64_t ldd, double lam, double thr, const double* fnorm,
                              double fcoef, const int* rlo, const int* rhi, const float* dref, int cap, int* lo,
                              int* cnt, float* dmin, uint8_t* flags, cudaStream_t stream, const double* dlife) {
  if (T <= 0) return cudaSuccess;
  cand_kernel<<<T, CNT, 0, stream>>>(D, T, L, ldd, lam, thr, fnorm, fcoef, rlo, rhi, dref, cap, lo, cnt, dmin, flags,
                                     dlife);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- counting sort by window start
__global__ void hist_kernel(const int* __restrict__ key, int T, int* __restrict__ bins) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) atomicAdd(&bins[key[t]], 1);
}

// exclusive scan of nb bins in one CTA (nb up to a few 10^5)
__global__ void __launch_bounds__(1024) scan_kernel(int* __restrict__ bins, int nb) {
  __shared__ int part[1024];
  const int per = (nb + 1023) / 1024;
  const int b0 = threadIdx.x * per;
  int s = 0;
  for (int i = 0; i < per && b0 + i < nb; ++i) s += bins[b0 + i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int v = threadIdx.x >= o ? part[threadIdx.x - o] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int i = 0; i < per && b0 + i < nb; ++i) {
    const int v = bins[b0 + i];
    bins[b0 + i] = run;
    run += v;
  }
}

__global__ void scatter_kernel(const int* __restrict__ key, int T, int* __restrict__ offs, int* __restrict__ perm) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < T) perm[atomicAdd(&offs[key[t]], 1)] = t;
}

cudaError_t launch_sort_by_key(const int* key, int T, int nbins, int* bins, int* perm, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(bins, 0, sizeof(int) * (size_t)nbins, stream);
  if (e != cudaSuccess) return e;
  hist_kernel<<<(T + 255) / 256, 256, 0, stream>>>(key, T, bins);
  scan_kernel<<<1, 1024, 0, stream>>>(bins, nbins);
  scatter_kernel<<<(T + 255) / 256, 256, 0, stream>>>(key, T, bins, perm);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- exact refinement tiles
namespace {
constexpr int RF = 32, RL = 32, RKC = 8, RNT = 256, RRS = RF + 2;
constexpr int RLOADS = RF * RKC / RNT;  // atoms*structures per thread per chunk (1)
}

// frames: raw fp32 AoS [T, n, 3] + fp64 centroid; landmarks: raw fp32 AoS [L, n, 3] + centroid;
// w [n] displacement weights.  perm: sorted frame order (nullable = identity).
// Frame group g = perm[32g .. 32g+32); its window = union of [lo_t, lo_t+cnt_t).
// Outputs per in-window pair: Dex[t*cap + (l - lo_t)] (fp64), Rex[...*9] (nullable),
// and when dense (lo == nullptr) Dd[t*ldd + l] (fp32).
__global__ void __launch_bounds__(RNT, 2)
refine_kernel(const float* __restrict__ fr, const double* __restrict__ fc, const float* __restrict__ lr,
              const double* __restrict__ lc, const double* __restrict__ w, const double* __restrict__ gx,
              const double* __restrict__ ga, int T, int L, int n, const int* __restrict__ perm,
              const int* __restrict__ lo, const int* __restrict__ cnt, int cap, double* __restrict__ Dex,
              double* __restrict__ Rex, float* __restrict__ Dd, int64_t ldd, uint8_t* __restrict__ flags) {
  __shared__ __align__(16) double sF[2][RKC * 3 * RRS];
  __shared__ __align__(16) double sL[2][RKC * 3 * RRS];
  __shared__ int s_t[RF], s_lo[RF], s_cnt[RF];
  __shared__ int s_wlo, s_whi;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int g = blockIdx.x;
  if (tid < RF) {
    const int k = g * RF + tid;
    int t = -1, a = 0, c = 0;
    if (k < T) {
      t = perm ? perm[k] : k;
      a = lo ? lo[t] : 0;
      c = lo ? cnt[t] : L;
    }
    s_t[tid] = t;
    s_lo[tid] = a;
    s_cnt[tid] = c;
  }
  __syncthreads();
  if (tid == 0) {
    int a = L, b = 0;
    for (int i = 0; i < RF; ++i)
      if (s_t[i] >= 0 && s_cnt[i] > 0) { a = min(a, s_lo[i]); b = max(b, s_lo[i] + s_cnt[i]); }
    s_wlo = a;
    s_whi = b;
  }
  __syncthreads();
  const int wlo = s_wlo, whi = s_whi;
  // per-thread staging of one (structure, atom) per chunk for each operand
  const int ls_struct = tid / RKC;   // 0..31
  const int ls_atom = tid % RKC;     // 0..7
  const int my_t = s_t[ls_struct];
  double fcx = 0, fcy = 0, fcz = 0;
  if (my_t >= 0) { fcx = fc[3 * my_t]; fcy = fc[3 * my_t + 1]; fcz = fc[3 * my_t + 2]; }
  for (int l0 = wlo; l0 < whi; l0 += RL) {
    const int my_l = l0 + ls_struct;
    double lcx = 0, lcy = 0, lcz = 0;
    if (my_l < L) { lcx = lc[3 * my_l]; lcy = lc[3 * my_l + 1]; lcz = lc[3 * my_l + 2]; }
    double acc[2][2][9];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int e = 0; e < 9; ++e) acc[a][c][e] = 0.0;
    // raw fp32 loads are issued one chunk ahead (gload) and only converted /
    // recentred when they are staged (sstore), so the load latency overlaps
    // the previous chunk's FMAs instead of stalling at the issue point
    float pf[3], pl[3];
    double pw;
    bool vf, vl;
    auto gload = [&](int k0) {
      const int j = k0 + ls_atom;
      vf = my_t >= 0 && j < n;
      vl = my_l < L && j < n;
      if (vf) {
        const float* p = fr + ((int64_t)my_t * n + j) * 3;
        pf[0] = p[0]; pf[1] = p[1]; pf[2] = p[2];
      }
      if (vl) {
        const float* p = lr + ((int64_t)my_l * n + j) * 3;
        pl[0] = p[0]; pl[1] = p[1]; pl[2] = p[2];
        pw = w[j];
      }
    };
    auto sstore = [&](int buf) {
      const double rf[3] = {vf ? (double)pf[0] - fcx : 0.0, vf ? (double)pf[1] - fcy : 0.0,
                            vf ? (double)pf[2] - fcz : 0.0};
      const double rl[3] = {vl ? pw * ((double)pl[0] - lcx) : 0.0, vl ? pw * ((double)pl[1] - lcy) : 0.0,
                            vl ? pw * ((double)pl[2] - lcz) : 0.0};
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        sF[buf][(ls_atom * 3 + b) * RRS + ls_struct] = rf[b];
        sL[buf][(ls_atom * 3 + b) * RRS + ls_struct] = rl[b];
      }
    };
    const int nch = (n + RKC - 1) / RKC;
    gload(0);
    __syncthreads();
    sstore(0);
    __syncthreads();
    for (int ch = 0; ch < nch; ++ch) {
      const int buf = ch & 1;
      if (ch + 1 < nch) gload((ch + 1) * RKC);
#pragma unroll
      for (int j = 0; j < RKC; ++j) {
        double2 xf[3], al[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          xf[b] = *reinterpret_cast<const double2*>(&sF[buf][(j * 3 + b) * RRS + 2 * ty]);
          al[b] = *reinterpret_cast<const double2*>(&sL[buf][(j * 3 + b) * RRS + 2 * tx]);
        }
#pragma unroll
        for (int b = 0; b < 3; ++b)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            acc[0][0][b * 3 + c] = fma(xf[b].x, al[c].x, acc[0][0][b * 3 + c]);
            acc[0][1][b * 3 + c] = fma(xf[b].x, al[c].y, acc[0][1][b * 3 + c]);
            acc[1][0][b * 3 + c] = fma(xf[b].y, al[c].x, acc[1][0][b * 3 + c]);
            acc[1][1][b * 3 + c] = fma(xf[b].y, al[c].y, acc[1][1][b * 3 + c]);
          }
      }
      if (ch + 1 < nch) sstore(buf ^ 1);
      __syncthreads();
    }
    // fused fit epilogue (exact fp64)
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int fi = 2 * ty + a;
      const int t = s_t[fi];
      if (t < 0) continue;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int l = l0 + 2 * tx + c;
        const int slot = l - s_lo[fi];
        if (l >= L || slot < 0 || slot >= s_cnt[fi]) continue;
        double q[4];
        bool ill = false;
        double msd = fit_fast(acc[a][c], gx[t], ga[l], Rex ? q : nullptr, &ill);
        uint8_t f = 0;
        if (ill) {
          double k4[4][4], V[4][4], ev[4];
          kearsley_from_S(acc[a][c], gx[t], ga[l], k4);
          if (!jacobi4(k4, ev, V)) f |= kFlagNoConverge;
          msd = ev[0];
          q[0] = V[0][0]; q[1] = V[1][0]; q[2] = V[2][0]; q[3] = V[3][0];
        }
        if (Dex) Dex[(int64_t)t * cap + slot] = msd;
        if (Dd) Dd[(int64_t)t * ldd + l] = (float)msd;
        if (Rex) {
          double r[9];
          quat_to_rot(q, r);
          double* o = Rex + ((int64_t)t * cap + slot) * 9;
#pragma unroll
          for (int e = 0; e < 9; ++e) o[e] = r[e];
        }
        if (f && flags) flags[t] |= f;
      }
    }
    __syncthreads();
  }
}

cudaError_t launch_refine(const float* fr, const double* fc, const float* lr, const double* lc, const double* w,
                          const double* gx, const double* ga, int T, int L, int n, const int* perm, const int* lo,
                          const int* cnt, int cap, double* Dex, double* Rex, float* Dd, int64_t ldd, uint8_t* flags,
                          cudaStream_t stream) {
  if (T <= 0 || L <= 0) return cudaSuccess;
  refine_kernel<<<(T + RF - 1) / RF, RNT, 0, stream>>>(fr, fc, lr, lc, w, gx, ga, T, L, n, perm, lo, cnt, cap, Dex,
                                                        Rex, Dd, ldd, flags);
  return cudaGetLastError();
}

}  // namespace mc
