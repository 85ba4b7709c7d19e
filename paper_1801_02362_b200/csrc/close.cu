// K5 — floating close-structure driver (Alg. 2, PAPER.md:168-194;
// SPEC.md:133-141,157-162), device side.
//
// The refresh decisions are inherently sequential (y changes only at a
// refresh), so the device work is split into:
//   1. a speculative window: D(x_s, x_{s-k}) for k = 1..K for every frame
//      in parallel (cov_pairs + Newton; fp64, so |dD| ~ 1e-16),
//   2. this scan kernel, one CTA per walker.  First a parallel pass: the next
//      refresh after a refresh at r is next(r) = the first s in (r, r + K] with
//      D(x_s, x_r) > eps (from the window), so the refresh chain 0 -> next(0) ->
//      ... is a linked list; pointer doubling in shared memory marks every node
//      of the chain from frame 0 in log2(steps) rounds, and a prefix-max scan
//      gives every frame its close structure.  Only if the chain reaches a
//      refresh whose successor lies beyond the window (or the walker is too long
//      for shared memory) does the CTA fall back to walking its frames in order,
//      computing the fit on the fly when the close structure is older than K,
//   3. xy_eig_kernel: the full x<->y spectrum (reference Jacobi) of every
//      non-refresh frame, which Eq. 6's dR_xy/dx term needs.
// Strict '>' and first-frame refresh follow SPEC.md:159,162.
#include <algorithm>
#include <cstdlib>

#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int SCAN_NT = 256;
constexpr int SCAN_CHUNK = 256;  // frames staged per shared-memory chunk
}

// frames of walker w are global indices w*steps + s; planes fp64 [.,3,npad].
__global__ void __launch_bounds__(SCAN_NT)
close_scan_kernel(const double* __restrict__ fpl, const double* __restrict__ gx, int steps, int npad,
                  const double* __restrict__ w, const double* __restrict__ dwin, int K, double eps,
                  uint8_t* __restrict__ refresh, int* __restrict__ ridx, double* __restrict__ dxy,
                  int* __restrict__ n_onthefly, int par) {
  extern __shared__ double sw[];  // [SCAN_CHUNK * K] (serial) or the chain arrays (parallel)
  __shared__ double scratch[SCAN_NT / 32];
  __shared__ int s_r, s_pos, s_miss;
  __shared__ int s_seg[SCAN_NT];
  const int walker = blockIdx.x;
  const int64_t base = (int64_t)walker * steps;
  const int tid = threadIdx.x;
  if (par) {
    // ---- parallel pass: J = next-refresh pointers, M = chain marks (shared memory)
    int* J = reinterpret_cast<int*>(sw);
    int* J2 = J + steps;
    uint8_t* M = reinterpret_cast<uint8_t*>(J2 + steps);
    constexpr int END = 0x7fffffff, UNK = -1;
    auto next_of = [&](int r) {
      for (int k = 1; k <= K; ++k) {
        const int s = r + k;
        if (s >= steps) return END;
        if (dwin[(base + s) * K + (k - 1)] > eps) return s;
      }
      return r + K + 1 >= steps ? END : UNK;
    };
    for (int r = tid; r < steps; r += SCAN_NT) {
      J[r] = next_of(r);
      M[r] = r == 0;
    }
    __syncthreads();
    for (int span = 1; span < steps; span <<= 1) {
      for (int r = tid; r < steps; r += SCAN_NT) {
        const int j = J[r];
        if (M[r] && j >= 0 && j != END) M[j] = 1;
      }
      __syncthreads();
      for (int r = tid; r < steps; r += SCAN_NT) {
        const int j = J[r];
        J2[r] = (j >= 0 && j != END) ? J[j] : j;
      }
      __syncthreads();
      int* t = J;
      J = J2;
      J2 = t;
    }
    // a marked refresh whose successor is beyond the window: the chain is unresolved
    int miss = 0;
    for (int r = tid; r < steps; r += SCAN_NT) miss |= (M[r] && next_of(r) == UNK);
    if (!__syncthreads_or(miss)) {
      // prefix max of the marked positions: each frame's close structure
      const int per = (steps + SCAN_NT - 1) / SCAN_NT, s0 = tid * per, s1 = min(steps, s0 + per);
      int m = -1;
      for (int t = s0; t < s1; ++t) if (M[t]) m = t;
      s_seg[tid] = m;
      __syncthreads();
      int run = -1;
      for (int i = 0; i < tid; ++i) run = max(run, s_seg[i]);
      for (int t = s0; t < s1; ++t) {
        const int prev = run;  // last refresh before t
        if (M[t]) run = t;
        refresh[base + t] = M[t];
        ridx[base + t] = (int)(base + run);
        // D(x_t, y) with y the close structure t was tested against (0 for frame 0)
        dxy[base + t] = t == 0 ? 0.0 : dwin[(base + t) * K + (t - prev - 1)];
      }
      if (tid == 0 && n_onthefly) n_onthefly[walker] = 0;
      return;
    }
    __syncthreads();  // fall through to the serial walk (its staging reuses sw)
  }
  if (threadIdx.x == 0) { s_r = -1; s_pos = 0; }
  int fly = 0;
  for (int c0 = 0; c0 < steps; c0 += SCAN_CHUNK) {
    const int c1 = min(steps, c0 + SCAN_CHUNK);
    __syncthreads();
    for (int e = threadIdx.x; e < (c1 - c0) * K; e += SCAN_NT) sw[e] = dwin[(base + c0) * K + e];
    if (threadIdx.x == 0) s_pos = c0;
    __syncthreads();
    while (true) {
      if (threadIdx.x == 0) {
        int s = s_pos, r = s_r;
        s_miss = 0;
        for (; s < c1; ++s) {
          bool fresh;
          double d;
          if (r < 0) {
            fresh = true;
            d = 0.0;
          } else {
            const int k = s - r;
            if (k > K) { s_miss = 1; break; }
            d = sw[(s - c0) * K + (k - 1)];
            fresh = d > eps;
          }
          if (fresh) r = s;
          refresh[base + s] = fresh ? 1 : 0;
          ridx[base + s] = (int)(base + r);
          dxy[base + s] = d;
        }
        s_pos = s;
        s_r = r;
      }
      __syncthreads();
      if (!s_miss) break;
      // close structure older than the window: fit x_s <-> y on the fly
      const int s = s_pos, r = s_r;
      const double* x = fpl + (base + s) * 3 * npad;
      const double* y = fpl + (base + r) * 3 * npad;
      double acc[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) acc[e] = 0.0;
      for (int j = threadIdx.x; j < npad; j += SCAN_NT) {
        const double wj = w[j];
        const double x0 = x[j], x1 = x[npad + j], x2 = x[2 * npad + j];
        const double y0 = wj * y[j], y1 = wj * y[npad + j], y2 = wj * y[2 * npad + j];
        acc[0] += x0 * y0; acc[1] += x0 * y1; acc[2] += x0 * y2;
        acc[3] += x1 * y0; acc[4] += x1 * y1; acc[5] += x1 * y2;
        acc[6] += x2 * y0; acc[7] += x2 * y1; acc[8] += x2 * y2;
      }
#pragma unroll
      for (int e = 0; e < 9; ++e) acc[e] = block_sum<SCAN_NT>(acc[e], scratch);
      if (threadIdx.x == 0) {
        bool ill;
        const double d = fit_fast(acc, gx[base + s], gx[base + r], nullptr, &ill);
        const bool fresh = d > eps;
        int rr = fresh ? s : r;
        refresh[base + s] = fresh ? 1 : 0;
        ridx[base + s] = (int)(base + rr);
        dxy[base + s] = d;
        s_r = rr;
        s_pos = s + 1;
        ++fly;
      }
      __syncthreads();
    }
  }
  if (threadIdx.x == 0 && n_onthefly) n_onthefly[walker] = fly;
}

cudaError_t launch_close_scan(const double* fpl, const double* gx, int walkers, int steps, int npad,
                              const double* w, const double* dwin, int K, double eps, uint8_t* refresh,
                              int* ridx, double* dxy, int* n_onthefly, cudaStream_t stream) {
  if (walkers <= 0 || steps <= 0) return cudaSuccess;
  const size_t serial = (size_t)SCAN_CHUNK * K * sizeof(double);
  const size_t chain = (size_t)steps * 9;  // two int pointer arrays + the marks
  const bool par = chain <= 200 * 1024 && getenv("MC_CLOSE_SCAN_SERIAL") == nullptr;
  const size_t smem = std::max(serial, par ? (chain + 15) / 16 * 16 : (size_t)0);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(close_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  close_scan_kernel<<<walkers, SCAN_NT, smem, stream>>>(fpl, gx, steps, npad, w, dwin, K, eps, refresh, ridx, dxy,
                                                        n_onthefly, par ? 1 : 0);
  return cudaGetLastError();
}

// Full x<->y spectrum for every non-refresh frame t (warp per frame):
// xyeig[t] = {eigvals[4], eigvecs row-major[16]}, rxy[t] = R(q0).
__global__ void __launch_bounds__(256)
xy_eig_kernel(const double* __restrict__ fpl, const double* __restrict__ gx, int64_t T, int npad,
              const double* __restrict__ w, const uint8_t* __restrict__ refresh, const int* __restrict__ ridx,
              double* __restrict__ xyeig, double* __restrict__ rxy, uint8_t* __restrict__ flags) {
  const int64_t t = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  if (refresh[t]) {
    if (lane == 0) {
      // y = x: R_xy = I (unused by the refresh path; written for completeness)
      for (int e = 0; e < 9; ++e) rxy[t * 9 + e] = (e % 4 == 0) ? 1.0 : 0.0;
      if (flags) flags[t] = 0;
    }
    return;
  }
  const int r = ridx[t];
  const double* x = fpl + t * 3 * npad;
  const double* y = fpl + (int64_t)r * 3 * npad;
  double acc[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) acc[e] = 0.0;
  for (int j = lane; j < npad; j += 32) {
    const double wj = w[j];
    const double x0 = x[j], x1 = x[npad + j], x2 = x[2 * npad + j];
    const double y0 = wj * y[j], y1 = wj * y[npad + j], y2 = wj * y[2 * npad + j];
    acc[0] = fma(x0, y0, acc[0]); acc[1] = fma(x0, y1, acc[1]); acc[2] = fma(x0, y2, acc[2]);
    acc[3] = fma(x1, y0, acc[3]); acc[4] = fma(x1, y1, acc[4]); acc[5] = fma(x1, y2, acc[5]);
    acc[6] = fma(x2, y0, acc[6]); acc[7] = fma(x2, y1, acc[7]); acc[8] = fma(x2, y2, acc[8]);
  }
#pragma unroll
  for (int e = 0; e < 9; ++e) acc[e] = warp_sum(acc[e]);
  if (lane != 0) return;
  double k[4][4], V[4][4], ev[4];
  kearsley_from_S(acc, gx[t], gx[r], k);
  const bool ok = jacobi4(k, ev, V);
  uint8_t f = ok ? 0 : kFlagNoConverge;
  if (ev[1] - ev[0] < kDegeneracyTol) f |= kFlagDegenerate;
  double* e = xyeig + t * 20;
#pragma unroll
  for (int i = 0; i < 4; ++i) e[i] = ev[i];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr)
#pragma unroll
    for (int c = 0; c < 4; ++c) e[4 + rr * 4 + c] = V[rr][c];
  const double q[4] = {V[0][0], V[1][0], V[2][0], V[3][0]};
  double R[9];
  quat_to_rot(q, R);
#pragma unroll
  for (int i = 0; i < 9; ++i) rxy[t * 9 + i] = R[i];
  if (flags) flags[t] = f;
}

cudaError_t launch_xy_eig(const double* fpl, const double* gx, int64_t T, int npad, const double* w,
                          const uint8_t* refresh, const int* ridx, double* xyeig, double* rxy, uint8_t* flags,
                          cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  xy_eig_kernel<<<(unsigned)((T + 7) / 8), 256, 0, stream>>>(fpl, gx, T, npad, w, refresh, ridx, xyeig, rxy, flags);
  return cudaGetLastError();
}

// Window pair indices: pair (s, s-k) for k = 1..K within each walker.
__global__ void window_pairs_kernel(int walkers, int steps, int K, int* __restrict__ xi, int* __restrict__ ai) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t P = (int64_t)walkers * steps * K;
  if (p >= P) return;
  const int64_t f = p / K;
  const int k = (int)(p - f * K) + 1;
  const int s = (int)(f % steps);
  xi[p] = (int)f;
  ai[p] = s - k >= 0 ? (int)(f - k) : -1;
}

cudaError_t launch_window_pairs(int walkers, int steps, int K, int* xi, int* ai, cudaStream_t stream) {
  const int64_t P = (int64_t)walkers * steps * K;
  if (P <= 0) return cudaSuccess;
  window_pairs_kernel<<<(unsigned)((P + 255) / 256), 256, 0, stream>>>(walkers, steps, K, xi, ai);
  return cudaGetLastError();
}

}  // namespace mc
