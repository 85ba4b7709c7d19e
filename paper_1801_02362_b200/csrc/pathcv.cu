// K4 — fused path-CV reduction (Eq. 2) and its gradient.
//
// s = sum_i q_i p_i,  z = D_min - (1/lam) ln sum_i e^{-lam (D_i - D_min)},
// p = softmax(-lam D) with the min-D shift.
// ds = sum_i cs_i dD_i with cs_i = -lam p_i (q_i - s);  dz = sum_i p_i dD_i.
//
// Every dD_i has the form (w.r.t. the centred x)
//     2 w (x - Rhat_i a_i)  [+ <M_i, dR_xy/dx> for close-structure frames]
// and the raw-coordinate gradient subtracts w' * sum_k (.) (the centring
// chain rule).  Rhat_i is the exact fit rotation of (x, a_i) or, on a
// non-refresh frame, R_xy R_{a_i y} (Eq. 5).  Because everything is linear
// in the coefficients, the per-landmark work is folded into per-frame
// quantities here (cv_weights_kernel) and a single pass over atoms
// (cv_grad_kernel) writes the gradients:
//   U_k   = sum_i c_i Rhat_i a_{i,k}               (only significant i)
//   M     = -2 [ sum_i c_i S_i R_i^T - R_xy sum_i c_i R_i A_i R_i^T ]
//   g_c   = <M, dR/dq_c>,  v = sum_m (q_m.g)/(l_0 - l_m) q_m
//   dR-term_k = v^T (dK/dx_k) q_0                     (closed form, mc_math)
// Landmarks with lam (D_i - D_min) > cutoff (default 50) contribute
// < e^-50 relative to the leading term and are skipped.
#include <algorithm>
#include <cstdlib>

#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int WNT = 256;
constexpr int FVEC = 16;  // sumcs, sumcz, corr_s[3], corr_z[3], v_s[4], v_z[4]
}

__device__ __forceinline__ void mat3_mul(const double* a, const double* b, double* c) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[i * 3 + j] = a[i * 3] * b[j] + a[i * 3 + 1] * b[3 + j] + a[i * 3 + 2] * b[6 + j];
}

// Neighbour-list restriction (SPEC neighbourlist / colvar "active set"): row t
// sums over the landmarks listed in nb_idx[nb_row[t] * nb_m ..] only (dense
// rows); dmode 1 = write the row distances (Eq. 5 on non-refresh rows) and stop,
// dmode 2 = distances already in D (no recomputation).
struct NbArgs {
  const int* idx;
  const int* row;
  int m;
  int dmode;
};
constexpr int kNbMaxL = 16384;  // bitmap capacity (landmarks) for the active set

__global__ void __launch_bounds__(WNT)
cv_weights_kernel(int T, int t0, int L, double lam, double cutoff, int cap, int ld, NbArgs nb, const int* __restrict__ rowlo,
                  const int* __restrict__ rowcnt, double* __restrict__ D,
                  const double* __restrict__ q, const double* __restrict__ R, const double* __restrict__ fwbar,
                  const double* __restrict__ lwbar, const uint8_t* __restrict__ refresh,
                  const int* __restrict__ ridx, const double* __restrict__ S, const double* __restrict__ rxy,
                  const double* __restrict__ xyeig, const double* __restrict__ gx, const double* __restrict__ ga,
                  const double* __restrict__ lmom, double* __restrict__ s_out, double* __restrict__ z_out,
                  int* __restrict__ sig_idx, double* __restrict__ sig_coef, int* __restrict__ nsig,
                  double* __restrict__ fvec, uint8_t* __restrict__ flags) {
  __shared__ double scratch[WNT / 32];
  __shared__ int wcount[WNT / 32];
  __shared__ uint32_t act[kNbMaxL / 32];
  // frame t (global index; rows of D/S/R and the per-frame inputs) and its
  // chunk-local slot tl (the significant-list outputs of this launch)
  const int t = t0 + blockIdx.x, tl = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool masked = nb.idx != nullptr && nb.dmode != 1;
  if (masked) {
    for (int wv = tid; wv < (L + 31) / 32; wv += WNT) act[wv] = 0u;
    __syncthreads();
    const int* lst = nb.idx + (int64_t)nb.row[t] * nb.m;
    for (int k = tid; k < nb.m; k += WNT) atomicOr(&act[lst[k] >> 5], 1u << (lst[k] & 31));
    __syncthreads();
  }
  auto active = [&](int i) { return !masked || ((act[i >> 5] >> (i & 31)) & 1u); };
  const bool approx = refresh && !refresh[t];
  const int r = approx ? ridx[t] : t;
  double Rxy[9];
  if (approx) {
#pragma unroll
    for (int e = 0; e < 9; ++e) Rxy[e] = rxy[(int64_t)t * 9 + e];
  }
  // row layout: dense rows (ld = L, landmark = column) or sparse windows
  // (row t holds landmarks rowlo[t] .. rowlo[t] + rowcnt[t] - 1, stride ld)
  double* Dt = D + (int64_t)t * ld;
  const int nrow = rowcnt ? rowcnt[t] : L;
  const int off = rowlo ? rowlo[t] : 0;
  // pass 1: distances (Eq. 5 on non-refresh frames) and their minimum
  double dmin = INFINITY;
  bool finite = true;
  for (int i = tid; i < nrow; i += WNT) {
    double d;
    if (approx && nb.dmode != 2) {
      const double* Ri = R + ((int64_t)r * ld + i) * 9;
      const double* Si = S + ((int64_t)t * ld + i) * 9;
      double Rr[9], Rh[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) Rr[e] = Ri[e];
      mat3_mul(Rxy, Rr, Rh);
      double dot = 0.0;
#pragma unroll
      for (int e = 0; e < 9; ++e) dot = fma(Rh[e], Si[e], dot);
      d = gx[t] + ga[off + i] - 2.0 * dot;
      Dt[i] = d;
    } else {
      d = Dt[i];
    }
    if (!active(i)) continue;
    finite = finite && isfinite(d);
    dmin = fmin(dmin, d);
  }
  if (nb.dmode == 1) return;  // distances only (block-uniform)
  dmin = block_min<WNT>(dmin, scratch);
  const int nonfinite = __syncthreads_or(!finite);
  // pass 2: partition function
  double zs = 0.0, qs = 0.0;
  for (int i = tid; i < nrow; i += WNT) {
    if (!active(i)) continue;
    const double e = exp(-lam * (Dt[i] - dmin));
    zs += e;
    qs += q[off + i] * e;
  }
  zs = block_sum<WNT>(zs, scratch);
  qs = block_sum<WNT>(qs, scratch);
  const double sval = qs / zs;
  const double zval = dmin - log(zs) / lam;
  // pass 3: ordered compaction of the significant landmarks + per-frame sums
  double acc[44];
#pragma unroll
  for (int e = 0; e < 44; ++e) acc[e] = 0.0;
  int total = 0;
  for (int b0 = 0; b0 < nrow; b0 += WNT) {
    const int i = b0 + tid;
    double di = 0.0;
    bool sig = false;
    if (i < nrow && active(i)) {
      di = Dt[i];
      sig = lam * (di - dmin) <= cutoff;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, sig);
    __syncthreads();
    if (lane == 0) wcount[warp] = __popc(bal);
    __syncthreads();
    int pos = total + __popc(bal & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) pos += wcount[w];
    int blk = 0;
    for (int w = 0; w < WNT / 32; ++w) blk += wcount[w];
    if (sig) {
      const double p = exp(-lam * (di - dmin)) / zs;
      const int li = off + i;
      const double cs = -lam * p * (q[li] - sval);
      const double cz = p;
      double Rh[9], Rr[9];
      if (approx) {
#pragma unroll
        for (int e = 0; e < 9; ++e) Rr[e] = R[((int64_t)r * ld + i) * 9 + e];
        mat3_mul(Rxy, Rr, Rh);
      } else {
#pragma unroll
        for (int e = 0; e < 9; ++e) Rh[e] = R[((int64_t)t * ld + i) * 9 + e];
      }
      if (pos < cap) {
        sig_idx[(int64_t)tl * cap + pos] = li;
        double* co = sig_coef + ((int64_t)tl * cap + pos) * 18;
#pragma unroll
        for (int e = 0; e < 9; ++e) { co[e] = cs * Rh[e]; co[9 + e] = cz * Rh[e]; }
      }
      acc[0] += cs;
      acc[1] += cz;
      const double wb0 = lwbar[3 * li], wb1 = lwbar[3 * li + 1], wb2 = lwbar[3 * li + 2];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double rw = Rh[a * 3] * wb0 + Rh[a * 3 + 1] * wb1 + Rh[a * 3 + 2] * wb2;
        acc[2 + a] += cs * rw;
        acc[5 + a] += cz * rw;
      }
      if (approx) {
        // S_i R_i^T and R_i A_i R_i^T (R_i = saved rotation of landmark i)
        const double* Si = S + ((int64_t)t * ld + i) * 9;
        const double* m = lmom + 6 * (int64_t)li;
        const double A[9] = {m[0], m[1], m[2], m[1], m[3], m[4], m[2], m[4], m[5]};
        double SRt[9], RA[9], RAR[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            SRt[a * 3 + b] = Si[a * 3] * Rr[b * 3] + Si[a * 3 + 1] * Rr[b * 3 + 1] + Si[a * 3 + 2] * Rr[b * 3 + 2];
        mat3_mul(Rr, A, RA);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            RAR[a * 3 + b] = RA[a * 3] * Rr[b * 3] + RA[a * 3 + 1] * Rr[b * 3 + 1] + RA[a * 3 + 2] * Rr[b * 3 + 2];
#pragma unroll
        for (int e = 0; e < 9; ++e) {
          acc[8 + e] += cs * SRt[e];
          acc[17 + e] += cz * SRt[e];
          acc[26 + e] += cs * RAR[e];
          acc[35 + e] += cz * RAR[e];
        }
      }
    }
    total += blk;
  }
  const int nacc = approx ? 44 : 8;
  for (int e = 0; e < nacc; ++e) acc[e] = block_sum<WNT>(acc[e], scratch);
  if (tid != 0) return;
  s_out[t] = sval;
  z_out[t] = zval;
  nsig[tl] = min(total, cap);
  double* fv = fvec + (int64_t)tl * FVEC;
  const double fw[3] = {fwbar[3 * t], fwbar[3 * t + 1], fwbar[3 * t + 2]};
  double corr[2][3], vv[2][4];
  for (int c = 0; c < 2; ++c) {
    const double sumc = acc[c];
    for (int a = 0; a < 3; ++a) corr[c][a] = 2.0 * (sumc * fw[a] - acc[2 + 3 * c + a]);
    vv[c][0] = vv[c][1] = vv[c][2] = vv[c][3] = 0.0;
  }
  if (approx) {
    const double* e = xyeig + (int64_t)t * 20;
    double q0[4], qm[3][4], inv[3];
    for (int rr = 0; rr < 4; ++rr) q0[rr] = e[4 + rr * 4];
    for (int m = 0; m < 3; ++m) {
      for (int rr = 0; rr < 4; ++rr) qm[m][rr] = e[4 + rr * 4 + m + 1];
      inv[m] = 1.0 / (e[0] - e[m + 1]);
    }
    double J[4][9];
    rot_quat_jacobian(q0, J);
    const double yw[3] = {fwbar[3 * r], fwbar[3 * r + 1], fwbar[3 * r + 2]};
    for (int c = 0; c < 2; ++c) {
      // M = -2 [ SR - Rxy RAR ]
      const double* SR = acc + 8 + 9 * c;
      const double* RAR = acc + 26 + 9 * c;
      double XR[9], M[9];
      mat3_mul(Rxy, RAR, XR);
      for (int k = 0; k < 9; ++k) M[k] = -2.0 * (SR[k] - XR[k]);
      double g[4];
      for (int cc = 0; cc < 4; ++cc) {
        double sacc = 0.0;
        for (int k = 0; k < 9; ++k) sacc += M[k] * J[cc][k];
        g[cc] = sacc;
      }
      for (int m = 0; m < 3; ++m) {
        const double h = (qm[m][0] * g[0] + qm[m][1] * g[1] + qm[m][2] * g[2] + qm[m][3] * g[3]) * inv[m];
        for (int rr = 0; rr < 4; ++rr) vv[c][rr] += h * qm[m][rr];
      }
      double dsum[3];
      dk_contract(vv[c], q0, 1.0, fw, yw, dsum);
      for (int a = 0; a < 3; ++a) corr[c][a] += dsum[a];
    }
  }
  fv[0] = acc[0];
  fv[1] = acc[1];
  for (int a = 0; a < 3; ++a) { fv[2 + a] = corr[0][a]; fv[5 + a] = corr[1][a]; }
  for (int rr = 0; rr < 4; ++rr) { fv[8 + rr] = vv[0][rr]; fv[12 + rr] = vv[1][rr]; }
  if (flags) {
    uint8_t f = 0;
    if (total > cap) f |= kFlagSigOverflow;
    if (nonfinite || !isfinite(sval) || !isfinite(zval)) f |= kFlagNonFinite;
    flags[tl] = f;
  }
}

// One warp per frame for the exact sparse-window rows of the fp32 path (no close
// structure, no neighbour list): the ~80-entry windows fill a warp, so the
// reductions are shuffles and the significant-list compaction is one ballot per
// 32 entries -- no CTA barriers.  Same outputs as cv_weights_kernel.
constexpr int WWPB = 8;  // frames (warps) per CTA

__global__ void __launch_bounds__(WWPB * 32)
cv_weights_warp_kernel(int T, int t0, double lam, double cutoff, int cap, int ld, const int* __restrict__ rowlo,
                       const int* __restrict__ rowcnt, const double* __restrict__ D, const double* __restrict__ q,
                       const double* __restrict__ R, const double* __restrict__ fwbar,
                       const double* __restrict__ lwbar, double* __restrict__ s_out, double* __restrict__ z_out,
                       int* __restrict__ sig_idx, double* __restrict__ sig_coef, int* __restrict__ nsig,
                       double* __restrict__ fvec, uint8_t* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int tl = blockIdx.x * WWPB + (threadIdx.x >> 5);
  if (tl >= T) return;
  const int t = t0 + tl;
  const int nrow = rowcnt[t], off = rowlo[t];
  if (nrow == 0) {
    // empty window: only in landmark-sharded evaluation (this shard holds no landmark
    // near the frame): Z_g = 0, i.e. z_g = +inf, and no significant entries
    if (lane < FVEC) fvec[(int64_t)tl * FVEC + lane] = 0.0;
    if (lane == 0) {
      s_out[t] = 0.0;
      z_out[t] = INFINITY;
      nsig[tl] = 0;
      if (flags) flags[tl] = 0;
    }
    return;
  }
  const double* Dt = D + (int64_t)t * ld;
  double dmin = INFINITY;
  bool finite = true;
  for (int i = lane; i < nrow; i += 32) {
    const double d = Dt[i];
    finite = finite && isfinite(d);
    dmin = fmin(dmin, d);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
  const bool nonfinite = __any_sync(0xffffffffu, !finite);
  double zs = 0.0, qs = 0.0;
  for (int i = lane; i < nrow; i += 32) {
    const double e = exp(-lam * (Dt[i] - dmin));
    zs += e;
    qs += q[off + i] * e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    zs += __shfl_xor_sync(0xffffffffu, zs, o);
    qs += __shfl_xor_sync(0xffffffffu, qs, o);
  }
  const double sval = qs / zs;
  const double zval = dmin - log(zs) / lam;
  double acc[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) acc[e] = 0.0;
  int total = 0;
  for (int b0 = 0; b0 < nrow; b0 += 32) {
    const int i = b0 + lane;
    const double di = i < nrow ? Dt[i] : 0.0;
    const bool sig = i < nrow && lam * (di - dmin) <= cutoff;
    const unsigned bal = __ballot_sync(0xffffffffu, sig);
    if (sig) {
      const int pos = total + __popc(bal & ((1u << lane) - 1u));
      const double p = exp(-lam * (di - dmin)) / zs;
      const int li = off + i;
      const double cs = -lam * p * (q[li] - sval);
      const double cz = p;
      double Rh[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) Rh[e] = R[((int64_t)t * ld + i) * 9 + e];
      if (pos < cap) {
        sig_idx[(int64_t)tl * cap + pos] = li;
        double* co = sig_coef + ((int64_t)tl * cap + pos) * 18;
#pragma unroll
        for (int e = 0; e < 9; ++e) { co[e] = cs * Rh[e]; co[9 + e] = cz * Rh[e]; }
      }
      acc[0] += cs;
      acc[1] += cz;
      const double wb0 = lwbar[3 * li], wb1 = lwbar[3 * li + 1], wb2 = lwbar[3 * li + 2];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double rw = Rh[a * 3] * wb0 + Rh[a * 3 + 1] * wb1 + Rh[a * 3 + 2] * wb2;
        acc[2 + a] += cs * rw;
        acc[5 + a] += cz * rw;
      }
    }
    total += __popc(bal);
  }
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
  if (lane != 0) return;
  s_out[t] = sval;
  z_out[t] = zval;
  nsig[tl] = min(total, cap);
  double* fv = fvec + (int64_t)tl * FVEC;
  fv[0] = acc[0];
  fv[1] = acc[1];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    fv[2 + a] = 2.0 * (acc[0] * fwbar[3 * t + a] - acc[2 + a]);
    fv[5 + a] = 2.0 * (acc[1] * fwbar[3 * t + a] - acc[5 + a]);
  }
#pragma unroll
  for (int rr = 0; rr < 8; ++rr) fv[8 + rr] = 0.0;
  if (flags) {
    uint8_t f = 0;
    if (total > cap) f |= kFlagSigOverflow;
    if (nonfinite || !isfinite(sval) || !isfinite(zval)) f |= kFlagNonFinite;
    flags[tl] = f;
  }
}

// Warp-per-frame form of cv_weights_kernel for close-structure rows (refresh != NULL,
// no neighbour list): the same three passes (Eq. 5 distances of non-refresh rows and
// their minimum, the partition function, the ordered significant list with the
// per-frame sums and the Eq. 6 M-matrix terms), with warp shuffles instead of block
// reductions -- one frame per warp, 8 frames per CTA.  Same values as the block kernel
// up to the summation order.
__global__ void __launch_bounds__(WWPB * 32)
cv_weights_close_warp_kernel(int T, int t0, double lam, double cutoff, int cap, int ld,
                             const int* __restrict__ rowlo, const int* __restrict__ rowcnt, int L,
                             double* __restrict__ D, const double* __restrict__ q, const double* __restrict__ R,
                             const double* __restrict__ fwbar, const double* __restrict__ lwbar,
                             const uint8_t* __restrict__ refresh, const int* __restrict__ ridx,
                             const double* __restrict__ S, const double* __restrict__ rxy,
                             const double* __restrict__ xyeig, const double* __restrict__ gx,
                             const double* __restrict__ ga, const double* __restrict__ lmom,
                             double* __restrict__ s_out, double* __restrict__ z_out, int* __restrict__ sig_idx,
                             double* __restrict__ sig_coef, int* __restrict__ nsig, double* __restrict__ fvec,
                             uint8_t* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int tl = blockIdx.x * WWPB + (threadIdx.x >> 5);
  if (tl >= T) return;
  const int t = t0 + tl;
  const bool approx = !refresh[t];
  const int r = approx ? ridx[t] : t;
  double Rxy[9];
  if (approx) {
#pragma unroll
    for (int e = 0; e < 9; ++e) Rxy[e] = rxy[(int64_t)t * 9 + e];
  }
  double* Dt = D + (int64_t)t * ld;
  const int nrow = rowcnt ? rowcnt[t] : L;
  const int off = rowlo ? rowlo[t] : 0;
  double dmin = INFINITY;
  bool finite = true;
  for (int i = lane; i < nrow; i += 32) {
    double d;
    if (approx) {
      const double* Ri = R + ((int64_t)r * ld + i) * 9;
      const double* Si = S + ((int64_t)t * ld + i) * 9;
      double Rr[9], Rh[9];
#pragma unroll
      for (int e = 0; e < 9; ++e) Rr[e] = Ri[e];
      mat3_mul(Rxy, Rr, Rh);
      double dot = 0.0;
#pragma unroll
      for (int e = 0; e < 9; ++e) dot = fma(Rh[e], Si[e], dot);
      d = gx[t] + ga[off + i] - 2.0 * dot;
      Dt[i] = d;
    } else {
      d = Dt[i];
    }
    finite = finite && isfinite(d);
    dmin = fmin(dmin, d);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) dmin = fmin(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
  const bool nonfinite = __any_sync(0xffffffffu, !finite);
  double zs = 0.0, qs = 0.0;
  for (int i = lane; i < nrow; i += 32) {
    const double e = exp(-lam * (Dt[i] - dmin));
    zs += e;
    qs += q[off + i] * e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    zs += __shfl_xor_sync(0xffffffffu, zs, o);
    qs += __shfl_xor_sync(0xffffffffu, qs, o);
  }
  const double sval = qs / zs;
  const double zval = dmin - log(zs) / lam;
  double acc[44];
#pragma unroll
  for (int e = 0; e < 44; ++e) acc[e] = 0.0;
  int total = 0;
  for (int b0 = 0; b0 < nrow; b0 += 32) {
    const int i = b0 + lane;
    const double di = i < nrow ? Dt[i] : 0.0;
    const bool sig = i < nrow && lam * (di - dmin) <= cutoff;
    const unsigned bal = __ballot_sync(0xffffffffu, sig);
    if (sig) {
      const int pos = total + __popc(bal & ((1u << lane) - 1u));
      const double p = exp(-lam * (di - dmin)) / zs;
      const int li = off + i;
      const double cs = -lam * p * (q[li] - sval);
      const double cz = p;
      double Rh[9], Rr[9];
      if (approx) {
#pragma unroll
        for (int e = 0; e < 9; ++e) Rr[e] = R[((int64_t)r * ld + i) * 9 + e];
        mat3_mul(Rxy, Rr, Rh);
      } else {
#pragma unroll
        for (int e = 0; e < 9; ++e) Rh[e] = R[((int64_t)t * ld + i) * 9 + e];
      }
      if (pos < cap) {
        sig_idx[(int64_t)tl * cap + pos] = li;
        double* co = sig_coef + ((int64_t)tl * cap + pos) * 18;
#pragma unroll
        for (int e = 0; e < 9; ++e) { co[e] = cs * Rh[e]; co[9 + e] = cz * Rh[e]; }
      }
      acc[0] += cs;
      acc[1] += cz;
      const double wb0 = lwbar[3 * li], wb1 = lwbar[3 * li + 1], wb2 = lwbar[3 * li + 2];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const double rw = Rh[a * 3] * wb0 + Rh[a * 3 + 1] * wb1 + Rh[a * 3 + 2] * wb2;
        acc[2 + a] += cs * rw;
        acc[5 + a] += cz * rw;
      }
      if (approx) {
        const double* Si = S + ((int64_t)t * ld + i) * 9;
        const double* m = lmom + 6 * (int64_t)li;
        const double A[9] = {m[0], m[1], m[2], m[1], m[3], m[4], m[2], m[4], m[5]};
        double SRt[9], RA[9], RAR[9];
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            SRt[a * 3 + b] = Si[a * 3] * Rr[b * 3] + Si[a * 3 + 1] * Rr[b * 3 + 1] + Si[a * 3 + 2] * Rr[b * 3 + 2];
        mat3_mul(Rr, A, RA);
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
          for (int b = 0; b < 3; ++b)
            RAR[a * 3 + b] = RA[a * 3] * Rr[b * 3] + RA[a * 3 + 1] * Rr[b * 3 + 1] + RA[a * 3 + 2] * Rr[b * 3 + 2];
#pragma unroll
        for (int e = 0; e < 9; ++e) {
          acc[8 + e] += cs * SRt[e];
          acc[17 + e] += cz * SRt[e];
          acc[26 + e] += cs * RAR[e];
          acc[35 + e] += cz * RAR[e];
        }
      }
    }
    total += __popc(bal);
  }
#pragma unroll
  for (int e = 0; e < 8; ++e)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
  if (approx) {  // warp-uniform
#pragma unroll
    for (int e = 8; e < 44; ++e)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], o);
  }
  if (lane != 0) return;
  s_out[t] = sval;
  z_out[t] = zval;
  nsig[tl] = min(total, cap);
  double* fv = fvec + (int64_t)tl * FVEC;
  const double fw[3] = {fwbar[3 * t], fwbar[3 * t + 1], fwbar[3 * t + 2]};
  double corr[2][3], vv[2][4];
  for (int c = 0; c < 2; ++c) {
    const double sumc = acc[c];
    for (int a = 0; a < 3; ++a) corr[c][a] = 2.0 * (sumc * fw[a] - acc[2 + 3 * c + a]);
    vv[c][0] = vv[c][1] = vv[c][2] = vv[c][3] = 0.0;
  }
  if (approx) {
    const double* e = xyeig + (int64_t)t * 20;
    double q0[4], qm[3][4], inv[3];
    for (int rr = 0; rr < 4; ++rr) q0[rr] = e[4 + rr * 4];
    for (int m = 0; m < 3; ++m) {
      for (int rr = 0; rr < 4; ++rr) qm[m][rr] = e[4 + rr * 4 + m + 1];
      inv[m] = 1.0 / (e[0] - e[m + 1]);
    }
    double J[4][9];
    rot_quat_jacobian(q0, J);
    const double yw[3] = {fwbar[3 * r], fwbar[3 * r + 1], fwbar[3 * r + 2]};
    for (int c = 0; c < 2; ++c) {
      const double* SR = acc + 8 + 9 * c;
      const double* RAR = acc + 26 + 9 * c;
      double XR[9], M[9];
      mat3_mul(Rxy, RAR, XR);
      for (int k = 0; k < 9; ++k) M[k] = -2.0 * (SR[k] - XR[k]);
      double g[4];
      for (int cc = 0; cc < 4; ++cc) {
        double sacc = 0.0;
        for (int k = 0; k < 9; ++k) sacc += M[k] * J[cc][k];
        g[cc] = sacc;
      }
      for (int m = 0; m < 3; ++m) {
        const double h = (qm[m][0] * g[0] + qm[m][1] * g[1] + qm[m][2] * g[2] + qm[m][3] * g[3]) * inv[m];
        for (int rr = 0; rr < 4; ++rr) vv[c][rr] += h * qm[m][rr];
      }
      double dsum[3];
      dk_contract(vv[c], q0, 1.0, fw, yw, dsum);
      for (int a = 0; a < 3; ++a) corr[c][a] += dsum[a];
    }
  }
  fv[0] = acc[0];
  fv[1] = acc[1];
  for (int a = 0; a < 3; ++a) { fv[2 + a] = corr[0][a]; fv[5 + a] = corr[1][a]; }
  for (int rr = 0; rr < 4; ++rr) { fv[8 + rr] = vv[0][rr]; fv[12 + rr] = vv[1][rr]; }
  if (flags) {
    uint8_t f = 0;
    if (total > cap) f |= kFlagSigOverflow;
    if (nonfinite || !isfinite(sval) || !isfinite(zval)) f |= kFlagNonFinite;
    flags[tl] = f;
  }
}

cudaError_t launch_cv_weights(int T, int t0, int L, double lam, double cutoff, int cap, int ld, const int* rowlo,
                              const int* rowcnt, double* D, const double* q,
                              const double* R, const double* fwbar, const double* lwbar, const uint8_t* refresh,
                              const int* ridx, const double* S, const double* rxy, const double* xyeig,
                              const double* gx, const double* ga, const double* lmom, double* s, double* z,
                              int* sig_idx, double* sig_coef, int* nsig, double* fvec, uint8_t* flags,
                              cudaStream_t stream, const int* nb_idx, const int* nb_row, int nb_m, int dmode) {
  if (T <= 0) return cudaSuccess;
  if (!refresh && !nb_idx && dmode == 0 && rowlo && rowcnt) {
    cv_weights_warp_kernel<<<(T + WWPB - 1) / WWPB, WWPB * 32, 0, stream>>>(
        T, t0, lam, cutoff, cap, ld, rowlo, rowcnt, D, q, R, fwbar, lwbar, s, z, sig_idx, sig_coef, nsig, fvec, flags);
    return cudaGetLastError();
  }
  if (refresh && !nb_idx && dmode == 0 && getenv("MC_WEIGHTS_BLOCK") == nullptr) {
    cv_weights_close_warp_kernel<<<(T + WWPB - 1) / WWPB, WWPB * 32, 0, stream>>>(
        T, t0, lam, cutoff, cap, ld, rowlo, rowcnt, L, D, q, R, fwbar, lwbar, refresh, ridx, S, rxy, xyeig, gx, ga,
        lmom, s, z, sig_idx, sig_coef, nsig, fvec, flags);
    return cudaGetLastError();
  }
  cv_weights_kernel<<<T, WNT, 0, stream>>>(T, t0, L, lam, cutoff, cap, ld, NbArgs{nb_idx, nb_row, nb_m, dmode}, rowlo,
                                           rowcnt, D, q, R, fwbar, lwbar, refresh, ridx, S, rxy,
                                           xyeig, gx, ga, lmom, s, z, sig_idx, sig_coef, nsig, fvec, flags);
  return cudaGetLastError();
}

// Landmark-sharded evaluation: shard g computed s_g, z_g and
// its coefficients cs, cz against its own landmarks.  With the merged s and
// w_g = Z_g / Z, the global coefficients of its landmarks are
//   cs' = w_g (cs - lam (s_g - s) cz) = alpha (cs + beta cz),   cz' = alpha cz,
// and every per-entry / per-frame quantity of the gradient pass is linear in
// (cs, cz): sig_coef [.., 0:9 | 9:18], fvec [0 | 1], [2:5 | 5:8], [8:12 | 12:16].
__global__ void __launch_bounds__(256)
shard_rescale_kernel(int T, int cap, const int* __restrict__ nsig, const double* __restrict__ alpha,
                     const double* __restrict__ beta, double* __restrict__ sig_coef, double* __restrict__ fvec) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (t >= T) return;
  const double a = alpha[t], b = beta[t];
  const int ns = nsig[t];
  double* co = sig_coef + (int64_t)t * cap * 18;
  for (int e = lane; e < ns * 9; e += 32) {
    const int i = e / 9, k = e - 9 * i;
    const double cs = co[i * 18 + k], cz = co[i * 18 + 9 + k];
    co[i * 18 + k] = a * (cs + b * cz);
    co[i * 18 + 9 + k] = a * cz;
  }
  if (lane < 8) {
    // (s, z) pairs of fvec: (0, 1), (2..4, 5..7), (8..11, 12..15)
    double* fv = fvec + (int64_t)t * FVEC;
    const int is = lane == 0 ? 0 : (lane < 4 ? 1 + lane : 4 + lane);
    const int iz = lane == 0 ? 1 : (lane < 4 ? 4 + lane : 8 + lane);
    const double cs = fv[is], cz = fv[iz];
    fv[is] = a * (cs + b * cz);
    fv[iz] = a * cz;
  }
}

cudaError_t launch_shard_rescale(int T, int cap, const int* nsig, const double* alpha, const double* beta,
                                 double* sig_coef, double* fvec, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  shard_rescale_kernel<<<(T + 7) / 8, 256, 0, stream>>>(T, cap, nsig, alpha, beta, sig_coef, fvec);
  return cudaGetLastError();
}

namespace {
constexpr int GNT = 128, APT = 4, GCH = 64;
}

template <typename OT>
__global__ void __launch_bounds__(GNT)
cv_grad_kernel(int n, int npad, int cap, const double* __restrict__ fpl, const double* __restrict__ lpl,
               const double* __restrict__ w, const double* __restrict__ wa, const int* __restrict__ sig_idx,
               const double* __restrict__ sig_coef, const int* __restrict__ nsig, const double* __restrict__ fvec,
               const uint8_t* __restrict__ refresh, const int* __restrict__ ridx, const double* __restrict__ xyeig,
               OT* __restrict__ ds, OT* __restrict__ dz, const float* __restrict__ fraw,
               const double* __restrict__ fcen, const float* __restrict__ lraw, const double* __restrict__ lcen,
               const int* __restrict__ perm) {
  // Coordinates come either from centred fp64 planes (fpl/lpl) or, on the
  // fp32 path, from the raw AoS input recentred on the fly with the fp64
  // centroids (fraw/fcen, lraw/lcen) — no fp64 copy of the big operands.
  __shared__ double sc[GCH * 18];
  __shared__ int si[GCH];
  const int t = perm ? perm[blockIdx.x] : blockIdx.x;  // sorted order: neighbours share landmarks in L2
  const int k0 = blockIdx.y * GNT * APT;
  const int tid = threadIdx.x;
  const int ns = nsig[t];
  double us[APT][3], uz[APT][3];
#pragma unroll
  for (int m = 0; m < APT; ++m)
#pragma unroll
    for (int a = 0; a < 3; ++a) us[m][a] = uz[m][a] = 0.0;
  for (int c0 = 0; c0 < ns; c0 += GCH) {
    const int cn = min(GCH, ns - c0);
    __syncthreads();
    for (int e = tid; e < cn * 18; e += GNT) sc[e] = sig_coef[((int64_t)t * cap + c0) * 18 + e];
    for (int e = tid; e < cn; e += GNT) si[e] = sig_idx[(int64_t)t * cap + c0 + e];
    __syncthreads();
    for (int e = 0; e < cn; ++e) {
      const int li = si[e];
      const double* a = lpl ? lpl + (int64_t)li * 3 * npad : nullptr;
      const float* ar = lpl ? nullptr : lraw + (int64_t)li * n * 3;
      const double c0 = lpl ? 0.0 : lcen[3 * li], c1 = lpl ? 0.0 : lcen[3 * li + 1], c2 = lpl ? 0.0 : lcen[3 * li + 2];
      const double* C = sc + e * 18;
#pragma unroll
      for (int m = 0; m < APT; ++m) {
        const int k = k0 + tid + m * GNT;
        if (k < n) {
          double a0, a1, a2;
          if (a) {
            a0 = a[k]; a1 = a[npad + k]; a2 = a[2 * npad + k];
          } else {
            a0 = (double)ar[3 * k] - c0; a1 = (double)ar[3 * k + 1] - c1; a2 = (double)ar[3 * k + 2] - c2;
          }
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            us[m][b] = fma(C[b * 3], a0, fma(C[b * 3 + 1], a1, fma(C[b * 3 + 2], a2, us[m][b])));
            uz[m][b] = fma(C[9 + b * 3], a0, fma(C[9 + b * 3 + 1], a1, fma(C[9 + b * 3 + 2], a2, uz[m][b])));
          }
        }
      }
    }
  }
  const double* fv = fvec + (int64_t)t * FVEC;
  const bool approx = refresh && !refresh[t];
  double q0[4] = {0, 0, 0, 0};
  const double* y = nullptr;
  if (approx) {
    const double* e = xyeig + (int64_t)t * 20;
#pragma unroll
    for (int rr = 0; rr < 4; ++rr) q0[rr] = e[4 + rr * 4];
    y = fpl + (int64_t)ridx[t] * 3 * npad;
  }
  const double* x = fpl ? fpl + (int64_t)t * 3 * npad : nullptr;
  const float* xr = fpl ? nullptr : fraw + (int64_t)t * n * 3;
  const double fc0 = fpl ? 0.0 : fcen[3 * t], fc1 = fpl ? 0.0 : fcen[3 * t + 1], fc2 = fpl ? 0.0 : fcen[3 * t + 2];
  const double vs[4] = {fv[8], fv[9], fv[10], fv[11]};
  const double vz[4] = {fv[12], fv[13], fv[14], fv[15]};
#pragma unroll
  for (int m = 0; m < APT; ++m) {
    const int k = k0 + tid + m * GNT;
    if (k >= n) continue;
    const double wk = w[k], wak = wa[k];
    double xk[3];
    if (x) {
      xk[0] = x[k]; xk[1] = x[npad + k]; xk[2] = x[2 * npad + k];
    } else {
      xk[0] = (double)xr[3 * k] - fc0; xk[1] = (double)xr[3 * k + 1] - fc1; xk[2] = (double)xr[3 * k + 2] - fc2;
    }
    double gs[3], gz[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      gs[a] = 2.0 * wk * (fv[0] * xk[a] - us[m][a]) - wak * fv[2 + a];
      gz[a] = 2.0 * wk * (fv[1] * xk[a] - uz[m][a]) - wak * fv[5 + a];
    }
    if (approx) {
      const double yk[3] = {y[k], y[npad + k], y[2 * npad + k]};
      double d[3];
      dk_contract(vs, q0, wk, xk, yk, d);
#pragma unroll
      for (int a = 0; a < 3; ++a) gs[a] += d[a];
      dk_contract(vz, q0, wk, xk, yk, d);
#pragma unroll
      for (int a = 0; a < 3; ++a) gz[a] += d[a];
    }
    OT* os = ds + ((int64_t)t * n + k) * 3;
    OT* oz = dz + ((int64_t)t * n + k) * 3;
#pragma unroll
    for (int a = 0; a < 3; ++a) { os[a] = (OT)gs[a]; oz[a] = (OT)gz[a]; }
  }
}

cudaError_t launch_cv_grad(int T, int n, int npad, int cap, const double* fpl, const double* lpl, const double* w,
                           const double* wa, const int* sig_idx, const double* sig_coef, const int* nsig,
                           const double* fvec, const uint8_t* refresh, const int* ridx, const double* xyeig,
                           void* ds, void* dz, int out_f32, const float* fraw, const double* fcen,
                           const float* lraw, const double* lcen, const int* perm, cudaStream_t stream) {
  if (T <= 0 || n <= 0) return cudaSuccess;
  dim3 grid(T, (n + GNT * APT - 1) / (GNT * APT));
  if (out_f32)
    cv_grad_kernel<float><<<grid, GNT, 0, stream>>>(n, npad, cap, fpl, lpl, w, wa, sig_idx, sig_coef, nsig, fvec,
                                                    refresh, ridx, xyeig, (float*)ds, (float*)dz, fraw, fcen, lraw,
                                                    lcen, perm);
  else
    cv_grad_kernel<double><<<grid, GNT, 0, stream>>>(n, npad, cap, fpl, lpl, w, wa, sig_idx, sig_coef, nsig, fvec,
                                                     refresh, ridx, xyeig, (double*)ds, (double*)dz, fraw, fcen, lraw,
                                                     lcen, perm);
  return cudaGetLastError();
}

// Eq. 6 dR_xy term of the non-refresh frames, added after the contraction part of
// the gradient came from the DMMA kernel (cv_grad_dmma_kernel).  Same closed form as
// the approx branch of cv_grad_kernel, on raw fp32 coordinates recentred with the
// fp64 centroids: x = frame t0 + t, y = its close structure ridx[t0 + t].
template <typename OT>
__global__ void __launch_bounds__(256)
close_grad_fix_kernel(int t0, int n, const uint8_t* __restrict__ refresh, const int* __restrict__ ridx,
                      const double* __restrict__ xyeig, const double* __restrict__ fvec, const double* __restrict__ w,
                      const float* __restrict__ fraw, const double* __restrict__ fcen, OT* __restrict__ ds,
                      OT* __restrict__ dz) {
  const int tl = blockIdx.y;
  const int t = t0 + tl;
  if (refresh[t]) return;
  const int r = ridx[t];
  const double* e = xyeig + (int64_t)t * 20;
  double q0[4];
#pragma unroll
  for (int rr = 0; rr < 4; ++rr) q0[rr] = e[4 + rr * 4];
  const double* fv = fvec + (int64_t)tl * FVEC;
  const double vs[4] = {fv[8], fv[9], fv[10], fv[11]};
  const double vz[4] = {fv[12], fv[13], fv[14], fv[15]};
  const double cx[3] = {fcen[3 * t], fcen[3 * t + 1], fcen[3 * t + 2]};
  const double cy[3] = {fcen[3 * r], fcen[3 * r + 1], fcen[3 * r + 2]};
  const float* xr = fraw + (int64_t)t * n * 3;
  const float* yr = fraw + (int64_t)r * n * 3;
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    double xk[3], yk[3], d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      xk[a] = (double)xr[3 * k + a] - cx[a];
      yk[a] = (double)yr[3 * k + a] - cy[a];
    }
    const double wk = w[k];
    OT* os = ds + ((int64_t)t * n + k) * 3;
    OT* oz = dz + ((int64_t)t * n + k) * 3;
    dk_contract(vs, q0, wk, xk, yk, d);
#pragma unroll
    for (int a = 0; a < 3; ++a) os[a] = (OT)((double)os[a] + d[a]);
    dk_contract(vz, q0, wk, xk, yk, d);
#pragma unroll
    for (int a = 0; a < 3; ++a) oz[a] = (OT)((double)oz[a] + d[a]);
  }
}

cudaError_t launch_close_grad_fix(int T, int t0, int n, const uint8_t* refresh, const int* ridx, const double* xyeig,
                                  const double* fvec, const double* w, const float* fraw, const double* fcen, void* ds,
                                  void* dz, int out_f32, cudaStream_t stream) {
  if (T <= 0 || n <= 0) return cudaSuccess;
  if (T > 65535) {
    for (int c = 0; c < T; c += 65535) {
      cudaError_t e = launch_close_grad_fix(std::min(65535, T - c), t0 + c, n, refresh, ridx, xyeig,
                                            fvec + (int64_t)c * FVEC, w, fraw, fcen, ds, dz, out_f32, stream);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  const dim3 grid((unsigned)std::min(8, (n + 255) / 256), (unsigned)T);
  if (out_f32)
    close_grad_fix_kernel<float><<<grid, 256, 0, stream>>>(t0, n, refresh, ridx, xyeig, fvec, w, fraw, fcen,
                                                            (float*)ds, (float*)dz);
  else
    close_grad_fix_kernel<double><<<grid, 256, 0, stream>>>(t0, n, refresh, ridx, xyeig, fvec, w, fraw, fcen,
                                                             (double*)ds, (double*)dz);
  return cudaGetLastError();
}

}  // namespace mc
