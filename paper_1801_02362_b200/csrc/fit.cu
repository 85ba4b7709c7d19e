// K3 — per-pair quaternion fit from the 3x3 covariance (fp64).
//
// Replaces jacobi_eigh + _quat_to_rot + the MSD read-out of kearsley_fit
// (geometry.py:106-164, 227-249).  The hot path uses Newton on Horn's
// characteristic quartic for lambda_max plus the adjugate eigenvector
// (mc_math.cuh); pairs whose eigenvector is ill-conditioned fall back to the
// reference's cyclic Jacobi on K.  The per-pair API path (kearsley_fit,
// jacobi_eigh, rot_grad) runs the Jacobi solver so its full spectrum and
// eigenvectors follow the reference algorithm.
#include "mc_math.cuh"

namespace mc {

// Jacobi fallback for a single pair: fills msd and quat.
__device__ __forceinline__ bool fit_jacobi(const double* S, double gx, double ga, double* msd, double q[4]) {
  double k[4][4], V[4][4], w[4];
  kearsley_from_S(S, gx, ga, k);
  const bool ok = jacobi4(k, w, V);
  *msd = w[0];
  q[0] = V[0][0]; q[1] = V[1][0]; q[2] = V[2][0]; q[3] = V[3][0];
  return ok;
}

// Dense (frame x landmark) fit: thread per pair; rows with rowmask[t]==0 skipped.
__global__ void __launch_bounds__(256)
fit_dense_kernel(const double* __restrict__ S, int T, int L, const double* __restrict__ gx,
                 const double* __restrict__ ga, const uint8_t* __restrict__ rowmask, double* __restrict__ D,
                 double* __restrict__ rot, double* __restrict__ quat, uint8_t* __restrict__ flags) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= (int64_t)T * L) return;
  const int t = (int)(p / L);
  const int l = (int)(p - (int64_t)t * L);
  if (rowmask && !rowmask[t]) return;
  double s[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) s[e] = S[p * 9 + e];
  const bool need_q = rot || quat;
  double q[4];
  bool ill = false;
  double msd = fit_fast(s, gx[t], ga[l], need_q ? q : nullptr, &ill);
  uint8_t f = 0;
  if (ill) {
    if (!fit_jacobi(s, gx[t], ga[l], &msd, q)) f |= kFlagNoConverge;
    f |= kFlagAdjFallback;
  }
  if (!isfinite(msd)) f |= kFlagNonFinite;
  D[p] = msd;
  if (quat) {
#pragma unroll
    for (int e = 0; e < 4; ++e) quat[p * 4 + e] = q[e];
  }
  if (rot) {
    double r[9];
    quat_to_rot(q, r);
#pragma unroll
    for (int e = 0; e < 9; ++e) rot[p * 9 + e] = r[e];
  }
  if (flags) flags[p] = f;
}

cudaError_t launch_fit_dense(const double* S, int T, int L, const double* gx, const double* ga,
                             const uint8_t* rowmask, double* D, double* rot, double* quat, uint8_t* flags,
                             cudaStream_t stream) {
  const int64_t P = (int64_t)T * L;
  if (P <= 0) return cudaSuccess;
  fit_dense_kernel<<<(unsigned)((P + 255) / 256), 256, 0, stream>>>(S, T, L, gx, ga, rowmask, D, rot, quat, flags);
  return cudaGetLastError();
}

// Listed pairs, MSD only (Newton): D[p] from S[p], gx[xi[p]], ga[ai[p]].
// Negative indices produce NaN (used for window slots before the first frame).
__global__ void __launch_bounds__(256)
fit_list_msd_kernel(const double* __restrict__ S, int64_t P, const int* __restrict__ xi,
                    const int* __restrict__ ai, const double* __restrict__ gx, const double* __restrict__ ga,
                    double* __restrict__ D) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int xs = xi ? xi[p] : (int)p;
  const int as = ai ? ai[p] : (int)p;
  if (xs < 0 || as < 0) { D[p] = __longlong_as_double(0x7ff8000000000000LL); return; }
  double s[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) s[e] = S[p * 9 + e];
  bool ill;
  D[p] = fit_fast(s, gx[xs], ga[as], nullptr, &ill);
}

cudaError_t launch_fit_list_msd(const double* S, int64_t P, const int* xi, const int* ai, const double* gx,
                                const double* ga, double* D, cudaStream_t stream) {
  if (P <= 0) return cudaSuccess;
  fit_list_msd_kernel<<<(unsigned)((P + 255) / 256), 256, 0, stream>>>(S, P, xi, ai, gx, ga, D);
  return cudaGetLastError();
}

// Full spectrum (reference Jacobi on K): eig[p] = {eigvals[4], eigvecs row-major [4][4]},
// quat = eigvecs[:,0], rot = R(quat).  flags: no-convergence, degeneracy
// (gap < 1e-9, only meaningful when derivatives are requested).
__global__ void __launch_bounds__(128)
fit_full_kernel(const double* __restrict__ S, int64_t P, const int* __restrict__ xi, const int* __restrict__ ai,
                const double* __restrict__ gx, const double* __restrict__ ga, double* __restrict__ eig,
                double* __restrict__ quat, double* __restrict__ rot, uint8_t* __restrict__ flags) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int xs = xi ? xi[p] : (int)p;
  const int as = ai ? ai[p] : (int)p;
  double k[4][4], V[4][4], w[4];
  kearsley_from_S(S + p * 9, gx[xs], ga[as], k);
  const bool ok = jacobi4(k, w, V);
  uint8_t f = ok ? 0 : kFlagNoConverge;
  if (w[1] - w[0] < kDegeneracyTol) f |= kFlagDegenerate;
  if (!isfinite(w[0]) || !isfinite(w[3])) f |= kFlagNonFinite;
  if (eig) {
    double* e = eig + p * 20;
#pragma unroll
    for (int i = 0; i < 4; ++i) e[i] = w[i];
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int c = 0; c < 4; ++c) e[4 + r * 4 + c] = V[r][c];
  }
  const double q[4] = {V[0][0], V[1][0], V[2][0], V[3][0]};
  if (quat) {
#pragma unroll
    for (int e = 0; e < 4; ++e) quat[p * 4 + e] = q[e];
  }
  if (rot) {
    double r[9];
    quat_to_rot(q, r);
#pragma unroll
    for (int e = 0; e < 9; ++e) rot[p * 9 + e] = r[e];
  }
  if (flags) flags[p] = f;
}

cudaError_t launch_fit_full(const double* S, int64_t P, const int* xi, const int* ai, const double* gx,
                            const double* ga, double* eig, double* quat, double* rot, uint8_t* flags,
                            cudaStream_t stream) {
  if (P <= 0) return cudaSuccess;
  fit_full_kernel<<<(unsigned)((P + 127) / 128), 128, 0, stream>>>(S, P, xi, ai, gx, ga, eig, quat, rot, flags);
  return cudaGetLastError();
}

// rot_grad[p, k, alpha, b, g] = dR_bg / dx_{k,alpha} (geometry.py:251-262):
//   dq = sum_{m>0} (q_m . dK_{k,alpha} q_0) / (lambda_0 - lambda_m) q_m,
//   dR = sum_c dq_c J_c.   Grid: (atom blocks, pairs).
__global__ void __launch_bounds__(128)
rot_grad_kernel(const double* __restrict__ xpl, const double* __restrict__ apl, const int* __restrict__ xi,
                const int* __restrict__ ai, int64_t P, int n, int npad, const double* __restrict__ w,
                const double* __restrict__ eig, double* __restrict__ out) {
  const int64_t p = blockIdx.x;
  const int k = blockIdx.y * blockDim.x + threadIdx.x;
  if (p >= P || k >= n) return;
  const int xs = xi ? xi[p] : (int)p;
  const int as = ai ? ai[p] : (int)p;
  const double* e = eig + p * 20;
  double q0[4], qm[3][4], inv[3];
#pragma unroll
  for (int r = 0; r < 4; ++r) q0[r] = e[4 + r * 4 + 0];
#pragma unroll
  for (int m = 0; m < 3; ++m) {
#pragma unroll
    for (int r = 0; r < 4; ++r) qm[m][r] = e[4 + r * 4 + m + 1];
    inv[m] = 1.0 / (e[0] - e[m + 1]);
  }
  double J[4][9];
  rot_quat_jacobian(q0, J);
  const double* x = xpl + (int64_t)xs * 3 * npad;
  const double* a = apl + (int64_t)as * 3 * npad;
  const double xk[3] = {x[k], x[npad + k], x[2 * npad + k]};
  const double ak[3] = {a[k], a[npad + k], a[2 * npad + k]};
  double coef[3][3];  // coef[m][alpha]
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    double c[3];
    dk_contract(qm[m], q0, w[k], xk, ak, c);
#pragma unroll
    for (int al = 0; al < 3; ++al) coef[m][al] = c[al] * inv[m];
  }
  double* o = out + ((int64_t)p * n + k) * 27;
#pragma unroll
  for (int al = 0; al < 3; ++al) {
    double dq[4];
#pragma unroll
    for (int r = 0; r < 4; ++r) dq[r] = coef[0][al] * qm[0][r] + coef[1][al] * qm[1][r] + coef[2][al] * qm[2][r];
#pragma unroll
    for (int bg = 0; bg < 9; ++bg)
      o[al * 9 + bg] =dq[0] * J[0][bg] + dq[1] * J[1][bg] + dq[2] * J[2][bg] + dq[3] * J[3][bg];
  }
}

cudaError_t launch_rot_grad(const double* xpl, const double* apl, const int* xi, const int* ai, int64_t P, int n,
                            int npad, const double* w, const double* eig, double* out, cudaStream_t stream) {
  if (P <= 0 || n <= 0) return cudaSuccess;
  dim3 grid((unsigned)P, (n + 127) / 128);
  rot_grad_kernel<<<grid, 128, 0, stream>>>(xpl, apl, xi, ai, P, n, npad, w, eig, out);
  return cudaGetLastError();
}

// jacobi_eigh on arbitrary symmetric 4x4 matrices (geometry.py:106-153).
__global__ void __launch_bounds__(128)
jacobi4_batch_kernel(const double* __restrict__ mats, int64_t B, double* __restrict__ vals,
                     double* __restrict__ vecs, uint8_t* __restrict__ flags) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  double a[4][4], V[4][4], w[4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) a[r][c] = mats[b * 16 + r * 4 + c];
  const bool ok = jacobi4(a, w, V);
#pragma unroll
  for (int i = 0; i < 4; ++i) vals[b * 4 + i] = w[i];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) vecs[b * 16 + r * 4 + c] = V[r][c];
  if (flags) flags[b] = ok ? 0 : kFlagNoConverge;
}

cudaError_t launch_jacobi4(const double* mats, int64_t B, double* vals, double* vecs, uint8_t* flags,
                           cudaStream_t stream) {
  if (B <= 0) return cudaSuccess;
  jacobi4_batch_kernel<<<(unsigned)((B + 127) / 128), 128, 0, stream>>>(mats, B, vals, vecs, flags);
  return cudaGetLastError();
}

// jacobi_eigh (geometry.py:106-153) for a general symmetric n x n matrix, one
// CTA per matrix (n <= 48): the same cyclic sweep order, rotation formula, tolerance floor
// max(tol, 4e-16 ||A||_F), stable ascending sort and largest-|component|-positive sign
// rule; each rotation updates the columns / rows / eigenvector columns with one thread per
// element (c x - s y without FMA contraction, as the reference's numpy expressions).
constexpr int kJnMax = 48;
__global__ void __launch_bounds__(kJnMax)
jacobi_n_kernel(const double* __restrict__ mats, int n, double tol, int max_sweeps, double* __restrict__ vals,
                double* __restrict__ vecs, uint8_t* __restrict__ flags) {
  __shared__ double a[kJnMax][kJnMax + 1], v[kJnMax][kJnMax + 1];
  __shared__ double red[kJnMax];
  __shared__ int s_done;
  const int b = blockIdx.x, k = threadIdx.x;
  const double* m = mats + (int64_t)b * n * n;
  for (int i = 0; i < n; ++i)
    if (k < n) {
      a[i][k] = m[i * n + k];
      v[i][k] = i == k ? 1.0 : 0.0;
    }
  __syncthreads();
  // Frobenius norm for the tolerance floor
  double fr = 0.0;
  if (k < n)
    for (int i = 0; i < n; ++i) fr = __fma_rn(a[i][k], a[i][k], fr);
  red[k] = fr;
  __syncthreads();
  if (k == 0) {
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += red[i];
    red[0] = fmax(tol, 4e-16 * sqrt(t));
  }
  __syncthreads();
  const double tl = red[0];
  __syncthreads();
  int converged = 0;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    double off = 0.0;
    if (k < n)
      for (int i = 0; i < n; ++i)
        if (i != k) off = __fma_rn(a[i][k], a[i][k], off);
    red[k] = off;
    __syncthreads();
    if (k == 0) {
      double t = 0.0;
      for (int i = 0; i < n; ++i) t += red[i];
      s_done = sqrt(t) < tl;
    }
    __syncthreads();
    if (s_done) { converged = 1; break; }
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a[p][q];
        __syncthreads();
        if (apq == 0.0) continue;  // uniform
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        const double t = copysign(1.0, theta) / (fabs(theta) + hypot(theta, 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), sn = t * c;
        if (k < n) {  // columns p, q
          const double xp = a[k][p], xq = a[k][q];
          a[k][p] = __dsub_rn(__dmul_rn(c, xp), __dmul_rn(sn, xq));
          a[k][q] = __dadd_rn(__dmul_rn(sn, xp), __dmul_rn(c, xq));
        }
        __syncthreads();
        if (k < n) {  // rows p, q
          const double xp = a[p][k], xq = a[q][k];
          a[p][k] = __dsub_rn(__dmul_rn(c, xp), __dmul_rn(sn, xq));
          a[q][k] = __dadd_rn(__dmul_rn(sn, xp), __dmul_rn(c, xq));
          const double vp = v[k][p], vq = v[k][q];
          v[k][p] = __dsub_rn(__dmul_rn(c, vp), __dmul_rn(sn, vq));
          v[k][q] = __dadd_rn(__dmul_rn(sn, vp), __dmul_rn(c, vq));
        }
        __syncthreads();
        if (k == 0) a[p][q] = a[q][p] = 0.0;
        __syncthreads();
      }
  }
  __syncthreads();
  if (k == 0) {
    // stable ascending sort of the diagonal (insertion sort keeps equal keys in order)
    int ord[kJnMax];
    for (int i = 0; i < n; ++i) ord[i] = i;
    for (int i = 1; i < n; ++i) {
      const int o = ord[i];
      int j = i - 1;
      while (j >= 0 && a[ord[j]][ord[j]] > a[o][o]) { ord[j + 1] = ord[j]; --j; }
      ord[j + 1] = o;
    }
    for (int j = 0; j < n; ++j) {
      const int c = ord[j];
      vals[(int64_t)b * n + j] = a[c][c];
      int im = 0;
      for (int i = 1; i < n; ++i)
        if (fabs(v[i][c]) > fabs(v[im][c])) im = i;  // first maximum, like np.argmax
      const double sg = v[im][c] < 0.0 ? -1.0 : 1.0;
      for (int i = 0; i < n; ++i) vecs[((int64_t)b * n + i) * n + j] = sg * v[i][c];
    }
    if (flags) flags[b] = converged ? 0 : kFlagNoConverge;
  }
}

cudaError_t launch_jacobi_n(const double* mats, int64_t B, int n, double tol, int max_sweeps, double* vals,
                            double* vecs, uint8_t* flags, cudaStream_t stream) {
  if (B <= 0) return cudaSuccess;
  if (n < 1 || n > kJnMax) return cudaErrorInvalidValue;
  jacobi_n_kernel<<<(unsigned)B, kJnMax, 0, stream>>>(mats, n, tol, max_sweeps, vals, vecs, flags);
  return cudaGetLastError();
}

}  // namespace mc
