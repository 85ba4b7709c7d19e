// Per-pair distance results of the reference-facing API (SPEC.md msd-engine):
//   exact_distance  (Eq. 3/4)  value + gradient
//   approx_distance (Eq. 5/6)  value + gradient
// and the property-map reduction over supplied DistanceResults
// plus the path-CV z.
//
// pair_grad_kernel: grid (P, atom blocks).  For pair p = (frame xi[p],
// landmark ai[p]) with rotation Rhat[p] it writes, w.r.t. the raw frame
// coordinates,
//   G_k = 2 w_k (x_k - Rhat a_k) [+ v^T dK_k q0  on approximate pairs]
//         - w'_k sum_j G_j
// where on approximate pairs Rhat = R_xy R_s (R_s the saved R_{a y}) and
//   M = -2 [ S R_s^T - R_xy R_s A R_s^T ],  g_c = <M, dR/dq_c>,
//   v = sum_m (q_m . g)/(l_0 - l_m) q_m
// using the x<->y spectrum xyeig and close structure y = frame yi[p].
// It also writes the distance value (exact: from D; approx: Eq. 5 via S).
#include "mc_math.cuh"

namespace mc {

__device__ __forceinline__ void m3(const double* a, const double* b, double* c) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[i * 3 + j] = a[i * 3] * b[j] + a[i * 3 + 1] * b[3 + j] + a[i * 3 + 2] * b[6 + j];
}

__global__ void __launch_bounds__(128)
pair_grad_kernel(int n, int npad, const double* __restrict__ xpl, const double* __restrict__ apl,
                 const int* __restrict__ xi, const int* __restrict__ ai, const double* __restrict__ rot,
                 const double* __restrict__ w, const double* __restrict__ wa, const double* __restrict__ xwbar,
                 const double* __restrict__ awbar, const int* __restrict__ approx, const int* __restrict__ yi,
                 const double* __restrict__ S, const double* __restrict__ amom, const double* __restrict__ xyeig,
                 const double* __restrict__ rxy, const double* __restrict__ gx, const double* __restrict__ ga,
                 double* __restrict__ value, double* __restrict__ grad) {
  __shared__ double sh[9 + 3 + 4 + 4];  // Rhat, corr, v, q0
  __shared__ int s_approx;
  const int p = blockIdx.x;
  const int x_s = xi[p], a_s = ai[p];
  const bool ap = approx && approx[p];
  if (threadIdx.x == 0) {
    double Rh[9], Rs[9], Rx[9];
    for (int e = 0; e < 9; ++e) Rs[e] = rot[(int64_t)p * 9 + e];
    double v[4] = {0, 0, 0, 0}, q0[4] = {0, 0, 0, 0};
    double corr[3];
    const double* xw = xwbar + 3 * (int64_t)x_s;
    const double* aw = awbar + 3 * (int64_t)a_s;
    if (ap) {
      for (int e = 0; e < 9; ++e) Rx[e] = rxy[(int64_t)p * 9 + e];
      m3(Rx, Rs, Rh);
      const double* Sp = S + (int64_t)p * 9;
      const double* mm = amom + 6 * (int64_t)a_s;
      const double A[9] = {mm[0], mm[1], mm[2], mm[1], mm[3], mm[4], mm[2], mm[4], mm[5]};
      double SRt[9], RA[9], RAR[9], XR[9], M[9];
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          SRt[a * 3 + b] = Sp[a * 3] * Rs[b * 3] + Sp[a * 3 + 1] * Rs[b * 3 + 1] + Sp[a * 3 + 2] * Rs[b * 3 + 2];
      m3(Rs, A, RA);
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          RAR[a * 3 + b] = RA[a * 3] * Rs[b * 3] + RA[a * 3 + 1] * Rs[b * 3 + 1] + RA[a * 3 + 2] * Rs[b * 3 + 2];
      m3(Rx, RAR, XR);
      for (int e = 0; e < 9; ++e) M[e] = -2.0 * (SRt[e] - XR[e]);
      const double* ev = xyeig + (int64_t)p * 20;
      for (int r = 0; r < 4; ++r) q0[r] = ev[4 + r * 4];
      double J[4][9];
      rot_quat_jacobian(q0, J);
      double g[4];
      for (int c = 0; c < 4; ++c) {
        double acc = 0.0;
        for (int e = 0; e < 9; ++e) acc += M[e] * J[c][e];
        g[c] = acc;
      }
      for (int m = 1; m < 4; ++m) {
        const double h = (ev[4 + m] * g[0] + ev[8 + m] * g[1] + ev[12 + m] * g[2] + ev[16 + m] * g[3]) / (ev[0] - ev[m]);
        for (int r = 0; r < 4; ++r) v[r] += h * ev[4 + r * 4 + m];
      }
      double dot = 0.0;
      for (int e = 0; e < 9; ++e) dot += Rh[e] * Sp[e];
      value[p] = gx[x_s] + ga[a_s] - 2.0 * dot;
    } else {
      for (int e = 0; e < 9; ++e) Rh[e] = Rs[e];
    }
    for (int a = 0; a < 3; ++a) corr[a] = 2.0 * (xw[a] - (Rh[a * 3] * aw[0] + Rh[a * 3 + 1] * aw[1] + Rh[a * 3 + 2] * aw[2]));
    if (ap) {
      double d3[3];
      dk_contract(v, q0, 1.0, xw, xwbar + 3 * (int64_t)yi[p], d3);
      for (int a = 0; a < 3; ++a) corr[a] += d3[a];
    }
    for (int e = 0; e < 9; ++e) sh[e] = Rh[e];
    for (int a = 0; a < 3; ++a) sh[9 + a] = corr[a];
    for (int r = 0; r < 4; ++r) { sh[12 + r] = v[r]; sh[16 + r] = q0[r]; }
    s_approx = ap;
  }
  __syncthreads();
  const int k = blockIdx.y * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const double* x = xpl + (int64_t)x_s * 3 * npad;
  const double* a = apl + (int64_t)a_s * 3 * npad;
  const double xk[3] = {x[k], x[npad + k], x[2 * npad + k]};
  const double ak[3] = {a[k], a[npad + k], a[2 * npad + k]};
  const double wk = w[k], wak = wa[k];
  double g[3];
#pragma unroll
  for (int b = 0; b < 3; ++b)
    g[b] = 2.0 * wk * (xk[b] - (sh[b * 3] * ak[0] + sh[b * 3 + 1] * ak[1] + sh[b * 3 + 2] * ak[2])) - wak * sh[9 + b];
  if (s_approx) {
    const double* y = xpl + (int64_t)yi[p] * 3 * npad;
    const double yk[3] = {y[k], y[npad + k], y[2 * npad + k]};
    double d3[3];
    dk_contract(sh + 12, sh + 16, wk, xk, yk, d3);
#pragma unroll
    for (int b = 0; b < 3; ++b) g[b] += d3[b];
  }
  double* o = grad + ((int64_t)p * n + k) * 3;
#pragma unroll
  for (int b = 0; b < 3; ++b) o[b] = g[b];
}

cudaError_t launch_pair_grad(int64_t P, int n, int npad, const double* xpl, const double* apl, const int* xi,
                             const int* ai, const double* rot, const double* w, const double* wa, const double* xwbar,
                             const double* awbar, const int* approx, const int* yi, const double* S,
                             const double* amom, const double* xyeig, const double* rxy, const double* gx,
                             const double* ga, double* value, double* grad, cudaStream_t stream) {
  if (P <= 0) return cudaSuccess;
  dim3 grid((unsigned)P, (n + 127) / 128);
  pair_grad_kernel<<<grid, 128, 0, stream>>>(n, npad, xpl, apl, xi, ai, rot, w, wa, xwbar, awbar, approx, yi, S, amom,
                                             xyeig, rxy, gx, ga, value, grad);
  return cudaGetLastError();
}

// property_map over supplied distances + path-CV z:
// D [L], grads [L, n, 3] (nullable), q [L] -> out {s, z}, ds, dz [n, 3].
__global__ void __launch_bounds__(256)
property_map_kernel(int L, int n, const double* __restrict__ D, const double* __restrict__ grads,
                    const double* __restrict__ q, double lam, double* __restrict__ out, double* __restrict__ ds,
                    double* __restrict__ dz) {
  __shared__ double scratch[8];
  double dmin = INFINITY;
  for (int i = threadIdx.x; i < L; i += 256) dmin = fmin(dmin, D[i]);
  dmin = block_min<256>(dmin, scratch);
  double zs = 0.0, qs = 0.0;
  for (int i = threadIdx.x; i < L; i += 256) {
    const double e = exp(-lam * (D[i] - dmin));
    zs += e;
    qs += q[i] * e;
  }
  zs = block_sum<256>(zs, scratch);
  qs = block_sum<256>(qs, scratch);
  const double s = qs / zs;
  if (threadIdx.x == 0) {
    out[0] = s;
    out[1] = dmin - log(zs) / lam;
  }
  if (!grads) return;
  for (int e = threadIdx.x; e < n * 3; e += 256) {
    double as = 0.0, az = 0.0;
    for (int i = 0; i < L; ++i) {
      const double p = exp(-lam * (D[i] - dmin)) / zs;
      const double g = grads[(int64_t)i * n * 3 + e];
      as += -lam * p * (q[i] - s) * g;
      az += p * g;
    }
    ds[e] = as;
    dz[e] = az;
  }
}

cudaError_t launch_property_map(int L, int n, const double* D, const double* grads, const double* q, double lam,
                                double* out, double* ds, double* dz, cudaStream_t stream) {
  if (L <= 0) return cudaSuccess;
  property_map_kernel<<<1, 256, 0, stream>>>(L, n, D, grads, q, lam, out, ds, dz);
  return cudaGetLastError();
}

}  // namespace mc
