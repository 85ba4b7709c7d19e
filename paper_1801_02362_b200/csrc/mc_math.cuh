// Per-pair fp64 quaternion-fit math shared by every kernel.
//
// Conventions follow the reference geometry module
// (/root/reference/pkg/src/metadyn_close/geometry.py):
//   * S[b*3+g] = sum_j w_j x_{j,b} a_{j,g}   (x fitted, a reference)
//   * Horn's 4x4 N(S) satisfies q^T N q = <R(q), S>_F with R(q) the
//     scalar-first quaternion rotation of geometry.py:156-164;
//   * Kearsley's K (geometry.py:180-196) equals (Gx + Ga) I - 2 N, so the
//     ascending eigenvalues of K are Gx + Ga - 2 mu (mu descending) and the
//     MSD is eigvals[0] = Gx + Ga - 2 lambda_max(N);
//   * eigenvectors are sign-normalised so the largest-|component| is
//     positive (geometry.py:149-152; ties -> first index, like np.argmax).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

namespace mc {

constexpr double kDegeneracyTol = 1e-9;  // geometry.py:22

// status bits written to per-item flag arrays
enum : uint8_t {
  kFlagDegenerate = 1,   // eigvals[1]-eigvals[0] < 1e-9 with derivatives requested
  kFlagNoConverge = 2,   // Jacobi did not converge in 60 sweeps
  kFlagNonFinite = 4,    // non-finite input or result
  kFlagAdjFallback = 8,  // adjugate eigenvector ill-conditioned; Jacobi used
  kFlagSigOverflow = 16, // significant-landmark list exceeded its capacity
};

struct Sym4 {
  double a00, a01, a02, a03, a11, a12, a13, a22, a23, a33;
};

// Horn's matrix from S (see header comment for the derivation).
__device__ __forceinline__ Sym4 horn(const double* S) {
  const double s00 = S[0], s01 = S[1], s02 = S[2];
  const double s10 = S[3], s11 = S[4], s12 = S[5];
  const double s20 = S[6], s21 = S[7], s22 = S[8];
  Sym4 n;
  n.a00 = s00 + s11 + s22;
  n.a01 = s21 - s12;
  n.a02 = s02 - s20;
  n.a03 = s10 - s01;
  n.a11 = s00 - s11 - s22;
  n.a12 = s01 + s10;
  n.a13 = s02 + s20;
  n.a22 = -s00 + s11 - s22;
  n.a23 = s12 + s21;
  n.a33 = -s00 - s11 + s22;
  return n;
}

// Largest eigenvalue of a traceless symmetric 4x4 by Newton on its
// characteristic polynomial P(l) = l^4 + c2 l^2 + c1 l + c0, started from
// an upper bound (monotone convergence from the right of the largest root):
// min(lam0, sqrt(3/4 tr N^2)) -- for a traceless 4x4, lmax^2 <= 3/4 sum l_i^2
// (exact when the three other eigenvalues are equal, e.g. identical
// structures), which cuts the iteration count for distant pairs, whose
// lmax sits far below the Cauchy-Schwarz bound (Gx + Ga) / 2.
// FAST (screening estimates only): stop at |step| <= 1e-10 |l| (quadratic
// convergence leaves ~1e-20 relative) and divide by a refined hardware
// reciprocal instead of the IEEE division.
struct Quartic {
  double c2, c1, c0;  // P(l) = l^4 + c2 l^2 + c1 l + c0
  double ub;          // sqrt(3/4 tr N^2) >= lambda_max
};

__device__ __forceinline__ Quartic charpoly(const Sym4& n) {
  // tr(N^2), tr(N^3), det(N)
  const double a00 = n.a00, a01 = n.a01, a02 = n.a02, a03 = n.a03;
  const double a11 = n.a11, a12 = n.a12, a13 = n.a13, a22 = n.a22, a23 = n.a23, a33 = n.a33;
  const double tr2 = a00 * a00 + a11 * a11 + a22 * a22 + a33 * a33 +
                     2.0 * (a01 * a01 + a02 * a02 + a03 * a03 + a12 * a12 + a13 * a13 + a23 * a23);
  // (N^2) rows needed for tr(N^3) = sum_ij (N^2)_ij N_ij
  const double b00 = a00 * a00 + a01 * a01 + a02 * a02 + a03 * a03;
  const double b11 = a01 * a01 + a11 * a11 + a12 * a12 + a13 * a13;
  const double b22 = a02 * a02 + a12 * a12 + a22 * a22 + a23 * a23;
  const double b33 = a03 * a03 + a13 * a13 + a23 * a23 + a33 * a33;
  const double b01 = a00 * a01 + a01 * a11 + a02 * a12 + a03 * a13;
  const double b02 = a00 * a02 + a01 * a12 + a02 * a22 + a03 * a23;
  const double b03 = a00 * a03 + a01 * a13 + a02 * a23 + a03 * a33;
  const double b12 = a01 * a02 + a11 * a12 + a12 * a22 + a13 * a23;
  const double b13 = a01 * a03 + a11 * a13 + a12 * a23 + a13 * a33;
  const double b23 = a02 * a03 + a12 * a13 + a22 * a23 + a23 * a33;
  const double tr3 = b00 * a00 + b11 * a11 + b22 * a22 + b33 * a33 +
                     2.0 * (b01 * a01 + b02 * a02 + b03 * a03 + b12 * a12 + b13 * a13 + b23 * a23);
  // det via 2x2 minors of rows (0,1) and (2,3)
  const double s0 = a00 * a11 - a01 * a01;
  const double s1 = a00 * a12 - a01 * a02;
  const double s2 = a00 * a13 - a01 * a03;
  const double s3 = a01 * a12 - a11 * a02;
  const double s4 = a01 * a13 - a11 * a03;
  const double s5 = a02 * a13 - a12 * a03;
  const double c5 = a22 * a33 - a23 * a23;
  const double c4 = a12 * a33 - a13 * a23;
  const double c3 = a12 * a23 - a13 * a22;
  const double c2m = a02 * a33 - a03 * a23;
  const double c1m = a02 * a23 - a03 * a22;
  const double c0m = a02 * a13 - a03 * a12;
  Quartic q;
  q.c0 = s0 * c5 - s1 * c4 + s2 * c3 + s3 * c2m - s4 * c1m + s5 * c0m;
  q.c2 = -0.5 * tr2;
  q.c1 = -tr3 / 3.0;
  q.ub = sqrt(0.75 * tr2) * (1.0 + 1e-12);
  return q;
}

__device__ __forceinline__ double newton_start(const Quartic& q, double lam0) {
  const double lam = fmin(lam0, q.ub);
  return lam == lam ? lam : lam0;
}

// One Newton step on P; returns true once converged (lam then final).
template <bool FAST>
__device__ __forceinline__ bool newton_step(const Quartic& q, double& lam) {
  const double l2 = lam * lam;
  const double b = (l2 + q.c2) * lam;
  const double a = b + q.c1;
  const double p = a * lam + q.c0;
  const double dp = 2.0 * l2 * lam + b + a;
  if (!(dp != 0.0)) return true;
  double delta;
  if (FAST) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(dp));
    r = fma(r, fma(-dp, r, 1.0), r);
    r = fma(r, fma(-dp, r, 1.0), r);
    delta = p * r;
    if (!isfinite(delta)) delta = p / dp;
  } else {
    delta = p / dp;
  }
  const double nl = lam - delta;
  lam = nl;
  return !(fabs(delta) > (FAST ? 1e-10 : 1e-15) * fabs(nl));
}

template <bool FAST = false>
__device__ __forceinline__ double newton_lmax(const Sym4& n, double lam0) {
  const Quartic q = charpoly(n);
  double lam = newton_start(q, lam0);
  for (int it = 0; it < 80; ++it)
    if (newton_step<FAST>(q, lam)) break;
  return lam;
}

// K independent pairs iterated in lockstep: the fp64 Newton chain is
// latency-bound, so interleaving K chains per thread fills the pipe, and a
// thread pays max (not sum) of the K iteration counts.  Screening estimates.
template <int K>
__device__ __forceinline__ void newton_lmax_batch(const Quartic (&q)[K], double (&lam)[K]) {
  unsigned done = 0;
  for (int it = 0; it < 80 && done != (1u << K) - 1u; ++it) {
#pragma unroll
    for (int i = 0; i < K; ++i)
      if (!((done >> i) & 1u) && newton_step<true>(q[i], lam[i])) done |= 1u << i;
  }
}

// Eigenvector of N for eigenvalue lam from the adjugate of (N - lam I):
// the column with the largest |diagonal| cofactor.  Returns the largest
// |diagonal| cofactor so the caller can judge conditioning.
__device__ __forceinline__ double adj_eigvec(const Sym4& n, double lam, double v[4]) {
  const double m00 = n.a00 - lam, m01 = n.a01, m02 = n.a02, m03 = n.a03;
  const double m11 = n.a11 - lam, m12 = n.a12, m13 = n.a13;
  const double m22 = n.a22 - lam, m23 = n.a23, m33 = n.a33 - lam;
  // symmetric: m10=m01, ...
  const double s0 = m00 * m11 - m01 * m01;
  const double s1 = m00 * m12 - m01 * m02;
  const double s2 = m00 * m13 - m01 * m03;
  const double s3 = m01 * m12 - m11 * m02;
  const double s4 = m01 * m13 - m11 * m03;
  const double s5 = m02 * m13 - m12 * m03;
  const double c5 = m22 * m33 - m23 * m23;
  const double c4 = m12 * m33 - m13 * m23;
  const double c3 = m12 * m23 - m13 * m22;
  const double c2 = m02 * m33 - m03 * m23;
  const double c1 = m02 * m23 - m03 * m22;
  const double c0 = m02 * m13 - m03 * m12;
  // adjugate entries (standard 4x4 inverse numerators, symmetric input)
  const double i00 = m11 * c5 - m12 * c4 + m13 * c3;
  const double i11 = m00 * c5 - m02 * c2 + m03 * c1;
  const double i22 = m03 * s4 - m13 * s2 + m33 * s0;
  const double i33 = m02 * s3 - m12 * s1 + m22 * s0;
  const double d0 = fabs(i00), d1 = fabs(i11), d2 = fabs(i22), d3 = fabs(i33);
  int j = 0;
  double best = d0;
  if (d1 > best) { best = d1; j = 1; }
  if (d2 > best) { best = d2; j = 2; }
  if (d3 > best) { best = d3; j = 3; }
  if (j == 0) {
    v[0] = i00;
    v[1] = -m01 * c5 + m12 * c2 - m13 * c1;
    v[2] = m01 * c4 - m11 * c2 + m13 * c0;
    v[3] = -m01 * c3 + m11 * c1 - m12 * c0;
  } else if (j == 1) {
    v[0] = -m01 * c5 + m02 * c4 - m03 * c3;
    v[1] = i11;
    v[2] = -m00 * c4 + m01 * c2 - m03 * c0;
    v[3] = m00 * c3 - m01 * c1 + m02 * c0;
  } else if (j == 2) {
    v[0] = m13 * s5 - m23 * s4 + m33 * s3;
    v[1] = -m03 * s5 + m23 * s2 - m33 * s1;
    v[2] = i22;
    v[3] = -m03 * s3 + m13 * s1 - m23 * s0;
  } else {
    v[0] = -m12 * s5 + m22 * s4 - m23 * s3;
    v[1] = m02 * s5 - m22 * s2 + m23 * s1;
    v[2] = -m02 * s4 + m12 * s2 - m23 * s0;
    v[3] = i33;
  }
  const double nrm = sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2] + v[3] * v[3]);
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  v[0] *= inv; v[1] *= inv; v[2] *= inv; v[3] *= inv;
  return best;
}

// geometry.py:149-152: largest-|component| positive, first index on ties.
__device__ __forceinline__ void sign_fix4(double v[4]) {
  int i = 0;
  double b = fabs(v[0]);
  if (fabs(v[1]) > b) { b = fabs(v[1]); i = 1; }
  if (fabs(v[2]) > b) { b = fabs(v[2]); i = 2; }
  if (fabs(v[3]) > b) { b = fabs(v[3]); i = 3; }
  const double pick = i == 0 ? v[0] : i == 1 ? v[1] : i == 2 ? v[2] : v[3];
  if (pick < 0.0) { v[0] = -v[0]; v[1] = -v[1]; v[2] = -v[2]; v[3] = -v[3]; }
}

// geometry.py:156-164
__device__ __forceinline__ void quat_to_rot(const double q[4], double r[9]) {
  const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
  r[0] = q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3;
  r[1] = 2.0 * (q1 * q2 - q0 * q3);
  r[2] = 2.0 * (q1 * q3 + q0 * q2);
  r[3] = 2.0 * (q1 * q2 + q0 * q3);
  r[4] = q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3;
  r[5] = 2.0 * (q2 * q3 - q0 * q1);
  r[6] = 2.0 * (q1 * q3 - q0 * q2);
  r[7] = 2.0 * (q2 * q3 + q0 * q1);
  r[8] = q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3;
}

// geometry.py:167-177: J[c][b*3+g] = dR_{bg}/dq_c
__device__ __forceinline__ void rot_quat_jacobian(const double q[4], double J[4][9]) {
  const double q0 = 2.0 * q[0], q1 = 2.0 * q[1], q2 = 2.0 * q[2], q3 = 2.0 * q[3];
  J[0][0] = q0;  J[0][1] = -q3; J[0][2] = q2;  J[0][3] = q3;  J[0][4] = q0;  J[0][5] = -q1; J[0][6] = -q2; J[0][7] = q1;  J[0][8] = q0;
  J[1][0] = q1;  J[1][1] = q2;  J[1][2] = q3;  J[1][3] = q2;  J[1][4] = -q1; J[1][5] = -q0; J[1][6] = q3;  J[1][7] = q0;  J[1][8] = -q1;
  J[2][0] = -q2; J[2][1] = q1;  J[2][2] = q0;  J[2][3] = q1;  J[2][4] = q2;  J[2][5] = q3;  J[2][6] = -q0; J[2][7] = q3;  J[2][8] = -q2;
  J[3][0] = -q3; J[3][1] = -q0; J[3][2] = q1;  J[3][3] = q0;  J[3][4] = -q3; J[3][5] = q2;  J[3][6] = q1;  J[3][7] = q2;  J[3][8] = q3;
}

// Fast per-pair fit: lambda_max by Newton, eigenvector by adjugate.
// Returns MSD (= eigvals[0] of K).  If quat != nullptr the sign-normalised
// quaternion is written; returns via *ill the conditioning flag (caller
// falls back to Jacobi when set).
__device__ __forceinline__ double fit_fast(const double* S, double gx, double ga, double* quat,
                                           bool* ill) {
  const Sym4 n = horn(S);
  const double lam = newton_lmax(n, 0.5 * (gx + ga));
  const double msd = gx + ga - 2.0 * lam;
  if (quat) {
    const double best = adj_eigvec(n, lam, quat);
    const double scale = fmax(fabs(lam), 1e-300);
    *ill = !(best > 1e-8 * scale * scale * scale) || !isfinite(best);
    sign_fix4(quat);
  } else {
    *ill = false;
  }
  return msd;
}

// ---------------------------------------------------------------------------
// Cyclic Jacobi (geometry.py:106-153) on a 4x4 symmetric matrix, fully
// unrolled.  On return w[] holds ascending eigenvalues and V[r][c] the
// sign-normalised eigenvector columns.  Returns false if not converged.
// ---------------------------------------------------------------------------
template <int P, int Q>
__device__ __forceinline__ void jacobi_rotate(double (&a)[4][4], double (&v)[4][4]) {
  const double apq = a[P][Q];
  if (apq == 0.0) return;
  const double theta = (a[Q][Q] - a[P][P]) / (2.0 * apq);
  const double t = copysign(1.0, theta) / (fabs(theta) + hypot(theta, 1.0));
  const double c = 1.0 / sqrt(t * t + 1.0);
  const double s = t * c;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double ap = a[r][P], aq = a[r][Q];
    a[r][P] = c * ap - s * aq;
    a[r][Q] = s * ap + c * aq;
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double ap = a[P][r], aq = a[Q][r];
    a[P][r] = c * ap - s * aq;
    a[Q][r] = s * ap + c * aq;
  }
  a[P][Q] = 0.0;
  a[Q][P] = 0.0;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const double vp = v[r][P], vq = v[r][Q];
    v[r][P] = c * vp - s * vq;
    v[r][Q] = s * vp + c * vq;
  }
}

__device__ __forceinline__ bool jacobi4(double (&a)[4][4], double w[4], double (&V)[4][4]) {
  double v[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) v[i][j] = (i == j) ? 1.0 : 0.0;
  double fro = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) fro += a[i][j] * a[i][j];
  const double tol = fmax(1e-14, 4e-16 * sqrt(fro));
  bool converged = false;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i != j) off += a[i][j] * a[i][j];
    if (sqrt(off) < tol) { converged = true; break; }
    jacobi_rotate<0, 1>(a, v);
    jacobi_rotate<0, 2>(a, v);
    jacobi_rotate<0, 3>(a, v);
    jacobi_rotate<1, 2>(a, v);
    jacobi_rotate<1, 3>(a, v);
    jacobi_rotate<2, 3>(a, v);
  }
  // stable ascending order of the diagonal
  const double d[4] = {a[0][0], a[1][1], a[2][2], a[3][3]};
  int rank[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) r += (d[j] < d[i]) || (d[j] == d[i] && j < i);
    rank[i] = r;
  }
#pragma unroll
  for (int o = 0; o < 4; ++o) {
    double wo = 0.0, c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (rank[i] == o) { wo = d[i]; c0 = v[0][i]; c1 = v[1][i]; c2 = v[2][i]; c3 = v[3][i]; }
    }
    double col[4] = {c0, c1, c2, c3};
    sign_fix4(col);
    w[o] = wo;
    V[0][o] = col[0]; V[1][o] = col[1]; V[2][o] = col[2]; V[3][o] = col[3];
  }
  return converged;
}

// K = (gx + ga) I - 2 N(S) as a dense 4x4
__device__ __forceinline__ void kearsley_from_S(const double* S, double gx, double ga, double (&k)[4][4]) {
  const Sym4 n = horn(S);
  const double g = gx + ga;
  k[0][0] = g - 2.0 * n.a00; k[0][1] = -2.0 * n.a01; k[0][2] = -2.0 * n.a02; k[0][3] = -2.0 * n.a03;
  k[1][1] = g - 2.0 * n.a11; k[1][2] = -2.0 * n.a12; k[1][3] = -2.0 * n.a13;
  k[2][2] = g - 2.0 * n.a22; k[2][3] = -2.0 * n.a23;
  k[3][3] = g - 2.0 * n.a33;
  k[1][0] = k[0][1]; k[2][0] = k[0][2]; k[3][0] = k[0][3];
  k[2][1] = k[1][2]; k[3][1] = k[1][3]; k[3][2] = k[2][3];
}

// v^T (dK/dx_{k,alpha}) q0 for all alpha, closed form of
// geometry.py:199-224 contracted with two quaternions (verified against
// the einsum in tests/test_kernels_math.py):
//   2 w [ v0 q0 m - (v0 u + q0 vv) x y - vv (y.u) - u (y.vv) + p (vv.u) ]
// with m = x - y, p = x + y, u = q0[1:], vv = v[1:], y the reference.
__device__ __forceinline__ void dk_contract(const double v[4], const double q[4], double w,
                                            const double x[3], const double y[3], double out[3]) {
  const double v0 = v[0], q0 = q[0];
  const double u0 = q[1], u1 = q[2], u2 = q[3];
  const double t0 = v[1], t1 = v[2], t2 = v[3];
  const double c0 = v0 * u0 + q0 * t0, c1 = v0 * u1 + q0 * t1, c2 = v0 * u2 + q0 * t2;
  // (c x y)
  const double cx0 = c1 * y[2] - c2 * y[1];
  const double cx1 = c2 * y[0] - c0 * y[2];
  const double cx2 = c0 * y[1] - c1 * y[0];
  const double yu = y[0] * u0 + y[1] * u1 + y[2] * u2;
  const double yt = y[0] * t0 + y[1] * t1 + y[2] * t2;
  const double tu = t0 * u0 + t1 * u1 + t2 * u2;
  const double vq = v0 * q0;
  const double w2 = 2.0 * w;
  out[0] = w2 * (vq * (x[0] - y[0]) - cx0 - t0 * yu - u0 * yt + (x[0] + y[0]) * tu);
  out[1] = w2 * (vq * (x[1] - y[1]) - cx1 - t1 * yu - u1 * yt + (x[1] + y[1]) * tu);
  out[2] = w2 * (vq * (x[2] - y[2]) - cx2 - t2 * yu - u2 * yt + (x[2] + y[2]) * tu);
}

// ----------------------------------------------------------- reductions
template <int NT>
__device__ __forceinline__ double block_sum(double v, double* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double r = 0.0;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) r += scratch[i];
  return r;
}

template <int NT>
__device__ __forceinline__ double block_min(double v, double* scratch) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  double r = scratch[0];
#pragma unroll
  for (int i = 1; i < NT / 32; ++i) r = fmin(r, scratch[i]);
  return r;
}

// power-of-two scale of an int8-digit row with max |v| = mx (refine_i8.cu / grad_i8.cu):
// 2^e with mx 2^(7 - e) <= 127, so every value's 31-bit integer rint(v 2^(31 - e)) has
// balanced base-256 digits with |d0| <= 127
__device__ __forceinline__ int mc_digit_exp(double mx) {
  if (!(mx > 0.0) || !isfinite(mx)) return 0;
  int e;
  frexp(mx, &e);  // mx < 2^e
  if (ldexp(mx, 7 - e) > 127.0) ++e;
  return e;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace mc
