// Shared epilogue of the tensor-core MSD-estimate kernels (tf32_gemm.cu,
// tf32_gemm_2sm.cu): one thread owns one frame row and finishes 8 landmark
// pairs from their fp32 covariances S (9 TMEM columns each): Horn's N(S),
// its characteristic quartic, and lambda_max by fp64 Newton with the 8
// chains interleaved (newton_lmax_batch) -> D = Gx + Ga - 2 lambda_max.
#pragma once
#include "mc_math.cuh"

namespace mc {

// lambda_max(N(S)) = max over rotations <R, S> = s1 + s2 + sign(det S) s3
// (Kabsch, s_i the singular values of S).  fp32 closed form: the eigenvalues
// of S^T S by the trigonometric solution of its characteristic cubic.  Used
// only as the Newton start, so fp32 accuracy (and the fast intrinsics) do.
__device__ __forceinline__ float lmax_kabsch_f32(const float (&S)[9]) {
  // M = S^T S (symmetric 3x3)
  float m[3][3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = i; j < 3; ++j) m[i][j] = S[i] * S[j] + S[3 + i] * S[3 + j] + S[6 + i] * S[6 + j];
  const float tr = (m[0][0] + m[1][1] + m[2][2]) * (1.0f / 3.0f);
  const float k00 = m[0][0] - tr, k11 = m[1][1] - tr, k22 = m[2][2] - tr;
  const float k01 = m[0][1], k02 = m[0][2], k12 = m[1][2];
  const float p2 = (k00 * k00 + k11 * k11 + k22 * k22 + 2.0f * (k01 * k01 + k02 * k02 + k12 * k12)) * (1.0f / 6.0f);
  const float detk = k00 * (k11 * k22 - k12 * k12) - k01 * (k01 * k22 - k12 * k02) + k02 * (k01 * k12 - k11 * k02);
  float e1 = tr, e2 = tr, e3 = tr;
  if (p2 > 0.0f) {
    const float pr = sqrtf(p2);
    const float r = fminf(1.0f, fmaxf(-1.0f, 0.5f * detk / (p2 * pr)));
    const float phi = acosf(r) * (1.0f / 3.0f);
    e1 = tr + 2.0f * pr * __cosf(phi);
    e3 = tr + 2.0f * pr * __cosf(phi + 2.0943951f);
    e2 = 3.0f * tr - e1 - e3;
  }
  const float dets = S[0] * (S[4] * S[8] - S[5] * S[7]) - S[1] * (S[3] * S[8] - S[5] * S[6]) +
                     S[2] * (S[3] * S[7] - S[4] * S[6]);
  const float s1 = sqrtf(fmaxf(e1, 0.0f)), s2 = sqrtf(fmaxf(e2, 0.0f)), s3 = sqrtf(fmaxf(e3, 0.0f));
  return s1 + s2 + (dets < 0.0f ? -s3 : s3);
}

// Eigenvector of the fp32 Horn matrix (entries n[10]: a00 a01 a02 a03 a11 a12
// a13 a22 a23 a33) for eigenvalue lam: the adjugate column of (N - lam I)
// with the largest |diagonal| cofactor (one inverse-iteration step), unnormalised.
__device__ __forceinline__ void adj_eigvec_f32(const float (&n)[10], float lam, float (&v)[4]) {
  const float m00 = n[0] - lam, m01 = n[1], m02 = n[2], m03 = n[3];
  const float m11 = n[4] - lam, m12 = n[5], m13 = n[6];
  const float m22 = n[7] - lam, m23 = n[8], m33 = n[9] - lam;
  const float s0 = m00 * m11 - m01 * m01, s1 = m00 * m12 - m01 * m02, s2 = m00 * m13 - m01 * m03;
  const float s3 = m01 * m12 - m11 * m02, s4 = m01 * m13 - m11 * m03, s5 = m02 * m13 - m12 * m03;
  const float c5 = m22 * m33 - m23 * m23, c4 = m12 * m33 - m13 * m23, c3 = m12 * m23 - m13 * m22;
  const float c2 = m02 * m33 - m03 * m23, c1 = m02 * m23 - m03 * m22, c0 = m02 * m13 - m03 * m12;
  const float i00 = m11 * c5 - m12 * c4 + m13 * c3;
  const float i11 = m00 * c5 - m02 * c2 + m03 * c1;
  const float i22 = m03 * s4 - m13 * s2 + m33 * s0;
  const float i33 = m02 * s3 - m12 * s1 + m22 * s0;
  const float d0 = fabsf(i00), d1 = fabsf(i11), d2 = fabsf(i22), d3 = fabsf(i33);
  const float b01 = fmaxf(d0, d1), b23 = fmaxf(d2, d3);
  if (b01 >= b23) {
    if (d0 >= d1) {
      v[0] = i00; v[1] = -m01 * c5 + m12 * c2 - m13 * c1;
      v[2] = m01 * c4 - m11 * c2 + m13 * c0; v[3] = -m01 * c3 + m11 * c1 - m12 * c0;
    } else {
      v[0] = -m01 * c5 + m02 * c4 - m03 * c3; v[1] = i11;
      v[2] = -m00 * c4 + m01 * c2 - m03 * c0; v[3] = m00 * c3 - m01 * c1 + m02 * c0;
    }
  } else {
    if (d2 >= d3) {
      v[0] = m13 * s5 - m23 * s4 + m33 * s3; v[1] = -m03 * s5 + m23 * s2 - m33 * s1;
      v[2] = i22; v[3] = -m03 * s3 + m13 * s1 - m23 * s0;
    } else {
      v[0] = -m12 * s5 + m22 * s4 - m23 * s3; v[1] = m02 * s5 - m22 * s2 + m23 * s1;
      v[2] = -m02 * s4 + m12 * s2 - m23 * s0; v[3] = i33;
    }
  }
}

// v[e][i]: S entry e (= b*3 + g) of pair i; pairs l0 + i >= L are padding.
// sc_f * sc_l[l] rescales the F16 operand format (sc_l == nullptr: TF32, unscaled).
//
// lambda_max = max over unit q of q^T N q / q^T q.  The quaternion is found in
// fp32 (Kabsch closed-form value, then the adjugate eigenvector of the fp32
// N); lambda_max is then the fp64 Rayleigh quotient of that q with N formed
// from S in fp64.  The quotient is stationary at the eigenvector, so an fp32
// eigenvector error e costs only ~gap * e^2 (worst case ~1e-7 |N|, below the
// fp32 tensor-core accumulation error of S itself), and it never exceeds
// lambda_max: D is never underestimated by the solve.  ~50 fp64 operations
// per pair instead of a characteristic polynomial and Newton iterations.
__device__ __forceinline__ void msd8_estimate(const float (&v)[9][8], double gx, const double* __restrict__ ga,
                                              double sc_f, const double* __restrict__ sc_l, int l0, int L,
                                              float (&out)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int l = l0 + i;
    const bool ok = l < L;
    const double sc = sc_l ? sc_f * (ok ? sc_l[l] : 1.0) : 1.0;
    const float scf = (float)sc;
    float sf[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) sf[e] = v[e][i] * scf;
    const float nf[10] = {sf[0] + sf[4] + sf[8],  sf[7] - sf[5],  sf[2] - sf[6],  sf[3] - sf[1],
                          sf[0] - sf[4] - sf[8],  sf[1] + sf[3],  sf[2] + sf[6],  -sf[0] + sf[4] - sf[8],
                          sf[5] + sf[7],          -sf[0] - sf[4] + sf[8]};
    float qf[4];
#ifdef MC_DIAG_EPI_KABSCH_ONLY
    // diagnostic build only: the fp32 Kabsch value as the estimate (timing)
    { out[i] = ok ? (float)(gx + ga[l] - 2.0 * (double)lmax_kabsch_f32(sf)) : 0.0f; continue; }
#endif
#ifdef MC_DIAG_EPI_NONE
    { out[i] = ok ? (float)(gx + ga[l] - 2.0 * (double)(nf[0] + nf[4])) : 0.0f; continue; }
#endif
    adj_eigvec_f32(nf, lmax_kabsch_f32(sf), qf);
    // fp64 Rayleigh quotient with N(S) in fp64
    double S[9];
#pragma unroll
    for (int e = 0; e < 9; ++e) S[e] = (double)v[e][i] * sc;
    const Sym4 n = horn(S);
    const double q0 = qf[0], q1 = qf[1], q2 = qf[2], q3 = qf[3];
    const double qq = q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3;
    const double qnq = n.a00 * q0 * q0 + n.a11 * q1 * q1 + n.a22 * q2 * q2 + n.a33 * q3 * q3 +
                       2.0 * (q0 * (n.a01 * q1 + n.a02 * q2 + n.a03 * q3) + q1 * (n.a12 * q2 + n.a13 * q3) +
                              q2 * n.a23 * q3);
    double lam = 0.0;
    if (qq > 0.0) {
      double r;
      asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(qq));
      r = fma(r, fma(-qq, r, 1.0), r);
      r = fma(r, fma(-qq, r, 1.0), r);
      lam = qnq * r;
    }
    out[i] = ok ? (float)(gx + ga[l] - 2.0 * lam) : 0.0f;
  }
}

}  // namespace mc
