// K1s + K2/K3 — fp32-coordinate path (configs 2/3/4).
//
// K1s  center_split_kernel: centre each structure in fp64 (geometry.py:67-76),
//      optionally fold the displacement weights w_j into the operand, and
//      split every centred coordinate v into two TF32 values hi + lo
//      (hi = rna_tf32(v), lo = rna_tf32(v - hi)), written plane-major
//      [3][B][kpad] fp32 so each plane of a structure tile is one TMA box.
//
// K2   msd_tf32_kernel: the all-pairs 3x3 covariance
//        S[t,l][b][g] = sum_j x_{t,j,b} (w_j a_{l,j,g})
//      as a dense contraction on the 5th-gen tensor cores with the 3xTF32
//      scheme (hi*hi + hi*lo + lo*hi, fp32 accumulation in TMEM), and
// K3   fused into its epilogue: Horn's lambda_max by fp64 Newton and the MSD
//      estimate D = Gx + Ga - 2 lambda_max (mc_math.cuh), written as fp32.
//
// Tile: 128 frames (TMEM lanes) x 48 landmarks.  For every frame plane b a
// separate accumulator D_b[128 x 144] holds columns (g, l) = g*48 + l, so
// the 9 entries S[b][g] of a pair live in the SAME TMEM lane and one
// epilogue thread owns whole pairs (no cross-lane shuffles, no padding of
// the 3-row structure to 4).  Per 8-atom k-step: 3 planes x 3 split terms
// = 9 tcgen05.mma (M=128, N=144, K=8, kind::tf32), A = frame plane tile,
// B = the 3 landmark planes stacked (144 rows).  Operands stream through a
// 3-stage TMA (SWIZZLE_64B, 16 atoms per stage) -> smem -> UMMA pipeline.
// Warp roles (256 threads, persistent over tiles, landmark tiles fastest so
// the landmark operand stays L2-resident while a frame tile is in use):
//   warp 0: TMA producer   warp 1: MMA issuer (one elected lane)
//   warp 2: TMEM allocator warps 4-7: epilogue (TMEM lane quarter = warp%4)
#include <algorithm>
#include <cstdlib>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "mc_math.cuh"
#include "tc_epilogue.cuh"

namespace mc {

// ------------------------------------------------------------------ K1s
__device__ __forceinline__ float tf32_rna(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return __uint_as_float(r);
}

// Operand formats.  TF32: hi/lo fp32 words holding TF32 values, unscaled.
// F16: hi/lo IEEE halves of the structure's values times a power of two 2^e
// chosen so every |value| < 2^14 (no overflow, no subnormal loss that
// matters); hi + lo carries the same 22 significant bits as the TF32 pair,
// the fp32 accumulation is identical, and the MMA (kind::f16, K = 16) moves
// twice the atoms per byte and per tensor-core cycle.  scale_inv[b] = 2^-e
// undoes the scaling exactly in the epilogue.
struct OpTF32 {
  using E = float;
  static constexpr bool kInterleave = false;
  static __device__ __forceinline__ double value(E h) { return (double)h; }
  static __device__ __forceinline__ void split(double v, E& h, E& l) {
    h = tf32_rna((float)v);
    l = tf32_rna((float)(v - (double)h));
  }
};
struct OpF16 {
  using E = __half;
  static __device__ __forceinline__ double value(E h) { return (double)__half2float(h); }
  // rows of 2 kpad halves: per 32-atom block [hi x32 | lo x32] = one 128 B
  // line, so one SWIZZLE_128B TMA box row carries both parts of a k-block.
  // One-term mode (lo == nullptr on entry, see below): rows of kpad hi halves.
  static constexpr bool kInterleave = true;
  static __device__ __forceinline__ void split(double v, E& h, E& l) {
    h = __double2half(v);
    l = __double2half(v - (double)__half2float(h));
  }
};

template <typename T, typename OP, int NT>
__global__ void __launch_bounds__(NT)
center_split_kernel(const T* __restrict__ coords, int64_t B, int n, int kpad, const double* __restrict__ w_align,
                    const double* __restrict__ w_disp, int weighted, typename OP::E* __restrict__ hi,
                    typename OP::E* __restrict__ lo, double* __restrict__ scale_inv, double* __restrict__ centroid,
                    double* __restrict__ gnorm, double* __restrict__ wbar, double* __restrict__ mom,
                    uint8_t* __restrict__ flags, int one_term = 0, double* __restrict__ opnorm = nullptr,
                    double* __restrict__ rnorm = nullptr) {
  __shared__ double scratch[NT / 32];
  const int64_t b = blockIdx.x;
  const T* x = coords + b * (int64_t)n * 3;
  double c0 = 0.0, c1 = 0.0, c2 = 0.0, xmax = 0.0, wmax = 0.0;
  bool finite = true;
  for (int j = threadIdx.x; j < n; j += NT) {
    const double wa = w_align[j];
    const double x0 = (double)x[3 * j], x1 = (double)x[3 * j + 1], x2 = (double)x[3 * j + 2];
    finite = finite && isfinite(x0) && isfinite(x1) && isfinite(x2);
    c0 += wa * x0; c1 += wa * x1; c2 += wa * x2;
    if (scale_inv) {
      xmax = fmax(xmax, fmax(fabs(x0), fmax(fabs(x1), fabs(x2))));
      if (weighted) wmax = fmax(wmax, fabs(w_disp[j]));
    }
  }
  c0 = block_sum<NT>(c0, scratch);
  c1 = block_sum<NT>(c1, scratch);
  c2 = block_sum<NT>(c2, scratch);
  const int nonfinite = __syncthreads_or(!finite);
  // power-of-two operand scale from a bound on |value| (F16 only)
  double scale = 1.0;
  if (scale_inv) {
    double bound = -block_min<NT>(-xmax, scratch);
    if (weighted) bound *= -block_min<NT>(-wmax, scratch);
    // |x_j - c| <= 2 max|x| (c is a convex combination of the x_j)
    bound *= 2.0;
    int e = 0;
    if (bound > 0.0 && isfinite(bound)) {
      frexp(bound, &e);  // bound < 2^e
      e = 14 - e;
    }
    e = max(-1000, min(1000, e));
    scale = ldexp(1.0, e);
    if (threadIdx.x == 0) scale_inv[b] = ldexp(1.0, -e);
  }
  double g = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0, m00 = 0, m01 = 0, m02 = 0, m11 = 0, m12 = 0, m22 = 0, on2 = 0.0;
  double rn2 = 0.0;  // one-term: squared 2-norm of the operand's rounding residual
  const int64_t plane = B * (int64_t)kpad;
  for (int j = threadIdx.x; j < kpad; j += NT) {
    double v[3] = {0.0, 0.0, 0.0};
    double w = 0.0;
    if (j < n) {
      w = w_disp[j];
      v[0] = (double)x[3 * j] - c0;
      v[1] = (double)x[3 * j + 1] - c1;
      v[2] = (double)x[3 * j + 2] - c2;
    }
    const double wx0 = w * v[0], wx1 = w * v[1], wx2 = w * v[2];
    g += wx0 * v[0] + wx1 * v[1] + wx2 * v[2];
    b0 += wx0; b1 += wx1; b2 += wx2;
    m00 += wx0 * v[0]; m01 += wx0 * v[1]; m02 += wx0 * v[2];
    m11 += wx1 * v[1]; m12 += wx1 * v[2]; m22 += wx2 * v[2];
#pragma unroll
    for (int p = 0; p < 3; ++p) {
      const double uv = weighted ? w * v[p] : v[p];
      on2 += uv * uv;
      const double val = uv * scale;
      typename OP::E h, l;
      OP::split(val, h, l);
      if (OP::kInterleave && one_term) {
        hi[p * plane + b * kpad + j] = h;
        const double rd = OP::value(h) / scale - uv;
        rn2 += rd * rd;
      } else if (OP::kInterleave) {
        const int64_t o = 2 * (p * plane + b * kpad) + (j >> 5) * 64 + (j & 31);
        hi[o] = h;
        hi[o + 32] = l;
      } else {
        hi[p * plane + b * kpad + j] = h;
        lo[p * plane + b * kpad + j] = l;
      }
    }
  }
  g = block_sum<NT>(g, scratch);
  if (opnorm) on2 = block_sum<NT>(on2, scratch);
  if (rnorm) rn2 = block_sum<NT>(rn2, scratch);
  if (wbar) { b0 = block_sum<NT>(b0, scratch); b1 = block_sum<NT>(b1, scratch); b2 = block_sum<NT>(b2, scratch); }
  if (mom) {
    m00 = block_sum<NT>(m00, scratch); m01 = block_sum<NT>(m01, scratch); m02 = block_sum<NT>(m02, scratch);
    m11 = block_sum<NT>(m11, scratch); m12 = block_sum<NT>(m12, scratch); m22 = block_sum<NT>(m22, scratch);
  }
  if (threadIdx.x == 0) {
    if (centroid) { centroid[3 * b] = c0; centroid[3 * b + 1] = c1; centroid[3 * b + 2] = c2; }
    gnorm[b] = g;
    if (wbar) { wbar[3 * b] = b0; wbar[3 * b + 1] = b1; wbar[3 * b + 2] = b2; }
    if (mom) {
      mom[6 * b] = m00; mom[6 * b + 1] = m01; mom[6 * b + 2] = m02;
      mom[6 * b + 3] = m11; mom[6 * b + 4] = m12; mom[6 * b + 5] = m22;
    }
    if (flags) flags[b] = nonfinite ? kFlagNonFinite : 0;
    if (opnorm) opnorm[b] = sqrt(on2);
    if (rnorm) rnorm[b] = sqrt(rn2);
  }
}

// Fast K1s for the one-term F16 frame operand (fp32 input, unweighted operand,
// N % 4 == 0): 4-atom groups move as float4 triples (the second pass re-reads the
// structure from L2), the scaled halves go out as 8-byte rows of 4 atoms per
// axis, and the sums of each pass are reduced in one shared-memory round.  Same
// centroid / G / wbar / opnorm as center_split_kernel<float, OpF16> (fp64 centring);
// the halves are rn16(fl32(v) 2^e) and rnorm a rigorous upper bound of the exact
// residual norm (see below).

template <int NT, int K>
__device__ __forceinline__ void block_sum_n(double (&v)[K], double* scratch) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < K; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], o);
  __syncthreads();
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < K; ++k) scratch[k * (NT / 32) + warp] = v[k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double r = 0.0;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) r += scratch[k * (NT / 32) + i];
    v[k] = r;
  }
}

template <int CSF_NT>
__global__ void __launch_bounds__(CSF_NT, 1024 / CSF_NT)
center_split_f16x1_kernel(const float* __restrict__ coords, int64_t B, int n, int kpad,
                          const double* __restrict__ w_align, const double* __restrict__ w_disp,
                          __half* __restrict__ hi, double* __restrict__ scale_inv, double* __restrict__ centroid,
                          double* __restrict__ gnorm, double* __restrict__ wbar, uint8_t* __restrict__ flags,
                          double* __restrict__ opnorm, double* __restrict__ rnorm) {
  __shared__ double scratch[6 * (CSF_NT / 32)];
  const int64_t b = blockIdx.x;
  const float4* x4 = reinterpret_cast<const float4*>(coords + b * (int64_t)n * 3);
  const int G = n / 4;
  double c[3] = {0.0, 0.0, 0.0};
  float xmax = 0.0f;
  bool finite = true;
#pragma unroll 2
  for (int gi = threadIdx.x; gi < G; gi += CSF_NT) {
    const float4 q0 = x4[3 * gi], q1 = x4[3 * gi + 1], q2 = x4[3 * gi + 2];
    const float f[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const double wa = w_align[4 * gi + a];
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const float x = f[3 * a + p];
        finite = finite && isfinite(x);
        xmax = fmaxf(xmax, fabsf(x));
        c[p] = fma(wa, (double)x, c[p]);
      }
    }
  }
  const double xm = -block_min<CSF_NT>(-(double)xmax, scratch);
  block_sum_n<CSF_NT, 3>(c, scratch);
  const int nonfinite = __syncthreads_or(!finite);
  const double bound = 2.0 * xm;  // |x_j - c| <= 2 max|x|
  int e = 0;
  if (bound > 0.0 && isfinite(bound)) {
    frexp(bound, &e);
    e = 14 - e;
  }
  e = max(-1000, min(1000, e));
  // fp32 scaling and residuals (exact while 2^e and 2^-e are normal floats): the
  // rounding residual of each half is measured against vf = fl32(v), exactly (Sterbenz:
  // h 2^-e and vf are within a factor 2), and rnorm is returned as the rigorous upper
  // bound ||h 2^-e - vf|| (1 + 1e-5) + 2^-24 ||v|| of ||h 2^-e - v|| -- half the fp64
  // work per coordinate of the exact residual (the kernel is issue-bound, not HBM-bound)
  const bool f32s = e >= -126 && e <= 126;
  const float scf = f32s ? ldexpf(1.0f, e) : 0.0f, sif = f32s ? ldexpf(1.0f, -e) : 0.0f;
  const double scale = ldexp(1.0, e);
  const int64_t plane = B * (int64_t)kpad;
  __half* h0 = hi + b * kpad;
  double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // g, wbar (3), |operand|^2, |rounding residual|^2
  const double sinv = ldexp(1.0, -e);
#pragma unroll 2
  for (int gi = threadIdx.x; gi < kpad / 4; gi += CSF_NT) {
    uint2 o[3] = {make_uint2(0u, 0u), make_uint2(0u, 0u), make_uint2(0u, 0u)};
    if (gi < G) {
      const float4 q0 = x4[3 * gi], q1 = x4[3 * gi + 1], q2 = x4[3 * gi + 2];
      const float f[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
      __half h[3][4];
      float r2 = 0.0f;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const double wd = w_disp[4 * gi + a];
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          const double v = (double)f[3 * a + p] - c[p];
          const double tv = wd * v;
          acc[0] = fma(tv, v, acc[0]);
          acc[1 + p] += tv;
          acc[4] = fma(v, v, acc[4]);
          if (f32s) {
            const float vf = (float)v;
            h[p][a] = __float2half_rn(vf * scf);
            const float r = fmaf(__half2float(h[p][a]), sif, -vf);
            r2 = fmaf(r, r, r2);
          } else {
            h[p][a] = __double2half(v * scale);
            const double rd = (double)__half2float(h[p][a]) * sinv - v;
            acc[5] = fma(rd, rd, acc[5]);
          }
        }
      }
      acc[5] += (double)r2;
#pragma unroll
      for (int p = 0; p < 3; ++p) o[p] = *reinterpret_cast<const uint2*>(h[p]);
    }
#pragma unroll
    for (int p = 0; p < 3; ++p) *reinterpret_cast<uint2*>(h0 + p * plane + 4 * gi) = o[p];
  }
  block_sum_n<CSF_NT, 6>(acc, scratch);
  if (threadIdx.x == 0) {
    if (centroid) { centroid[3 * b] = c[0]; centroid[3 * b + 1] = c[1]; centroid[3 * b + 2] = c[2]; }
    gnorm[b] = acc[0];
    if (wbar) { wbar[3 * b] = acc[1]; wbar[3 * b + 1] = acc[2]; wbar[3 * b + 2] = acc[3]; }
    if (flags) flags[b] = nonfinite ? kFlagNonFinite : 0;
    const double on = sqrt(acc[4]);
    if (opnorm) opnorm[b] = on;
    // ||h 2^-e - v|| <= ||h 2^-e - vf|| + ||vf - v||, |vf - v| <= 2^-24 |v|; 1e-5 covers the
    // fp32 accumulation of the <= 12 (kpad / 4 / CSF_NT + 1) squares per thread
    if (rnorm) rnorm[b] = f32s ? sqrt(acc[5]) * (1.0 + 1e-5) + ldexp(on, -24) : sqrt(acc[5]);
    scale_inv[b] = sinv;
  }
}

// K1s for uniform weights (w = w' = wuni on the n atoms; the configs' case): every
// per-structure sum comes out of the FIRST pass as moments shifted by the first atom p
// (U1 = sum (x - p), U2 = sum (x - p)^2 per axis, fp64; no cancellation: |c - p| is of
// the structure's size), so the second pass is pure fp32: vf = fl32(x - fl32(c)),
// h = rn16(vf 2^e) and the residual |h 2^-e - vf|^2.  Per coordinate 5 instructions in
// pass 1 (3 fp64) and 6 fp32 in pass 2, against ~20 with 5 fp64 in center_split_f16x1.
//   c = p + U1 / n,  sum |x - c|^2 = sum_b (U2_b - U1_b^2 / n),  G = wuni * that,
//   wbar = sum w (x - c) = 0,
//   rnorm: ||h 2^-e - v|| <= ||h 2^-e - vf|| (1 + 1e-5) + ||vf - v||, and per coordinate
//   |vf - v| <= 2^-24 |x - c32| + |c - c32| <= 2^-24 (|v| + 2 |c|), so
//   ||vf - v|| <= 2^-24 (1 + 2^-20) (||v|| + 2 sqrt(n) |c|_2).
template <int NT>
__global__ void __launch_bounds__(NT, 1024 / NT)
center_split_f16x1_uni_kernel(const float* __restrict__ coords, int64_t B, int n, int kpad, double wuni,
                              __half* __restrict__ hi, double* __restrict__ scale_inv, double* __restrict__ centroid,
                              double* __restrict__ gnorm, double* __restrict__ wbar, uint8_t* __restrict__ flags,
                              double* __restrict__ opnorm, double* __restrict__ rnorm, int* __restrict__ dexp) {
  __shared__ double scratch[6 * (NT / 32)];
  __shared__ float s_ext[6][NT / 32];
  const int64_t b = blockIdx.x;
  const float* xb = coords + b * (int64_t)n * 3;
  const float4* x4 = reinterpret_cast<const float4*>(xb);
  const int G = n / 4;
  const double p0 = (double)__ldg(xb), p1 = (double)__ldg(xb + 1), p2 = (double)__ldg(xb + 2);
  double u[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // U1 (3), U2 (3)
  // per-axis maximum and (negated) minimum of the raw coordinates: max|x - c| per axis
  // (the frame's int8 row-digit exponents) = max(xmax - c, c - xmin), no extra pass
  float ext[6] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll 2
  for (int gi = threadIdx.x; gi < G; gi += NT) {
    const float4 q0 = x4[3 * gi], q1 = x4[3 * gi + 1], q2 = x4[3 * gi + 2];
    const float f[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
#pragma unroll
    for (int a = 0; a < 4; ++a) {
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        const double y = (double)f[3 * a + p] - (p == 0 ? p0 : (p == 1 ? p1 : p2));
        u[p] += y;
        u[3 + p] = fma(y, y, u[3 + p]);
        ext[p] = fmaxf(ext[p], f[3 * a + p]);
        ext[3 + p] = fmaxf(ext[3 + p], -f[3 * a + p]);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 6; ++k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ext[k] = fmaxf(ext[k], __shfl_xor_sync(0xffffffffu, ext[k], o));
    if ((threadIdx.x & 31) == 0) s_ext[k][threadIdx.x >> 5] = ext[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    float m = s_ext[k][0];
#pragma unroll
    for (int i = 1; i < NT / 32; ++i) m = fmaxf(m, s_ext[k][i]);
    ext[k] = m;
  }
  const double xm = (double)fmaxf(fmaxf(fmaxf(ext[0], ext[3]), fmaxf(ext[1], ext[4])), fmaxf(ext[2], ext[5]));
  block_sum_n<NT, 6>(u, scratch);
  const double inv_n = 1.0 / (double)n;
  const double c[3] = {p0 + u[0] * inv_n, p1 + u[1] * inv_n, p2 + u[2] * inv_n};
  const double on2 = fmax(0.0, (u[3] - u[0] * u[0] * inv_n) + (u[4] - u[1] * u[1] * inv_n) +
                                   (u[5] - u[2] * u[2] * inv_n));
  const bool nonfinite = !isfinite(u[0] + u[1] + u[2] + u[3] + u[4] + u[5]) || !isfinite(xm);
  const double bound = 2.0 * xm;  // |x_j - c| <= 2 max|x|
  int e = 0;
  if (bound > 0.0 && isfinite(bound)) {
    frexp(bound, &e);
    e = 14 - e;
  }
  e = max(-1000, min(1000, e));
  const bool f32s = e >= -126 && e <= 126;
  const float scf = f32s ? ldexpf(1.0f, e) : 0.0f, sif = f32s ? ldexpf(1.0f, -e) : 0.0f;
  const double scale = ldexp(1.0, e), sinv = ldexp(1.0, -e);
  const float c32[3] = {(float)c[0], (float)c[1], (float)c[2]};
  const int64_t plane = B * (int64_t)kpad;
  __half* h0 = hi + b * kpad;
  double r2d = 0.0;
#pragma unroll 2
  for (int gi = threadIdx.x; gi < kpad / 4; gi += NT) {
    uint2 o[3] = {make_uint2(0u, 0u), make_uint2(0u, 0u), make_uint2(0u, 0u)};
    if (gi < G) {
      const float4 q0 = x4[3 * gi], q1 = x4[3 * gi + 1], q2 = x4[3 * gi + 2];
      const float f[12] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
      __half h[3][4];
      float r2 = 0.0f;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
#pragma unroll
        for (int p = 0; p < 3; ++p) {
          if (f32s) {
            const float vf = f[3 * a + p] - c32[p];
            h[p][a] = __float2half_rn(vf * scf);
            const float r = fmaf(__half2float(h[p][a]), sif, -vf);
            r2 = fmaf(r, r, r2);
          } else {  // extreme scales: fp64 (rare)
            const double v = (double)f[3 * a + p] - c[p];
            h[p][a] = __double2half(v * scale);
            const double rd = (double)__half2float(h[p][a]) * sinv - v;
            r2d = fma(rd, rd, r2d);
          }
        }
      }
      r2d += (double)r2;
#pragma unroll
      for (int p = 0; p < 3; ++p) o[p] = *reinterpret_cast<const uint2*>(h[p]);
    }
#pragma unroll
    for (int p = 0; p < 3; ++p) *reinterpret_cast<uint2*>(h0 + p * plane + 4 * gi) = o[p];
  }
  r2d = block_sum<NT>(r2d, scratch);
  if (threadIdx.x == 0) {
    if (centroid) { centroid[3 * b] = c[0]; centroid[3 * b + 1] = c[1]; centroid[3 * b + 2] = c[2]; }
    gnorm[b] = wuni * on2;
    if (wbar) { wbar[3 * b] = 0.0; wbar[3 * b + 1] = 0.0; wbar[3 * b + 2] = 0.0; }
    if (flags) flags[b] = nonfinite ? kFlagNonFinite : 0;
    const double on = sqrt(on2);
    if (opnorm) opnorm[b] = on;
    if (dexp)  // the exponents mc_row_digits would compute for this frame (unweighted rows)
#pragma unroll
      for (int p = 0; p < 3; ++p) dexp[3 * b + p] = mc_digit_exp(fmax((double)ext[p] - c[p], c[p] + (double)ext[3 + p]));
    const double cn = sqrt(c[0] * c[0] + c[1] * c[1] + c[2] * c[2]);
    if (rnorm)
      rnorm[b] = f32s ? sqrt(r2d) * (1.0 + 1e-5) + ldexp(1.0 + ldexp(1.0, -20), -24) * (on + 2.0 * sqrt((double)n) * cn)
                      : sqrt(r2d);
    scale_inv[b] = sinv;
  }
}

cudaError_t launch_center_split16_uniform(const float* coords, int64_t B, int n, int kpad, double wuni, void* hl,
                                          double* scale_inv, double* opnorm, double* rnorm, double* centroid,
                                          double* gnorm, double* wbar, uint8_t* flags, int* dexp,
                                          cudaStream_t stream) {
  if (B <= 0) return cudaSuccess;
  if (n % 4 || kpad % 4 || (reinterpret_cast<uintptr_t>(coords) & 15) || B > 0x7fffffffLL) return cudaErrorInvalidValue;
  center_split_f16x1_uni_kernel<256><<<(unsigned)B, 256, 0, stream>>>(coords, B, n, kpad, wuni, (__half*)hl, scale_inv,
                                                                      centroid, gnorm, wbar, flags, opnorm, rnorm,
                                                                      dexp);
  return cudaGetLastError();
}

cudaError_t launch_center_split(const void* coords, int dtype, int64_t B, int n, int kpad, const double* w_align,
                                const double* w_disp, int weighted, float* hi, float* lo, double* centroid,
                                double* gnorm, double* wbar, double* mom, uint8_t* flags, cudaStream_t stream) {
  if (B <= 0) return cudaSuccess;
  if (dtype == 0)
    center_split_kernel<float, OpTF32, 256><<<(unsigned)B, 256, 0, stream>>>(
        (const float*)coords, B, n, kpad, w_align, w_disp, weighted, hi, lo, nullptr, centroid, gnorm, wbar, mom, flags);
  else
    center_split_kernel<double, OpTF32, 256><<<(unsigned)B, 256, 0, stream>>>(
        (const double*)coords, B, n, kpad, w_align, w_disp, weighted, hi, lo, nullptr, centroid, gnorm, wbar, mom, flags);
  return cudaGetLastError();
}

cudaError_t launch_center_split16(const void* coords, int dtype, int64_t B, int n, int kpad, const double* w_align,
                                  const double* w_disp, int weighted, int terms, void* hl, double* scale_inv,
                                  double* opnorm, double* rnorm, double* centroid, double* gnorm, double* wbar,
                                  double* mom, uint8_t* flags, cudaStream_t stream) {
  if (B <= 0) return cudaSuccess;
  const int one = terms == 1 ? 1 : 0;
  if (dtype == 0 && one && !weighted && !mom && n % 4 == 0 && kpad % 4 == 0 &&
      (reinterpret_cast<uintptr_t>(coords) & 15) == 0 && B <= 0x7fffffffLL) {
    // 256 threads x 4 CTAs per SM: 1.25x the 512 x 2 rate (tools/_diag/k1_sweep.sh)
    static const int nt = getenv("MC_K1_NT") ? atoi(getenv("MC_K1_NT")) : 256;
    auto k = nt == 256 ? center_split_f16x1_kernel<256>
                       : (nt == 128 ? center_split_f16x1_kernel<128> : center_split_f16x1_kernel<512>);
    k<<<(unsigned)B, nt == 256 ? 256 : (nt == 128 ? 128 : 512), 0, stream>>>(
        (const float*)coords, B, n, kpad, w_align, w_disp, (__half*)hl, scale_inv, centroid, gnorm, wbar, flags,
        opnorm, rnorm);
    return cudaGetLastError();
  }
  if (dtype == 0)
    center_split_kernel<float, OpF16, 256><<<(unsigned)B, 256, 0, stream>>>(
        (const float*)coords, B, n, kpad, w_align, w_disp, weighted, (__half*)hl, nullptr, scale_inv, centroid,
        gnorm, wbar, mom, flags, one, opnorm, rnorm);
  else
    center_split_kernel<double, OpF16, 256><<<(unsigned)B, 256, 0, stream>>>(
        (const double*)coords, B, n, kpad, w_align, w_disp, weighted, (__half*)hl, nullptr, scale_inv, centroid,
        gnorm, wbar, mom, flags, one, opnorm, rnorm);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ K2/K3
namespace gemm {
constexpr int BM = 128;            // frames per tile (TMEM lanes)
#ifndef MC_TF32_BL
#define MC_TF32_BL 48
#endif
constexpr int BL = MC_TF32_BL;     // landmarks per tile
constexpr int BN = 3 * BL;         // 144 accumulator columns per frame plane
constexpr int ROWB = 64;           // bytes per operand row per stage (SWIZZLE_64B): 16 tf32 / 32 f16 atoms
#ifndef MC_STAGES
#define MC_STAGES 3
#endif
constexpr int STAGES = MC_STAGES;
constexpr int A_BYTES = BM * ROWB;          // 8 KB: one (plane, hi|lo) frame tile
constexpr int B_BYTES = BN * ROWB;          // 9 KB: hi or lo, 3 landmark planes stacked
constexpr int BP_BYTES = BL * ROWB;         // 3 KB: one landmark plane box
constexpr int STAGE_BYTES = 6 * A_BYTES + 2 * B_BYTES;  // 66 KB
// F16 (interleaved hi|lo rows, SWIZZLE_128B): per stage 32 atoms, 128 B rows
constexpr int A2_BYTES = BM * 128;          // 16 KB: one frame plane tile, hi and lo
constexpr int BP2_BYTES = BL * 128;         // 6 KB: one landmark plane box, hi and lo
static_assert(3 * A2_BYTES + 3 * BP2_BYTES == STAGE_BYTES, "both formats stage 66 KB");
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 512;
// warps 4.. are the epilogue: two per TMEM lane quarter, each finishing half
// of the 8-landmark column chunks, so the latency-bound fp64 Newton runs on
// two warps per SM sub-partition and the accumulator is released sooner
#ifndef MC_K2_EPI_WARPS
#define MC_K2_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = MC_K2_EPI_WARPS;  // 8 measured best (12: 128-register cap)
constexpr int NT = 32 * (4 + EPI_WARPS);
}  // namespace gemm

// per-operand-format constants: element size, atoms per stage, and the MMA
// instruction descriptor (D = F32 (bits 4-5 = 1), A = B = TF32 (2) or F16 (0),
// K-major, N >> 3, M >> 4); one MMA consumes 32 B of each row in both formats
template <bool F16>
struct Fmt {
  static constexpr int ESZ = F16 ? 2 : 4;
  static constexpr int KB = gemm::ROWB / ESZ;
  static constexpr uint32_t AB = F16 ? 0u : 2u;
  __host__ __device__ static constexpr uint32_t idesc(int n, int m) {
    return (1u << 4) | (AB << 7) | (AB << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
  }
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// SM100 UMMA shared-memory descriptor, K-major, SWIZZLE_64B (64 B rows,
// 8-row groups 512 B apart): start>>4 | LBO=1 | SBO=32 | version 1 | layout 4
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)((8 * gemm::ROWB) >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

// K-major SWIZZLE_128B (128 B rows, 8-row groups 1024 B apart), layout 2
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <bool F16>
__device__ __forceinline__ void umma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  constexpr uint32_t idesc = Fmt<F16>::idesc(gemm::BN, gemm::BM);
  if (F16)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

// Commit with the barrier's GENERIC address.  Measured (tools/mma_probe.cu):
// the .shared::cluster form (a cluster-window address) stalls the issuing
// thread for roughly the MMA pipeline depth on every commit (one commit per 18
// MMAs: 649 TF32 TF/s); the generic local-shared address does not (908 TF/s).
// one lane of the (converged) warp
__device__ __forceinline__ bool umma_elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.b32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(
                   reinterpret_cast<uint64_t>(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float v[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// Grouped tile order: GROUP_M frame tiles x all landmark tiles per group, frame
// tile fastest inside a group, so the ~148 concurrently running CTAs (which
// advance through K in near lockstep) cover ~4 frame tiles x ~37 landmark
// tiles and both operands are re-used out of L2 instead of streaming every
// landmark tile from HBM once per frame tile.
#ifndef MC_GROUP_M
#define MC_GROUP_M 4
#endif
__device__ __forceinline__ void tile_coords(int tile, int ntm, int ntl, int& tm, int& tl) {
  constexpr int GROUP_M = MC_GROUP_M;
  const int gsize = GROUP_M * ntl;
  const int g = tile / gsize;
  const int r = tile - g * gsize;
  const int gm = min(GROUP_M, ntm - g * GROUP_M);
  tl = r / gm;
  tm = g * GROUP_M + (r - tl * gm);
}


template <bool F16, bool ONE = false>
__global__ void __launch_bounds__(gemm::NT, 1)
msd_tf32_kernel(const __grid_constant__ CUtensorMap mfh, const __grid_constant__ CUtensorMap mfl,
                const __grid_constant__ CUtensorMap mlh, const __grid_constant__ CUtensorMap mll,
                const double* __restrict__ gx, const double* __restrict__ ga, const double* __restrict__ fsc,
                const double* __restrict__ lsc, int T, int L, int kpad, float* __restrict__ D, int64_t ldd,
                const int* __restrict__ tlist, const int* __restrict__ nlist) {
  using namespace gemm;
  constexpr int KB = Fmt<F16>::KB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ntm = (T + BM - 1) / BM, ntl = (L + BL - 1) / BL;
  // tile list (pruned / banded work, pairs (tm, tl)) or the full grouped raster
  const int ntiles = tlist ? *nlist : ntm * ntl;
  auto coords = [&](int tile, int& tm, int& tl) {
    if (tlist) { tm = tlist[2 * tile]; tl = tlist[2 * tile + 1]; } else { tile_coords(tile, ntm, ntl, tm, tl); }
  };
  // ONE (one-term F16 screen): 64 hi atoms per 128 B row and stage
  const int nkb = ONE ? kpad / 64 : kpad / KB;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mfh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mfl)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mlh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mll)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tfull, 1);
    mbar_init(tempty, EPI_WARPS);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer (the warp walks the loop converged; one elect.sync lane issues)
    {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int tm, tl;
        coords(tile, tm, tl);
        const int t0 = tm * BM, l0 = tl * BL;
        for (int kb = 0; kb < nkb; ++kb) {
#ifdef MC_DIAG_TRACE
          // diagnostic build only: CTA 0 logs producer wait intervals into D (results invalid)
          long long* trace = reinterpret_cast<long long*>(D + (int64_t)T * ldd);
          const int ev = tile == blockIdx.x ? kb : -1;
          if (blockIdx.x == 0 && ev >= 0 && ev < 4096) trace[4 * ev + 0] = clock64();
          mbar_wait(&empty[stage], phase ^ 1);
          if (blockIdx.x == 0 && ev >= 0 && ev < 4096) trace[4 * ev + 1] = clock64();
#else
          mbar_wait(&empty[stage], phase ^ 1);
#endif
          uint8_t* st = smem + stage * STAGE_BYTES;
#ifdef MC_TF32_NOTMA
          // diagnostic build only: MMAs run on stale shared memory, no operand traffic
          if (umma_elect_one()) mbar_arrive(&full[stage]);
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          continue;
#endif
          if (umma_elect_one()) {
#if defined(MC_DIAG_NOA)
          if (!F16) mbar_expect_tx(&full[stage], STAGE_BYTES); else asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[stage])), "r"(3 * BP2_BYTES) : "memory");
#elif defined(MC_DIAG_NOB)
          if (!F16) mbar_expect_tx(&full[stage], STAGE_BYTES); else asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[stage])), "r"(3 * A2_BYTES) : "memory");
#else
          mbar_expect_tx(&full[stage], STAGE_BYTES);
#endif
          if constexpr (F16) {
            const int c0 = kb * 64;  // [hi x32 | lo x32] per k-block
#if defined(MC_DIAG_NOA) || defined(MC_DIAG_NOB)
            // diagnostic builds only: drop one operand's traffic (results invalid)
            mbar_arrive(&full[stage]);
#endif
#ifndef MC_DIAG_NOA
#pragma unroll
            for (int p = 0; p < 3; ++p) tma_load_2d(&mfh, &full[stage], st + p * A2_BYTES, c0, p * T + t0);
#endif
#ifndef MC_DIAG_NOB
#pragma unroll
            for (int g = 0; g < 3; ++g)
              tma_load_2d(&mlh, &full[stage], st + 3 * A2_BYTES + g * BP2_BYTES, c0, g * L + l0);
#endif
          } else {
            const int k0 = kb * KB;
#pragma unroll
            for (int p = 0; p < 3; ++p) {
              tma_load_2d(&mfh, &full[stage], st + (2 * p) * A_BYTES, k0, p * T + t0);
              tma_load_2d(&mfl, &full[stage], st + (2 * p + 1) * A_BYTES, k0, p * T + t0);
            }
            uint8_t* bh = st + 6 * A_BYTES;
            uint8_t* bl = bh + B_BYTES;
#pragma unroll
            for (int g = 0; g < 3; ++g) {
              tma_load_2d(&mlh, &full[stage], bh + g * BP_BYTES, k0, g * L + l0);
              tma_load_2d(&mll, &full[stage], bl + g * BP_BYTES, k0, g * L + l0);
            }
          }
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
#ifdef MC_DIAG_TRACE
      if (blockIdx.x == 0 && lane == 0 && it < 256)
        reinterpret_cast<long long*>(D + (int64_t)T * ldd)[4 * 4096 + 2 * it] = clock64();
      mbar_wait(tempty, (it & 1) ^ 1);
      if (blockIdx.x == 0 && lane == 0 && it < 256)
        reinterpret_cast<long long*>(D + (int64_t)T * ldd)[4 * 4096 + 2 * it + 1] = clock64();
#else
      mbar_wait(tempty, (it & 1) ^ 1);
#endif
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (int kb = 0; kb < nkb; ++kb) {
#ifdef MC_DIAG_TRACE
        long long* trace = reinterpret_cast<long long*>(D + (int64_t)T * ldd);
        const int ev = tile == blockIdx.x ? kb : -1;
        if (blockIdx.x == 0 && lane == 0 && ev >= 0 && ev < 4096) trace[4 * ev + 2] = clock64();
        mbar_wait(&full[stage], phase);
        if (blockIdx.x == 0 && lane == 0 && ev >= 0 && ev < 4096) trace[4 * ev + 3] = clock64();
#else
        mbar_wait(&full[stage], phase);
#endif
        asm volatile("tcgen05.fence::after_thread_sync;");
        // one lane chosen by elect.sync issues: under `if (lane == 0)` ptxas wraps every
        // tcgen05.mma / commit in an ELECT ... BRA.U.ANY retry loop (~85 clk of issue path per
        // MMA against 72 clk of tensor-pipe work for M = 128, N = 144, K = 16)
        if (umma_elect_one()) {
          const uint32_t st = smem_u32(smem + stage * STAGE_BYTES);
          if constexpr (F16) {
            // 128 B rows: hi atoms at byte 0..63, lo at 64..127; one MMA = 16 atoms = 32 B
            const uint32_t bb = st + 3 * A2_BYTES;
            if constexpr (ONE) {
              // one-term screen: hi x hi over 64 atoms (4 MMAs of K = 16 per 128 B row)
#pragma unroll
              for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int p = 0; p < 3; ++p)
                  umma<F16>(tmem_base + p * BN, umma_desc_sw128(st + p * A2_BYTES + k * 32),
                            umma_desc_sw128(bb + k * 32), (kb | k) != 0 ? 1u : 0u);
            } else
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const uint32_t koff = k * 32;
              const uint64_t dbh = umma_desc_sw128(bb + koff);
              const uint64_t dbl = umma_desc_sw128(bb + 64 + koff);
#pragma unroll
              for (int term = 0; term < 3; ++term) {
#pragma unroll
                for (int p = 0; p < 3; ++p) {
                  const uint64_t a = umma_desc_sw128(st + p * A2_BYTES + (term == 2 ? 64 : 0) + koff);
                  umma<F16>(tmem_base + p * BN, a, term == 1 ? dbl : dbh, (term | kb | k) != 0 ? 1u : 0u);
                }
              }
            }
          } else {
          const uint32_t bh = st + 6 * A_BYTES, bl = bh + B_BYTES;
#pragma unroll
          for (int k = 0; k < ROWB / 32; ++k) {
            const uint32_t koff = k * 32;  // one MMA = 32 B (8 tf32) inside the 64 B swizzled row
            const uint64_t dbh = umma_desc_sw64(bh + koff);
            const uint64_t dbl = umma_desc_sw64(bl + koff);
            // term-major order: consecutive MMAs target different accumulators,
            // so no MMA waits on the read-modify-write of the one before it
#pragma unroll
            for (int term = 0; term < 3; ++term) {
#pragma unroll
              for (int p = 0; p < 3; ++p) {
                const uint32_t d = tmem_base + p * BN;
                const uint64_t a = umma_desc_sw64(st + (2 * p + (term == 2 ? 1 : 0)) * A_BYTES + koff);
                umma<F16>(d, a, term == 1 ? dbl : dbh, (term | kb | k) != 0 ? 1u : 0u);
              }
            }
          }
          }
          umma_commit(&empty[stage]);
          if (kb == nkb - 1) umma_commit(tfull);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: lane = frame, whole 3x3 blocks per thread
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int row = q * 32 + lane;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      int tm, tl;
      coords(tile, tm, tl);
      const int t = tm * BM + row;
      const int l0 = tl * BL;
      mbar_wait(tfull, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#ifdef MC_DIAG_TRACE
      if (blockIdx.x == 0 && lane == 0 && it < 256)
        reinterpret_cast<long long*>(D + (int64_t)T * ldd)[5 * 4096 + 16 * it + 2 * (warp - 4)] = clock64();
#endif
      const double gxt = t < T ? gx[t] : 0.0;
      const double fst = (F16 && t < T) ? fsc[t] : 1.0;
      const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = half; c < BL / 8; c += EPI_WARPS / 4) {
        float v[9][8];
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
          for (int g = 0; g < 3; ++g) tmem_ld8(lane_base + p * BN + g * BL + c * 8, v[p * 3 + g]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#ifdef MC_DIAG_TRACE
        long long tq0 = clock64();
#endif
        if (t < T) {
          float out[8];
          msd8_estimate(v, gxt, ga, fst, F16 ? lsc : nullptr, l0 + c * 8, L, out);
#ifdef MC_DIAG_TRACE
          __syncwarp();
          if (blockIdx.x == 0 && lane == 0 && it < 256 && warp == 4)
            reinterpret_cast<long long*>(D + (int64_t)T * ldd)[6 * 4096 + 8 * it + c] = clock64() - tq0;
#endif
          float* dst = D + (int64_t)t * ldd + l0 + c * 8;
          if (l0 + c * 8 + 8 <= L && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
            reinterpret_cast<float4*>(dst)[0] = make_float4(out[0], out[1], out[2], out[3]);
            reinterpret_cast<float4*>(dst)[1] = make_float4(out[4], out[5], out[6], out[7]);
          } else {
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (l0 + c * 8 + i < L) dst[i] = out[i];
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
#ifdef MC_DIAG_TRACE
      if (blockIdx.x == 0 && lane == 0 && it < 256)
        reinterpret_cast<long long*>(D + (int64_t)T * ldd)[5 * 4096 + 16 * it + 2 * (warp - 4) + 1] = clock64();
#endif
      if (lane == 0) mbar_arrive(tempty);
    }
  }
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(gemm::TMEM_COLS));
  }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

// 2-D map over a plane-major operand [rows][row_elems] of esz-byte elements;
// one box = box_rows rows x 64 B (SWIZZLE_64B: TF32 hi or lo planes) or x 128 B
// (SWIZZLE_128B: interleaved F16 hi|lo rows).  Shared with tf32_gemm_2sm.cu.
bool make_operand_map(CUtensorMap* m, const void* base, int esz, int64_t rows, int64_t row_elems, int box_rows,
                      bool sw128) {
  auto enc = get_encode();
  if (!enc) return false;
  const int box_bytes = sw128 ? 128 : 64;
  cuuint64_t dims[2] = {(cuuint64_t)row_elems, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)row_elems * esz};
  cuuint32_t box[2] = {(cuuint32_t)(box_bytes / esz), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   sw128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool F16, bool ONE = false>
static cudaError_t launch_gemm1(const void* fh, const void* fl, const void* lh, const void* ll, const double* gx,
                                const double* ga, const double* fsc, const double* lsc, int T, int L, int kpad,
                                float* D, int64_t ldd, int grid, cudaStream_t stream, const int* tlist = nullptr,
                                const int* nlist = nullptr) {
  using namespace gemm;
  if (T <= 0 || L <= 0) return cudaSuccess;
  if (kpad % (ONE ? 64 : Fmt<F16>::KB)) return cudaErrorInvalidValue;
  constexpr int esz = Fmt<F16>::ESZ;
  CUtensorMap mfh, mfl, mlh, mll;
  if (F16) {
    // interleaved rows of 2 kpad halves (one-term: kpad hi halves); the lo maps are unused
    const int64_t re = ONE ? kpad : 2LL * kpad;
    if (!make_operand_map(&mfh, fh, esz, 3LL * T, re, BM, true) || !make_operand_map(&mlh, lh, esz, 3LL * L, re, BL, true))
      return cudaErrorInvalidValue;
    mfl = mfh;
    mll = mlh;
  } else if (!make_operand_map(&mfh, fh, esz, 3LL * T, kpad, BM, false) ||
             !make_operand_map(&mfl, fl, esz, 3LL * T, kpad, BM, false) ||
             !make_operand_map(&mlh, lh, esz, 3LL * L, kpad, BL, false) ||
             !make_operand_map(&mll, ll, esz, 3LL * L, kpad, BL, false)) {
    return cudaErrorInvalidValue;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(msd_tf32_kernel<F16, ONE>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  // with a device-side tile list the count is only known on the device: one CTA per SM
  const int ntiles = tlist ? 1 << 30 : ((T + BM - 1) / BM) * ((L + BL - 1) / BL);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int g = grid > 0 ? grid : (ntiles < nsm ? ntiles : nsm);
  msd_tf32_kernel<F16, ONE><<<g, NT, SMEM_BYTES, stream>>>(mfh, mfl, mlh, mll, gx, ga, fsc, lsc, T, L, kpad, D, ldd,
                                                           tlist, nlist);
  return cudaGetLastError();
}

cudaError_t launch_msd_tf32(const float* fh, const float* fl, const float* lh, const float* ll, const double* gx,
                            const double* ga, int T, int L, int kpad, float* D, int64_t ldd, int grid,
                            cudaStream_t stream) {
  return launch_gemm1<false>(fh, fl, lh, ll, gx, ga, nullptr, nullptr, T, L, kpad, D, ldd, grid, stream);
}

cudaError_t launch_msd_f16(const void* fhl, const void* lhl, const double* fsc, const double* lsc, const double* gx,
                           const double* ga, int T, int L, int kpad, int terms, float* D, int64_t ldd, int grid,
                           cudaStream_t stream, const int* tlist, const int* nlist) {
  if (terms == 1)
    return launch_gemm1<true, true>(fhl, nullptr, lhl, nullptr, gx, ga, fsc, lsc, T, L, kpad, D, ldd, grid, stream,
                                    tlist, nlist);
  return launch_gemm1<true>(fhl, nullptr, lhl, nullptr, gx, ga, fsc, lsc, T, L, kpad, D, ldd, grid, stream, tlist,
                            nlist);
}

}  // namespace mc
