// K1 — per-structure centring and norms (geometry.py:67-76 batched).
//
// One CTA per structure.  Reads AoS coordinates [B, N, 3] (fp32 or fp64,
// coalesced: a warp covers 32 consecutive atoms = 384/768 contiguous bytes),
// writes the centred structure as three zero-padded fp64 planes
// [B, 3, npad] (the layout every downstream kernel and the GEMM operands
// use), plus per-structure scalars:
//   centroid c = sum_j w'_j x_j                   (geometry.py:67-69)
//   G          = sum_j w_j |x_j - c|^2            (the Gx / Ga of Horn's form)
//   wbar       = sum_j w_j (x_j - c)              (closed-form gradient sums)
//   mom        = sum_j w_j (x_j - c)(x_j - c)^T   (6 entries, landmark A_i)
// Optionally also the w-weighted planes w_j (x_j - c) (GEMM B operand).
// All reductions are fixed-order (deterministic).
#include "mc_math.cuh"

namespace mc {

template <typename T, int NT>
__global__ void __launch_bounds__(NT) center_kernel(const T* __restrict__ coords, int n, int npad,
                                                   const double* __restrict__ w_align,
                                                   const double* __restrict__ w_disp,
                                                   double* __restrict__ planes,
                                                   double* __restrict__ wplanes,
                                                   double* __restrict__ centroid,
                                                   double* __restrict__ gnorm,
                                                   double* __restrict__ wbar,
                                                   double* __restrict__ mom,
                                                   uint8_t* __restrict__ flags) {
  __shared__ double scratch[NT / 32];
  const int64_t b = blockIdx.x;
  const T* x = coords + b * (int64_t)n * 3;
  double cx = 0.0, cy = 0.0, cz = 0.0;
  bool finite = true;
  // w_align == nullptr: keep the coordinates as given (kearsley_fit inputs
  // are "expected to be centered" and are used as-is, geometry.py:231-232)
  for (int j = threadIdx.x; j < n; j += NT) {
    const double wa = w_align ? w_align[j] : 0.0;
    const double x0 = (double)x[3 * j], x1 = (double)x[3 * j + 1], x2 = (double)x[3 * j + 2];
    finite = finite && isfinite(x0) && isfinite(x1) && isfinite(x2);
    cx += wa * x0;
    cy += wa * x1;
    cz += wa * x2;
  }
  cx = block_sum<NT>(cx, scratch);
  cy = block_sum<NT>(cy, scratch);
  cz = block_sum<NT>(cz, scratch);
  const int nonfinite = __syncthreads_or(!finite);
  double g = 0.0, b0 = 0.0, b1 = 0.0, b2 = 0.0;
  double m00 = 0.0, m01 = 0.0, m02 = 0.0, m11 = 0.0, m12 = 0.0, m22 = 0.0;
  double* p0 = planes + b * 3 * (int64_t)npad;
  double* wp0 = wplanes ? wplanes + b * 3 * (int64_t)npad : nullptr;
  for (int j = threadIdx.x; j < npad; j += NT) {
    double x0 = 0.0, x1 = 0.0, x2 = 0.0, w = 0.0;
    if (j < n) {
      w = w_disp[j];
      x0 = (double)x[3 * j] - cx;
      x1 = (double)x[3 * j + 1] - cy;
      x2 = (double)x[3 * j + 2] - cz;
    }
    p0[j] = x0;
    p0[npad + j] = x1;
    p0[2 * npad + j] = x2;
    if (wp0) {
      wp0[j] = w * x0;
      wp0[npad + j] = w * x1;
      wp0[2 * npad + j] = w * x2;
    }
    const double wx0 = w * x0, wx1 = w * x1, wx2 = w * x2;
    g += wx0 * x0 + wx1 * x1 + wx2 * x2;
    b0 += wx0; b1 += wx1; b2 += wx2;
    m00 += wx0 * x0; m01 += wx0 * x1; m02 += wx0 * x2;
    m11 += wx1 * x1; m12 += wx1 * x2; m22 += wx2 * x2;
  }
  g = block_sum<NT>(g, scratch);
  if (wbar) {
    b0 = block_sum<NT>(b0, scratch);
    b1 = block_sum<NT>(b1, scratch);
    b2 = block_sum<NT>(b2, scratch);
  }
  if (mom) {
    m00 = block_sum<NT>(m00, scratch);
    m01 = block_sum<NT>(m01, scratch);
    m02 = block_sum<NT>(m02, scratch);
    m11 = block_sum<NT>(m11, scratch);
    m12 = block_sum<NT>(m12, scratch);
    m22 = block_sum<NT>(m22, scratch);
  }
  if (threadIdx.x == 0) {
    if (centroid) { centroid[3 * b] = cx; centroid[3 * b + 1] = cy; centroid[3 * b + 2] = cz; }
    gnorm[b] = g;
    if (wbar) { wbar[3 * b] = b0; wbar[3 * b + 1] = b1; wbar[3 * b + 2] = b2; }
    if (mom) {
      mom[6 * b] = m00; mom[6 * b + 1] = m01; mom[6 * b + 2] = m02;
      mom[6 * b + 3] = m11; mom[6 * b + 4] = m12; mom[6 * b + 5] = m22;
    }
    if (flags) flags[b] = nonfinite ? kFlagNonFinite : 0;
  }
}

cudaError_t launch_center(const void* coords, int dtype, int64_t count, int n, int npad,
                          const double* w_align, const double* w_disp, double* planes, double* wplanes,
                          double* centroid, double* gnorm, double* wbar, double* mom, uint8_t* flags,
                          cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  constexpr int NT = 256;
  if (dtype == 0) {
    center_kernel<float, NT><<<(unsigned)count, NT, 0, stream>>>(
        (const float*)coords, n, npad, w_align, w_disp, planes, wplanes, centroid, gnorm, wbar, mom, flags);
  } else {
    center_kernel<double, NT><<<(unsigned)count, NT, 0, stream>>>(
        (const double*)coords, n, npad, w_align, w_disp, planes, wplanes, centroid, gnorm, wbar, mom, flags);
  }
  return cudaGetLastError();
}

}  // namespace mc
