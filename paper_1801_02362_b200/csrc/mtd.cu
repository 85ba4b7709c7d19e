// Metadynamics bias and bias force on the device (SPEC [MODULE] metadynamics,
// PAPER Eq. 1): consumes the path CVs (s, z) and their atom
// gradients where they already live and returns V and the bias force [T, N, 3].
//
//   mtd_bias_kernel    direct hill sum, one thread per frame, hills staged in
//                      shared memory tiles: V = sum_h w_h prod_i exp(-u_hi^2/2),
//                      dV/dS_i = sum_h V_h (-u_hi / sigma_hi)
//   mtd_deposit_kernel one thread per grid node: adds a hill (value, first
//                      derivatives, cross derivative) within 6 sigma
//   mtd_eval_kernel    cubic Hermite interpolation (tensor product for d = 2)
//   mtd_force_kernel   F = -sum_i dV/dS_i dS_i/dx, streaming (HBM-bound)
#include <type_traits>

#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int MNT = 256;
constexpr int MAXD = 3;
constexpr uint8_t kFlagOutOfGrid = 32;
}  // namespace

__global__ void __launch_bounds__(MNT)
mtd_bias_kernel(const double* __restrict__ cv, int T, int d, const double* __restrict__ centers,
                const double* __restrict__ sigmas, const double* __restrict__ heights, int H, double* __restrict__ V,
                double* __restrict__ dV) {
  __shared__ double sc[MNT * MAXD], sinv[MNT * MAXD], sw[MNT];
  const int t = blockIdx.x * MNT + threadIdx.x;
  double x[MAXD] = {0.0, 0.0, 0.0};
  if (t < T)
    for (int i = 0; i < d; ++i) x[i] = cv[(int64_t)t * d + i];
  double v = 0.0, g[MAXD] = {0.0, 0.0, 0.0};
  for (int h0 = 0; h0 < H; h0 += MNT) {
    const int nh = min(MNT, H - h0);
    __syncthreads();
    if (threadIdx.x < nh) {
      const int h = h0 + threadIdx.x;
      for (int i = 0; i < d; ++i) {
        sc[threadIdx.x * MAXD + i] = centers[(int64_t)h * d + i];
        sinv[threadIdx.x * MAXD + i] = 1.0 / sigmas[(int64_t)h * d + i];
      }
      sw[threadIdx.x] = heights[h];
    }
    __syncthreads();
    for (int k = 0; k < nh; ++k) {
      double u[MAXD], q = 0.0;
#pragma unroll
      for (int i = 0; i < MAXD; ++i) {
        u[i] = i < d ? (x[i] - sc[k * MAXD + i]) * sinv[k * MAXD + i] : 0.0;
        q = fma(u[i], u[i], q);
      }
      const double e = sw[k] * exp(-0.5 * q);
      v += e;
#pragma unroll
      for (int i = 0; i < MAXD; ++i) g[i] = fma(-e * u[i], i < d ? sinv[k * MAXD + i] : 0.0, g[i]);
    }
  }
  if (t < T) {
    V[t] = v;
    for (int i = 0; i < d; ++i) dV[(int64_t)t * d + i] = g[i];
  }
}

struct GridGeom {
  int d;
  double lo[2], h[2];
  int bins[2];
};

__global__ void __launch_bounds__(MNT)
mtd_deposit_kernel(double* __restrict__ val, double* __restrict__ dgrid, double* __restrict__ dxy, GridGeom gg,
                   const double* __restrict__ center, const double* __restrict__ sigma, double height, double cutoff,
                   uint8_t* __restrict__ flag) {
  const int n0 = gg.bins[0] + 1, n1 = gg.d == 2 ? gg.bins[1] + 1 : 1;
  const int64_t nodes = (int64_t)n0 * n1;
  const int64_t e = (int64_t)blockIdx.x * MNT + threadIdx.x;
  const double c0 = center[0], s0 = sigma[0];
  const double c1 = gg.d == 2 ? center[1] : 0.0, s1 = gg.d == 2 ? sigma[1] : 1.0;
  // a centre off the grid is rejected by every thread: the grid stays untouched, so grid and
  // direct-sum V agree for any deposition history (also for callers of the C ABI)
  bool out = !(c0 >= gg.lo[0] && c0 <= gg.lo[0] + gg.h[0] * gg.bins[0]);
  if (gg.d == 2) out = out || !(c1 >= gg.lo[1] && c1 <= gg.lo[1] + gg.h[1] * gg.bins[1]);
  if (e == 0 && flag) *flag = out ? kFlagOutOfGrid : 0;
  if (out || e >= nodes) return;
  const int i0 = (int)(e / n1), i1 = (int)(e - (int64_t)i0 * n1);
  const double u0 = (gg.lo[0] + gg.h[0] * i0 - c0) / s0;
  if (!(fabs(u0) <= cutoff)) return;
  if (gg.d == 1) {
    const double g = height * exp(-0.5 * u0 * u0);
    val[e] += g;
    dgrid[e] += g * (-u0 / s0);
    return;
  }
  const double u1 = (gg.lo[1] + gg.h[1] * i1 - c1) / s1;
  if (!(fabs(u1) <= cutoff)) return;
  const double g = height * exp(-0.5 * (u0 * u0 + u1 * u1));
  const double a0 = -u0 / s0, a1 = -u1 / s1;
  val[e] += g;
  dgrid[e] += g * a0;
  dgrid[nodes + e] += g * a1;
  dxy[e] += g * a0 * a1;
}

__device__ __forceinline__ void hermite(double t, double* b) {
  const double t2 = t * t, t3 = t2 * t;
  b[0] = 2 * t3 - 3 * t2 + 1;  // H0 at node 0
  b[1] = -2 * t3 + 3 * t2;     // H0 at node 1
  b[2] = t3 - 2 * t2 + t;      // H1 at node 0
  b[3] = t3 - t2;              // H1 at node 1
  b[4] = 6 * t2 - 6 * t;       // derivatives of the above
  b[5] = -6 * t2 + 6 * t;
  b[6] = 3 * t2 - 4 * t + 1;
  b[7] = 3 * t2 - 2 * t;
}

__global__ void __launch_bounds__(MNT)
mtd_eval_kernel(const double* __restrict__ val, const double* __restrict__ dgrid, const double* __restrict__ dxy,
                GridGeom gg, const double* __restrict__ cv, int T, double* __restrict__ V, double* __restrict__ dV,
                uint8_t* __restrict__ flags) {
  const int t = blockIdx.x * MNT + threadIdx.x;
  if (t >= T) return;
  const int d = gg.d;
  int k[2] = {0, 0};
  double tt[2] = {0.0, 0.0};
  bool out = false;
  for (int i = 0; i < d; ++i) {
    const double s = cv[(int64_t)t * d + i];
    const double x = (s - gg.lo[i]) / gg.h[i];
    out = out || !(x >= 0.0 && x <= (double)gg.bins[i]);
    int kk = (int)floor(x);
    kk = max(0, min(kk, gg.bins[i] - 1));
    k[i] = kk;
    tt[i] = x - kk;
  }
  if (flags) flags[t] = out ? kFlagOutOfGrid : 0;
  if (out) {
    V[t] = 0.0;
    for (int i = 0; i < d; ++i) dV[(int64_t)t * d + i] = 0.0;
    return;
  }
  double bx[8], by[8];
  hermite(tt[0], bx);
  if (d == 1) {
    const double h = gg.h[0];
    const double f0 = val[k[0]], f1 = val[k[0] + 1], g0 = dgrid[k[0]] * h, g1 = dgrid[k[0] + 1] * h;
    V[t] = bx[0] * f0 + bx[1] * f1 + bx[2] * g0 + bx[3] * g1;
    dV[t] = (bx[4] * f0 + bx[5] * f1 + bx[6] * g0 + bx[7] * g1) / h;
    return;
  }
  hermite(tt[1], by);
  const int n1 = gg.bins[1] + 1;
  const int64_t nodes = (int64_t)(gg.bins[0] + 1) * n1;
  const double hx = gg.h[0], hy = gg.h[1];
  double v = 0.0, vx = 0.0, vy = 0.0;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const int64_t e = (int64_t)(k[0] + a) * n1 + k[1] + b;
      const double f = val[e], fx = dgrid[e] * hx, fy = dgrid[nodes + e] * hy, fxy = dxy[e] * hx * hy;
      const double H0x = bx[a], H1x = bx[2 + a], D0x = bx[4 + a], D1x = bx[6 + a];
      const double H0y = by[b], H1y = by[2 + b], D0y = by[4 + b], D1y = by[6 + b];
      v += f * H0x * H0y + fx * H1x * H0y + fy * H0x * H1y + fxy * H1x * H1y;
      vx += f * D0x * H0y + fx * D1x * H0y + fy * D0x * H1y + fxy * D1x * H1y;
      vy += f * H0x * D0y + fx * H1x * D0y + fy * H0x * D1y + fxy * H1x * D1y;
    }
  V[t] = v;
  dV[(int64_t)t * 2] = vx / hx;
  dV[(int64_t)t * 2 + 1] = vy / hy;
}

// F[t, k, c] = -sum_i dV[t, i] G_i[t, k, c] (HBM-bound stream).  One CTA row per
// frame slice: blockIdx.y = frame, dV loaded once, 16-byte vectors when the
// frame's 3N elements are 16-byte aligned (VEC), scalar otherwise.
template <typename E, bool VEC>
__global__ void __launch_bounds__(MNT)
mtd_force_kernel(const double* __restrict__ dV, int d, const E* __restrict__ g0, const E* __restrict__ g1,
                 const E* __restrict__ g2, int64_t per_frame, int T, E* __restrict__ F) {
  for (int64_t t = blockIdx.y; t < T; t += gridDim.y) {
  const double a0 = -dV[t * d], a1 = d > 1 ? -dV[t * d + 1] : 0.0, a2 = d > 2 ? -dV[t * d + 2] : 0.0;
  const int64_t base = t * per_frame;
  constexpr int W = 16 / sizeof(E);
  using V = typename std::conditional<sizeof(E) == 4, float4, double2>::type;
  if (VEC) {
    const int64_t nv = per_frame / W;
    const V* p0 = reinterpret_cast<const V*>(g0 + base);
    const V* p1 = reinterpret_cast<const V*>(g1 + base);
    const V* p2 = reinterpret_cast<const V*>(g2 + base);
    V* out = reinterpret_cast<V*>(F + base);
    for (int64_t v = (int64_t)blockIdx.x * MNT + threadIdx.x; v < nv; v += (int64_t)gridDim.x * MNT) {
      const V x0 = p0[v];
      const E* x0e = reinterpret_cast<const E*>(&x0);
      double acc[W];
#pragma unroll
      for (int c = 0; c < W; ++c) acc[c] = a0 * (double)x0e[c];
      if (d > 1) {
        const V x1 = p1[v];
        const E* x1e = reinterpret_cast<const E*>(&x1);
#pragma unroll
        for (int c = 0; c < W; ++c) acc[c] += a1 * (double)x1e[c];
      }
      if (d > 2) {
        const V x2 = p2[v];
        const E* x2e = reinterpret_cast<const E*>(&x2);
#pragma unroll
        for (int c = 0; c < W; ++c) acc[c] += a2 * (double)x2e[c];
      }
      V r;
      E* re = reinterpret_cast<E*>(&r);
#pragma unroll
      for (int c = 0; c < W; ++c) re[c] = (E)acc[c];
      out[v] = r;
    }
    continue;
  }
  for (int64_t e = (int64_t)blockIdx.x * MNT + threadIdx.x; e < per_frame; e += (int64_t)gridDim.x * MNT) {
    double f = a0 * (double)g0[base + e];
    if (d > 1) f += a1 * (double)g1[base + e];
    if (d > 2) f += a2 * (double)g2[base + e];
    F[base + e] = (E)f;
  }
  }
}

cudaError_t launch_mtd_bias(const double* cv, int T, int d, const double* centers, const double* sigmas,
                            const double* heights, int H, double* V, double* dV, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  mtd_bias_kernel<<<(T + MNT - 1) / MNT, MNT, 0, stream>>>(cv, T, d, centers, sigmas, heights, H, V, dV);
  return cudaGetLastError();
}

static GridGeom geom(int d, const double* lo, const double* hi, const int* bins) {
  GridGeom g{d, {lo[0], d == 2 ? lo[1] : 0.0}, {0.0, 1.0}, {bins[0], d == 2 ? bins[1] : 1}};
  for (int i = 0; i < d; ++i) g.h[i] = (hi[i] - lo[i]) / bins[i];
  return g;
}

cudaError_t launch_mtd_deposit(double* val, double* dgrid, double* dxy, int d, const double* lo, const double* hi,
                               const int* bins, const double* center, const double* sigma, double height,
                               double cutoff, uint8_t* flag, cudaStream_t stream) {
  const GridGeom g = geom(d, lo, hi, bins);
  const int64_t nodes = (int64_t)(g.bins[0] + 1) * (d == 2 ? g.bins[1] + 1 : 1);
  mtd_deposit_kernel<<<(unsigned)((nodes + MNT - 1) / MNT), MNT, 0, stream>>>(val, dgrid, dxy, g, center, sigma, height,
                                                                             cutoff, flag);
  return cudaGetLastError();
}

cudaError_t launch_mtd_eval(const double* val, const double* dgrid, const double* dxy, int d, const double* lo,
                            const double* hi, const int* bins, const double* cv, int T, double* V, double* dV,
                            uint8_t* flags, cudaStream_t stream) {
  if (T <= 0) return cudaSuccess;
  mtd_eval_kernel<<<(T + MNT - 1) / MNT, MNT, 0, stream>>>(val, dgrid, dxy, geom(d, lo, hi, bins), cv, T, V, dV,
                                                          flags);
  return cudaGetLastError();
}

cudaError_t launch_mtd_force(const double* dV, int T, int d, const void* g0, const void* g1, const void* g2,
                             int dtype, int n, void* F, cudaStream_t stream) {
  const int64_t per = 3LL * n;
  if (T <= 0 || per <= 0) return cudaSuccess;
  const int esz = dtype == 0 ? 4 : 8;
  auto al = [](const void* p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool vec = (per * esz) % 16 == 0 && al(g0) && al(g1) && al(g2) && al(F);
  const int64_t units = vec ? per * esz / 16 : per;
  const unsigned bx = (unsigned)((units + MNT * 4 - 1) / (MNT * 4));  // ~4 vectors per thread per frame
  const dim3 grid(bx, (unsigned)(T < 65535 ? T : 65535));
  if (dtype == 0) {
    if (vec)
      mtd_force_kernel<float, true><<<grid, MNT, 0, stream>>>(dV, d, (const float*)g0, (const float*)g1,
                                                              (const float*)g2, per, T, (float*)F);
    else
      mtd_force_kernel<float, false><<<grid, MNT, 0, stream>>>(dV, d, (const float*)g0, (const float*)g1,
                                                               (const float*)g2, per, T, (float*)F);
  } else {
    if (vec)
      mtd_force_kernel<double, true><<<grid, MNT, 0, stream>>>(dV, d, (const double*)g0, (const double*)g1,
                                                               (const double*)g2, per, T, (double*)F);
    else
      mtd_force_kernel<double, false><<<grid, MNT, 0, stream>>>(dV, d, (const double*)g0, (const double*)g1,
                                                                (const double*)g2, per, T, (double*)F);
  }
  return cudaGetLastError();
}

}  // namespace mc
