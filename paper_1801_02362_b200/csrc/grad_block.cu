// K4 gradient pass, blocked over frame groups.
//
//   ds_t,k = 2 w_k (sum_i cs_i x_k - U^s_k) [+ v_s^T dK_k q0] - w'_k corr^s_t,
//   U^s_k  = sum_{i in sig(t)} (cs_i Rhat_i) a_{i,k}          (same for z)
//
// Per frame this is a [6 x 3W] . [3W x N] product with W significant
// landmarks; done frame by frame every landmark coordinate is re-read from
// L2/HBM once per frame.  Here frames are taken in groups of G = 8 whose
// significant windows nearly coincide (candidate-sort order on the fp32 path,
// consecutive trajectory frames on the fp64 / close-structure path), the
// group's coefficients c_i Rhat_i are staged in shared memory (zero where a
// landmark is outside a frame's list), and each thread owns one atom for all
// 8 frames (48 fp64 accumulators): every landmark coordinate is loaded once
// per group and feeds 8 x 18 FMAs, the coefficient reads are shared-memory
// broadcasts, and the next landmark's coordinates are in flight while the
// current one is consumed.  fp64 throughout (U and sum_i c_i x cancel to
// |d| ~ sqrt(D)).
//
// PL = false: coordinates from the raw fp32 AoS input + fp64 centroids (fp32
//             path, exact-refit rows only).
// PL = true:  coordinates from centred fp64 planes; non-refresh rows of the
//             close-structure replay add the Eq. 6 dR_xy term in closed form.
#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int GG = 8;         // frames per group
constexpr int GW = 96;        // landmarks per staged window chunk (110 KB of coefficients, dynamic smem)
constexpr int GNT2 = 256;     // threads (one atom each per pass)
constexpr int GATOMS = 2048;  // atoms per CTA (8 passes of 256)
constexpr int FVEC2 = 16;
}  // namespace

struct GradSrc {
  const float* fraw;
  const double* fcen;
  const float* lraw;
  const double* lcen;
  const double* fpl;
  const double* lpl;
  int npad;
  const uint8_t* refresh;
  const int* ridx;
  const double* xyeig;
  int t0;  // global index of the first frame of this launch (sig lists / fvec are chunk-local)
};

template <typename OT, bool PL>
__global__ void __launch_bounds__(GNT2)
cv_grad_block_kernel(int T, int n, int cap, GradSrc src, const double* __restrict__ w, const double* __restrict__ wa,
                     const int* __restrict__ sig_idx, const double* __restrict__ sig_coef,
                     const int* __restrict__ nsig, const double* __restrict__ fvec, const int* __restrict__ perm,
                     OT* __restrict__ ds, OT* __restrict__ dz) {
  extern __shared__ __align__(16) double sCraw[];
  double (*sC)[GW][18] = reinterpret_cast<double (*)[GW][18]>(sCraw);
  __shared__ int s_t[GG], s_ns[GG], s_flo[GG], s_fhi[GG], s_y[GG], s_ap[GG];
  __shared__ double s_fc[GG][3], s_fv[GG][16], s_q0[GG][4];
  __shared__ int s_wlo, s_whi;
  const int tid = threadIdx.x;
  const int g = blockIdx.x;
  const int katom0 = blockIdx.y * GATOMS;
  const int npad = src.npad;
  if (tid < GG) {
    const int k = g * GG + tid;
    int t = -1, ns = 0, tl = 0;
    if (k < T) {
      tl = perm ? perm[k] : k;
      t = src.t0 + tl;
      ns = nsig[tl];
    }
    s_t[tid] = t;
    s_ns[tid] = ns;
    s_flo[tid] = (t >= 0 && ns > 0) ? sig_idx[(int64_t)tl * cap] : 0x7fffffff;
    s_fhi[tid] = (t >= 0 && ns > 0) ? sig_idx[(int64_t)tl * cap + ns - 1] + 1 : -1;
    s_ap[tid] = 0;
    if (t >= 0) {
      for (int a = 0; a < 3; ++a) s_fc[tid][a] = PL ? 0.0 : src.fcen[3 * t + a];
      const double* fv = fvec + (int64_t)tl * FVEC2;
      for (int e = 0; e < 16; ++e) s_fv[tid][e] = fv[e];  // sumcs, sumcz, corr_s[3], corr_z[3], v_s[4], v_z[4]
      if (PL && src.refresh && !src.refresh[t]) {
        s_ap[tid] = 1;
        s_y[tid] = src.ridx[t];
        for (int r = 0; r < 4; ++r) s_q0[tid][r] = src.xyeig[(int64_t)t * 20 + 4 + r * 4];
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    int a = 0x7fffffff, b = -1;
    for (int f = 0; f < GG; ++f) { a = min(a, s_flo[f]); b = max(b, s_fhi[f]); }
    s_wlo = a;
    s_whi = b;
  }
  __syncthreads();
  const int wlo = s_wlo, whi = s_whi;
  // one staged chunk (the usual case): stage once for all atom passes
  const bool restage = whi - wlo > GW;
  bool staged = false;
  for (int k0 = katom0; k0 < min(n, katom0 + GATOMS); k0 += GNT2) {
    const int k = k0 + tid;
    const bool on = k < n;
    double us[GG][3], uz[GG][3];
#pragma unroll
    for (int f = 0; f < GG; ++f)
#pragma unroll
      for (int b = 0; b < 3; ++b) us[f][b] = uz[f][b] = 0.0;
    for (int w0 = wlo; w0 < whi; w0 += GW) {
      const int wn = min(GW, whi - w0);
      if (restage || !staged) {  // block-uniform condition
        staged = true;
        __syncthreads();
        for (int e = tid; e < GG * GW * 18; e += GNT2) (&sC[0][0][0])[e] = 0.0;
        __syncthreads();
        // scatter each frame's (ordered) significant slots that fall in [w0, w0 + wn)
        for (int f = 0; f < GG; ++f) {
          const int t = s_t[f];
          if (t < 0) continue;
          const int ns = s_ns[f];
          const int* idx = sig_idx + (int64_t)(t - src.t0) * cap;
          const double* co = sig_coef + (int64_t)(t - src.t0) * cap * 18;
          for (int e = tid; e < ns * 18; e += GNT2) {
            const int s = e / 18;
            const int l = idx[s] - w0;
            if (l >= 0 && l < wn) sC[f][l][e - s * 18] = co[e];
          }
        }
        __syncthreads();
      }
      // software-pipelined landmark loop (next landmark's coordinates in flight)
      double n0 = 0.0, n1 = 0.0, n2 = 0.0;
      auto load_a = [&](int li, double& a0, double& a1, double& a2) {
        if (PL) {
          const double* p = src.lpl + (int64_t)li * 3 * npad + k;
          a0 = p[0]; a1 = p[npad]; a2 = p[2 * npad];
        } else {
          const float* p = src.lraw + ((int64_t)li * n + k) * 3;
          a0 = (double)p[0]; a1 = (double)p[1]; a2 = (double)p[2];
        }
      };
      if (on && wn > 0) load_a(w0, n0, n1, n2);
      for (int l = 0; l < wn; ++l) {
        const int li = w0 + l;
        double a0 = n0, a1 = n1, a2 = n2;
        if (!PL) {
          a0 -= src.lcen[3 * li];
          a1 -= src.lcen[3 * li + 1];
          a2 -= src.lcen[3 * li + 2];
        }
        if (on && l + 1 < wn) load_a(li + 1, n0, n1, n2);
#pragma unroll
        for (int f = 0; f < GG; ++f) {
          const double2* C2 = reinterpret_cast<const double2*>(sC[f][l]);
          double C[18];
#pragma unroll
          for (int e = 0; e < 9; ++e) {
            const double2 v = C2[e];
            C[2 * e] = v.x;
            C[2 * e + 1] = v.y;
          }
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            us[f][b] = fma(C[b * 3], a0, fma(C[b * 3 + 1], a1, fma(C[b * 3 + 2], a2, us[f][b])));
            uz[f][b] = fma(C[9 + b * 3], a0, fma(C[9 + b * 3 + 1], a1, fma(C[9 + b * 3 + 2], a2, uz[f][b])));
          }
        }
      }
    }
    if (on) {
      const double wk = w[k], wak = wa[k];
#pragma unroll
      for (int f = 0; f < GG; ++f) {
        const int t = s_t[f];
        if (t < 0) continue;
        double x[3];
        if (PL) {
          const double* p = src.fpl + (int64_t)t * 3 * npad + k;
          x[0] = p[0]; x[1] = p[npad]; x[2] = p[2 * npad];
        } else {
          const float* xp = src.fraw + ((int64_t)t * n + k) * 3;
          x[0] = (double)xp[0] - s_fc[f][0];
          x[1] = (double)xp[1] - s_fc[f][1];
          x[2] = (double)xp[2] - s_fc[f][2];
        }
        double gs[3], gz[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          gs[b] = 2.0 * wk * (s_fv[f][0] * x[b] - us[f][b]) - wak * s_fv[f][2 + b];
          gz[b] = 2.0 * wk * (s_fv[f][1] * x[b] - uz[f][b]) - wak * s_fv[f][5 + b];
        }
        if (PL && s_ap[f]) {
          const double* py = src.fpl + (int64_t)s_y[f] * 3 * npad + k;
          const double y[3] = {py[0], py[npad], py[2 * npad]};
          double d[3];
          dk_contract(&s_fv[f][8], s_q0[f], wk, x, y, d);
#pragma unroll
          for (int b = 0; b < 3; ++b) gs[b] += d[b];
          dk_contract(&s_fv[f][12], s_q0[f], wk, x, y, d);
#pragma unroll
          for (int b = 0; b < 3; ++b) gz[b] += d[b];
        }
        OT* os = ds + ((int64_t)t * n + k) * 3;
        OT* oz = dz + ((int64_t)t * n + k) * 3;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          os[b] = (OT)gs[b];
          oz[b] = (OT)gz[b];
        }
      }
    }
  }
}

namespace {
template <typename OT, bool PL>
cudaError_t launch_gb(dim3 grid, int smem, cudaStream_t stream, int T, int n, int cap, const GradSrc& src,
                      const double* w, const double* wa, const int* sig_idx, const double* sig_coef,
                      const int* nsig, const double* fvec, const int* perm, void* ds, void* dz) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(cv_grad_block_kernel<OT, PL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  cv_grad_block_kernel<OT, PL><<<grid, GNT2, smem, stream>>>(T, n, cap, src, w, wa, sig_idx, sig_coef, nsig, fvec,
                                                              perm, (OT*)ds, (OT*)dz);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_cv_grad_block(int T, int n, int cap, const float* fraw, const double* fcen, const float* lraw,
                                 const double* lcen, const double* w, const double* wa, const int* sig_idx,
                                 const double* sig_coef, const int* nsig, const double* fvec, const int* perm,
                                 void* ds, void* dz, int out_f32, cudaStream_t stream) {
  if (T <= 0 || n <= 0) return cudaSuccess;
  dim3 grid((T + GG - 1) / GG, (n + GATOMS - 1) / GATOMS);
  const int smem = GG * GW * 18 * (int)sizeof(double);
  GradSrc src{fraw, fcen, lraw, lcen, nullptr, nullptr, 0, nullptr, nullptr, nullptr, 0};
  if (out_f32)
    return launch_gb<float, false>(grid, smem, stream, T, n, cap, src, w, wa, sig_idx, sig_coef, nsig, fvec, perm,
                                   ds, dz);
  return launch_gb<double, false>(grid, smem, stream, T, n, cap, src, w, wa, sig_idx, sig_coef, nsig, fvec, perm, ds,
                                  dz);
}

cudaError_t launch_cv_grad_block_planes(int T, int t0, int n, int npad, int cap, const double* fpl, const double* lpl,
                                        const double* w, const double* wa, const int* sig_idx,
                                        const double* sig_coef, const int* nsig, const double* fvec,
                                        const uint8_t* refresh, const int* ridx, const double* xyeig, void* ds,
                                        void* dz, int out_f32, cudaStream_t stream) {
  if (T <= 0 || n <= 0) return cudaSuccess;
  dim3 grid((T + GG - 1) / GG, (n + GATOMS - 1) / GATOMS);
  const int smem = GG * GW * 18 * (int)sizeof(double);
  GradSrc src{nullptr, nullptr, nullptr, nullptr, fpl, lpl, npad, refresh, ridx, xyeig, t0};
  if (out_f32)
    return launch_gb<float, true>(grid, smem, stream, T, n, cap, src, w, wa, sig_idx, sig_coef, nsig, fvec, nullptr,
                                  ds, dz);
  return launch_gb<double, true>(grid, smem, stream, T, n, cap, src, w, wa, sig_idx, sig_coef, nsig, fvec, nullptr,
                                 ds, dz);
}

}  // namespace mc
