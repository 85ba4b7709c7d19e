// K4 gradient pass, blocked over frame groups (fp32-coordinate path).
//
//   ds_t,k = 2 w_k (sum_i cs_i x_k - U^s_k) - w'_k corr^s_t,
//   U^s_k  = sum_{i in sig(t)} (cs_i Rhat_i) a_{i,k}          (same for z)
//
// Per frame this is a [6 x 3W] . [3W x N] product with W ~ 60-70 significant
// landmarks; done frame by frame every landmark coordinate is re-read from
// L2/HBM once per frame (~1 TB for config 4).  Here frames are taken in the
// candidate-sort order in groups of G = 8 (their significant windows nearly
// coincide), the group's coefficients c_i Rhat_i are staged in shared memory
// (zero where a landmark is outside a frame's list; warp-uniform skips), and
// each thread owns one atom for all 8 frames (48 fp64 accumulators): every
// landmark coordinate is loaded once per group and feeds 8 x 18 FMAs, and
// the coefficient reads are shared-memory broadcasts.  fp64 throughout
// (U and sum_i c_i x cancel to |d| ~ sqrt(D)).
#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int GG = 8;      // frames per group
constexpr int GW = 96;     // landmarks per staged window chunk (110 KB of coefficients, dynamic smem)
constexpr int GNT2 = 256;  // threads (one atom each per pass)
constexpr int GATOMS = 2048;  // atoms per CTA (8 passes of 256)
constexpr int FVEC2 = 16;
}  // namespace

template <typename OT>
__global__ void __launch_bounds__(GNT2)
cv_grad_block_kernel(int T, int n, int cap, const float* __restrict__ fraw, const double* __restrict__ fcen,
                     const float* __restrict__ lraw, const double* __restrict__ lcen, const double* __restrict__ w,
                     const double* __restrict__ wa, const int* __restrict__ sig_idx,
                     const double* __restrict__ sig_coef, const int* __restrict__ nsig,
                     const double* __restrict__ fvec, const int* __restrict__ perm, OT* __restrict__ ds,
                     OT* __restrict__ dz) {
  extern __shared__ __align__(16) double sCraw[];
  double (*sC)[GW][18] = reinterpret_cast<double (*)[GW][18]>(sCraw);
  __shared__ int s_t[GG], s_ns[GG], s_flo[GG], s_fhi[GG];
  __shared__ double s_fc[GG][3], s_fv[GG][8];
  __shared__ int s_wlo, s_whi;
  const int tid = threadIdx.x;
  const int g = blockIdx.x;
  const int katom0 = blockIdx.y * GATOMS;
  if (tid < GG) {
    const int k = g * GG + tid;
    int t = -1, ns = 0;
    if (k < T) {
      t = perm ? perm[k] : k;
      ns = nsig[t];
    }
    s_t[tid] = t;
    s_ns[tid] = ns;
    s_flo[tid] = (t >= 0 && ns > 0) ? sig_idx[(int64_t)t * cap] : 0x7fffffff;
    s_fhi[tid] = (t >= 0 && ns > 0) ? sig_idx[(int64_t)t * cap + ns - 1] + 1 : -1;
    if (t >= 0) {
      for (int a = 0; a < 3; ++a) s_fc[tid][a] = fcen[3 * t + a];
      const double* fv = fvec + (int64_t)t * FVEC2;
      for (int e = 0; e < 8; ++e) s_fv[tid][e] = fv[e];  // sumcs, sumcz, corr_s[3], corr_z[3]
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
          const int* idx = sig_idx + (int64_t)t * cap;
          const double* co = sig_coef + (int64_t)t * cap * 18;
          for (int e = tid; e < ns * 18; e += GNT2) {
            const int s = e / 18;
            const int l = idx[s] - w0;
            if (l >= 0 && l < wn) sC[f][l][e - s * 18] = co[e];
          }
        }
        __syncthreads();
      }
      // software-pipelined landmark loop: the next landmark's coordinates are
      // in flight while the current one feeds 8 x 18 FMAs (the L2 latency is
      // otherwise exposed at 8 warps/SM).  Coefficients outside a frame's list
      // are zero in sC, so the loop body is branch-free.
      float p0 = 0.f, p1 = 0.f, p2 = 0.f;
      if (on && wn > 0) {
        const float* p = lraw + ((int64_t)w0 * n + k) * 3;
        p0 = p[0]; p1 = p[1]; p2 = p[2];
      }
      for (int l = 0; l < wn; ++l) {
        const int li = w0 + l;
        const double a0 = (double)p0 - lcen[3 * li];
        const double a1 = (double)p1 - lcen[3 * li + 1];
        const double a2 = (double)p2 - lcen[3 * li + 2];
        if (on && l + 1 < wn) {
          const float* p = lraw + ((int64_t)(li + 1) * n + k) * 3;
          p0 = p[0]; p1 = p[1]; p2 = p[2];
        }
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
        const float* xp = fraw + ((int64_t)t * n + k) * 3;
        const double x[3] = {(double)xp[0] - s_fc[f][0], (double)xp[1] - s_fc[f][1], (double)xp[2] - s_fc[f][2]};
        OT* os = ds + ((int64_t)t * n + k) * 3;
        OT* oz = dz + ((int64_t)t * n + k) * 3;
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          os[b] = (OT)(2.0 * wk * (s_fv[f][0] * x[b] - us[f][b]) - wak * s_fv[f][2 + b]);
          oz[b] = (OT)(2.0 * wk * (s_fv[f][1] * x[b] - uz[f][b]) - wak * s_fv[f][5 + b]);
        }
      }
    }
  }
}

cudaError_t launch_cv_grad_block(int T, int n, int cap, const float* fraw, const double* fcen, const float* lraw,
                                 const double* lcen, const double* w, const double* wa, const int* sig_idx,
                                 const double* sig_coef, const int* nsig, const double* fvec, const int* perm,
                                 void* ds, void* dz, int out_f32, cudaStream_t stream) {
  if (T <= 0 || n <= 0) return cudaSuccess;
  dim3 grid((T + GG - 1) / GG, (n + GATOMS - 1) / GATOMS);
  const int smem = GG * GW * 18 * (int)sizeof(double);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(cv_grad_block_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(cv_grad_block_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  if (out_f32)
    cv_grad_block_kernel<float><<<grid, GNT2, smem, stream>>>(T, n, cap, fraw, fcen, lraw, lcen, w, wa, sig_idx,
                                                            sig_coef, nsig, fvec, perm, (float*)ds, (float*)dz);
  else
    cv_grad_block_kernel<double><<<grid, GNT2, smem, stream>>>(T, n, cap, fraw, fcen, lraw, lcen, w, wa, sig_idx,
                                                             sig_coef, nsig, fvec, perm, (double*)ds, (double*)dz);
  return cudaGetLastError();
}

}  // namespace mc
