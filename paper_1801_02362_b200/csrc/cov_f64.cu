// All-pairs 3x3 covariance in fp64 on CUDA cores (fp64-coordinate path,
// configs 0/1):  S[t, l, b*3+g] = sum_j x_{t,j,b} * (w_j a_{l,j,g}).
//
// It is the dense contraction [3T x N] . [N x 3L] that replaces the per-pair
// _kearsley_matrix (geometry.py:180-196): the 4x4 Kearsley form is a linear
// function of S and the two norms (mc_math.cuh).  fp64 inputs are exact here,
// so no split-precision is needed; the fp32 configs use the tcgen05 3xTF32
// kernel instead (tf32_gemm.cu).
//
// Tiling: CTA = 32 frames x 32 landmarks, 256 threads (16x16), each thread a
// 2x2 micro-tile of pairs (36 fp64 accumulators).  Atoms are staged through
// shared memory in chunks of 8 with a register prefetch of the next chunk.
#include <cstdlib>

#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int TF = 32, TL = 32, KC = 8, NT = 256;
constexpr int RS = TF + 2;          // padded row stride (doubles), keeps double2 alignment
constexpr int LOADS = TF * 3 * KC / NT;  // 3 per thread per operand
}

__global__ void __launch_bounds__(NT, 2)
cov_f64_kernel(const double* __restrict__ fpl, const double* __restrict__ lpl, int T, int L, int npad,
               double* __restrict__ S) {
  __shared__ __align__(16) double sF[2][KC * 3 * RS];
  __shared__ __align__(16) double sL[2][KC * 3 * RS];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int t0 = blockIdx.y * TF, l0 = blockIdx.x * TL;

  double rf[LOADS], rl[LOADS];
  auto gload = [&](int k0) {
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int e = tid + NT * r;
      const int f = e / (3 * KC);
      const int rem = e - f * 3 * KC;
      const int b = rem / KC;
      const int j = rem - b * KC;
      const int t = t0 + f, l = l0 + f;
      rf[r] = (t < T) ? fpl[((int64_t)t * 3 + b) * npad + k0 + j] : 0.0;
      rl[r] = (l < L) ? lpl[((int64_t)l * 3 + b) * npad + k0 + j] : 0.0;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int r = 0; r < LOADS; ++r) {
      const int e = tid + NT * r;
      const int f = e / (3 * KC);
      const int rem = e - f * 3 * KC;
      const int b = rem / KC;
      const int j = rem - b * KC;
      sF[buf][(j * 3 + b) * RS + f] = rf[r];
      sL[buf][(j * 3 + b) * RS + f] = rl[r];
    }
  };

  double acc[2][2][9];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int e = 0; e < 9; ++e) acc[a][c][e] = 0.0;

  const int nchunks = npad / KC;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nchunks) gload((ch + 1) * KC);
#pragma unroll 4
    for (int j = 0; j < KC; ++j) {
      double2 xf[3], al[3];
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        xf[b] = *reinterpret_cast<const double2*>(&sF[buf][(j * 3 + b) * RS + 2 * ty]);
        al[b] = *reinterpret_cast<const double2*>(&sL[buf][(j * 3 + b) * RS + 2 * tx]);
      }
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          acc[0][0][b * 3 + g] = fma(xf[b].x, al[g].x, acc[0][0][b * 3 + g]);
          acc[0][1][b * 3 + g] = fma(xf[b].x, al[g].y, acc[0][1][b * 3 + g]);
          acc[1][0][b * 3 + g] = fma(xf[b].y, al[g].x, acc[1][0][b * 3 + g]);
          acc[1][1][b * 3 + g] = fma(xf[b].y, al[g].y, acc[1][1][b * 3 + g]);
        }
    }
    if (ch + 1 < nchunks) sstore(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int t = t0 + 2 * ty + a;
    if (t >= T) continue;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int l = l0 + 2 * tx + c;
      if (l >= L) continue;
      double* out = S + ((int64_t)t * L + l) * 9;
#pragma unroll
      for (int e = 0; e < 9; ++e) out[e] = acc[a][c][e];
    }
  }
}

// The same contraction on the fp64 tensor cores (mma.sync m8n8k4 f64 -> DMMA: exact
// products, fp64 sums): CTA = 32 frames x 32 landmarks, GEMM rows r = b*32 + f (96),
// columns c = g*32 + l (96), K = atoms in chunks of 16 staged by cp.async (double
// buffer).  8 warps, each 6 m-tiles x 3 n-tiles (18 accumulator fragments): per k-step
// 6 A + 3 B fragment loads feed 18 DMMAs.  Row strides of 20 doubles (4 mod 16) keep
// the 8x4 fragment loads conflict-free.
namespace {
constexpr int DF = 32, DL = 32, DK = 16, DNT = 256, DSTR = DK + 4;
}

__device__ __forceinline__ void dmma_f64(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cpa16(void* dst, const void* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

__global__ void __launch_bounds__(DNT, 2)
cov_dmma_f64_kernel(const double* __restrict__ fpl, const double* __restrict__ lpl, int T, int L, int npad,
                    double* __restrict__ S) {
  extern __shared__ __align__(16) double dsm[];  // A[buf] = dsm + buf 96 DSTR, B[buf] = dsm + (2 + buf) 96 DSTR
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int t0 = blockIdx.y * DF, l0 = blockIdx.x * DL;
  const int wm = warp & 1, wn = warp >> 1;  // rows 48 wm .. +48, columns 24 wn .. +24
  // stage k-chunk k0: 96 rows x 16 doubles per operand = 8 x 16 B per row
  auto stage = [&](int buf, int k0) {
#pragma unroll
    for (int u = 0; u < 6; ++u) {
      const int e = tid + u * DNT;  // [0, 1536): operand, row, 16-byte piece
      const int op = e / 768, r = (e % 768) >> 3, q = e & 7;
      const int b = r >> 5, f = r & 31;
      const int s = (op ? l0 : t0) + f;
      const bool ok = s < (op ? L : T);
      const double* src = (op ? lpl : fpl) + ((int64_t)(ok ? s : 0) * 3 + b) * npad + k0 + 2 * q;
      cpa16(dsm + ((op ? 2 : 0) + buf) * 96 * DSTR + r * DSTR + 2 * q, src, ok);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double c[6][3][2];
#pragma unroll
  for (int m = 0; m < 6; ++m)
#pragma unroll
    for (int j = 0; j < 3; ++j) c[m][j][0] = c[m][j][1] = 0.0;
  const int nch = npad / DK;
  stage(0, 0);
  for (int ch = 0; ch < nch; ++ch) {
    const int buf = ch & 1;
    if (ch + 1 < nch) {
      stage(buf ^ 1, (ch + 1) * DK);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* a0 = dsm + buf * 96 * DSTR + (wm * 48 + gq) * DSTR + tq;
    const double* b0 = dsm + (2 + buf) * 96 * DSTR + (wn * 24 + gq) * DSTR + tq;
#pragma unroll
    for (int ks = 0; ks < DK / 4; ++ks) {
      double a[6], b[3];
#pragma unroll
      for (int m = 0; m < 6; ++m) a[m] = a0[m * 8 * DSTR + 4 * ks];
#pragma unroll
      for (int j = 0; j < 3; ++j) b[j] = b0[j * 8 * DSTR + 4 * ks];
#pragma unroll
      for (int m = 0; m < 6; ++m)
#pragma unroll
        for (int j = 0; j < 3; ++j) dmma_f64(c[m][j], a[m], b[j]);
    }
    __syncthreads();  // buf is restaged two chunks later
  }
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    const int r = wm * 48 + m * 8 + gq, b = r >> 5, f = r & 31;
    const int t = t0 + f;
    if (t >= T) continue;
#pragma unroll
    for (int j = 0; j < 3; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = wn * 24 + j * 8 + 2 * tq + e, g = cc >> 5, l = l0 + (cc & 31);
        if (l < L) S[((int64_t)t * L + l) * 9 + b * 3 + g] = c[m][j][e];
      }
  }
}

cudaError_t launch_cov_f64(const double* fpl, const double* lpl, int T, int L, int npad, double* S,
                           cudaStream_t stream) {
  if (T <= 0 || L <= 0) return cudaSuccess;
  static const bool cores = getenv("MC_COV_F64") && atoi(getenv("MC_COV_F64")) == 1;  // 1: CUDA-core kernel
  if (!cores && npad % DK == 0) {
    constexpr int smem = 4 * 96 * DSTR * (int)sizeof(double);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(cov_dmma_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    dim3 grid((L + DL - 1) / DL, (T + DF - 1) / DF);
    cov_dmma_f64_kernel<<<grid, DNT, smem, stream>>>(fpl, lpl, T, L, npad, S);
    return cudaGetLastError();
  }
  dim3 grid((L + TL - 1) / TL, (T + TF - 1) / TF);
  cov_f64_kernel<<<grid, NT, 0, stream>>>(fpl, lpl, T, L, npad, S);
  return cudaGetLastError();
}

// Paired covariance: S[p] = sum_j x_{xi[p],j} (w_j a_{ai[p],j})^T for an
// explicit list of (x, a) structure index pairs.  One warp per pair; used by
// the close-structure window (frame vs earlier frame) and by the per-pair API.
__global__ void __launch_bounds__(256)
cov_pairs_kernel(const double* __restrict__ xpl, const double* __restrict__ apl, const int* __restrict__ xi,
                 const int* __restrict__ ai, int64_t P, int npad, const double* __restrict__ w,
                 double* __restrict__ S) {
  const int64_t p = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= P) return;
  const int xs = xi ? xi[p] : (int)p;
  const int as = ai ? ai[p] : (int)p;
  double acc[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) acc[e] = 0.0;
  if (xs >= 0 && as >= 0) {
    const double* x = xpl + (int64_t)xs * 3 * npad;
    const double* a = apl + (int64_t)as * 3 * npad;
    for (int j = lane; j < npad; j += 32) {
      const double wj = w ? w[j] : 1.0;
      const double x0 = x[j], x1 = x[npad + j], x2 = x[2 * npad + j];
      const double a0 = wj * a[j], a1 = wj * a[npad + j], a2 = wj * a[2 * npad + j];
      acc[0] = fma(x0, a0, acc[0]); acc[1] = fma(x0, a1, acc[1]); acc[2] = fma(x0, a2, acc[2]);
      acc[3] = fma(x1, a0, acc[3]); acc[4] = fma(x1, a1, acc[4]); acc[5] = fma(x1, a2, acc[5]);
      acc[6] = fma(x2, a0, acc[6]); acc[7] = fma(x2, a1, acc[7]); acc[8] = fma(x2, a2, acc[8]);
    }
  }
#pragma unroll
  for (int e = 0; e < 9; ++e) acc[e] = warp_sum(acc[e]);
  if (lane == 0) {
#pragma unroll
    for (int e = 0; e < 9; ++e) S[p * 9 + e] = acc[e];
  }
}

cudaError_t launch_cov_pairs(const double* xpl, const double* apl, const int* xi, const int* ai, int64_t P,
                             int npad, const double* w, double* S, cudaStream_t stream) {
  if (P <= 0) return cudaSuccess;
  cov_pairs_kernel<<<(unsigned)((P + 7) / 8), 256, 0, stream>>>(xpl, apl, xi, ai, P, npad, w, S);
  return cudaGetLastError();
}

}  // namespace mc
