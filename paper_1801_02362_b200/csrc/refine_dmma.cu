// Exact refinement tiles on the fp64 tensor cores (DMMA).
//
// Same contract as refine_kernel (refine.cu): for a group of 32 sorted frames
// and each 32-landmark sub-tile of the group's window union, the exact fp64
// covariances
//   S[t,l][b][g] = sum_j (x_{t,j,b} - c_{t,b}) w_j (a_{l,j,g} - c_{l,g})
// followed by the fused Newton + adjugate fit of the in-window pairs.  Here
// the contraction is a [96 x n] . [n x 96] GEMM on mma.sync m8n8k4 f64
// (rows (axis b, frame), columns (axis g, landmark), exact fp64 products and
// sums), fed by a 4-stage cp.async ring of the raw fp32 rows (32 atoms per
// stage, 16-byte copies when N % 4 == 0); each fragment is centred / weighted
// in registers when it is read.  The accumulators are then staged through shared memory so one
// thread owns whole 3x3 blocks for the fit epilogue.
#include <algorithm>

#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int QF = 32;                 // frames per group
constexpr int QL = 32;                 // landmarks per sub-tile
constexpr int QKC = 32;                // atoms per ring stage
constexpr int QRS = 3 * QKC + 4;       // 100 floats per staged row: conflict-free fragment reads, 16 B aligned
constexpr int QNST = 4;                // ring stages
constexpr int QNT = 256;
constexpr int QSTAGE = (QF + QL) * QRS;              // floats per stage
constexpr int QCS = 3 * QL + 1;                      // staged accumulator row stride (doubles)
constexpr int QRING = QNST * QSTAGE * (int)sizeof(float);
constexpr int QCBYTES = 3 * QF * QCS * (int)sizeof(double);
constexpr int QSMEM = (QRING > QCBYTES ? QRING : QCBYTES) + QNST * QKC * (int)sizeof(double) +
                      2 * QNST * (int)sizeof(uint64_t);
constexpr int QLPT = (QF + QL) * 3 * QKC / QNT;     // 24 raw floats per thread per stage (scalar copies)
constexpr int QV4 = 3 * QKC / 4;                     // 24 float4 per staged row
constexpr int QVPT = (QF + QL) * QV4 / QNT;          // 6 float4 per thread per stage

__device__ __forceinline__ void cpa4(void* dst, const void* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cpa8(void* dst, const void* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cpa16(void* dst, const void* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(c));
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
// arrive on b once every cp.async this thread issued so far has landed
__device__ __forceinline__ void mb_cp_arrive(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          saddr(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
}  // namespace

// UNC (lwbar given): frames enter the contraction uncentred -- A = x, B = w (a - c_l) --
// and S = S_half - c_x lwbar^T with lwbar_l = sum_j w_j (a_lj - c_l) (zero in exact
// arithmetic when the displacement and alignment weights coincide), which saves the
// per-fragment frame centring (6 DADD and 12 registers per k-step); no cancellation,
// since S_half - S = c_x lwbar^T is itself ~0.
// RAW (uniform weights wuni, fwbar and lwbar given): both operands enter uncentred and
// unweighted -- A = x, B = a, fragments are plain fp32 -> fp64 conversions with no
// fp64 ALU work in the K loop (DADD/DMUL compete with DMMA for issue: 9 per 18 DMMA
// cost 14% of the DMMA rate, tools/_diag/dmma_probe2.cu) -- and the epilogue forms
//   S = wuni S_raw - fwbar c_l^T - c_x lwbar^T - W c_x c_l^T   (W = n wuni),
// whose cancellation costs ~1e-16 |c_x||c_l| / spread^2 relative (~1e-15 on config 4).
template <bool VEC, bool UNC, bool RAW = false>
__global__ void __launch_bounds__(QNT, 2)
refine_dmma_kernel(const float* __restrict__ fr, const double* __restrict__ fc, const float* __restrict__ lr,
                   const double* __restrict__ lc, const double* __restrict__ lwbar, const double* __restrict__ w,
                   const double* __restrict__ gx, const int* __restrict__ fmap, const double* __restrict__ fwbar,
                   double wuni,
                   const double* __restrict__ ga, int T, int L, int n, const int* __restrict__ perm,
                   const int* __restrict__ lo, const int* __restrict__ cnt, int cap, double* __restrict__ Dex,
                   double* __restrict__ Rex, float* __restrict__ Dd, int64_t ldd, uint8_t* __restrict__ flags,
                   int gbase, double* __restrict__ Sout) {
  extern __shared__ __align__(16) unsigned char qsm[];
  float* ring = reinterpret_cast<float*>(qsm);                                     // [QNST][QF + QL][QRS]
  double* sC = reinterpret_cast<double*>(qsm);                                      // [3 QF][QCS] (after the K loop)
  double* sW = reinterpret_cast<double*>(qsm + (QRING > QCBYTES ? QRING : QCBYTES));  // [QNST][QKC]
  // split-barrier ring: every thread's cp.async of a stage arrives on full[slot]
  // (cp.async.mbarrier.arrive), each warp releases the slot on empty[slot]; a thread
  // refills a slot once every warp has released it -- warps drift by up to QNST-2
  // stages instead of meeting at a CTA barrier every stage
  uint64_t* full = reinterpret_cast<uint64_t*>(sW + QNST * QKC);
  uint64_t* empty = full + QNST;
  __shared__ int s_t[QF], s_raw[QF], s_lo[QF], s_cnt[QF];
  __shared__ double s_fc[QF][3];
  __shared__ int s_wlo, s_whi;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;
  // rows: m-tiles 6 wm .. +6; columns: landmarks 8 wn .. +8, all three axes (n-tile j = axis j),
  // so a partial last sub-tile idles whole warps (their DMMA share goes to the co-resident CTA)
  const int wm = warp & 1, wn = warp >> 1;
  if (tid < QF) {
    const int k = (gbase + (int)blockIdx.y) * QF + tid;
    int t = -1, a = 0, c = 0;
    if (k < T) {
      t = perm ? perm[k] : k;
      a = lo ? lo[t] : 0;
      c = lo ? cnt[t] : L;
    }
    s_t[tid] = t;
    s_raw[tid] = (t >= 0 && fmap) ? fmap[t] : t;  // row of frame t in the raw coordinate array
    s_lo[tid] = a;
    s_cnt[tid] = c;
    for (int b = 0; b < 3; ++b) s_fc[tid][b] = t >= 0 ? fc[3 * t + b] : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    int a = L, b = 0;
    for (int i = 0; i < QF; ++i)
      if (s_t[i] >= 0 && s_cnt[i] > 0) { a = min(a, s_lo[i]); b = max(b, s_lo[i] + s_cnt[i]); }
    s_wlo = a;
    s_whi = b;
  }
  __syncthreads();
  const int wlo = s_wlo, whi = s_whi;
  // per-thread fragment constants: frame centroid of each A row tile (axis b = mt / 4)
  double fcA[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const int mt = wm * 6 + i;
    fcA[i] = UNC ? 0.0 : s_fc[(mt & 3) * 8 + gq][mt >> 2];
  }
  const int nch = (n + QKC - 1) / QKC;
  if (tid == 0) {
    for (int i = 0; i < QNST; ++i) { mb_init(&full[i], QNT); mb_init(&empty[i], QNT / 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t gch = 0;  // stages issued by this CTA (ring position / parity)
  // CTA x of a group takes sub-tiles x, x + gridDim.x, ... of the group's union: the
  // work unit is one 32 x 32 sub-tile (~1/3 of a group), so the last wave is short
  for (int l0 = wlo + (int)blockIdx.x * QL; l0 < whi; l0 += (int)gridDim.x * QL) {
    double lcB[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int l = l0 + wn * 8 + gq;
      lcB[i] = (!RAW && l < L) ? lc[3 * l + i] : 0.0;
    }
    const bool wact = l0 + wn * 8 < whi;  // this warp's landmarks intersect the window union
    // ring stage ch: rows 0..31 frames, 32..63 landmarks, 3 QKC floats each (atoms QKC ch ..)
    auto issue = [&](int ch, int slot) {
      const uint32_t g = gch + (uint32_t)ch;
      if (g >= (uint32_t)QNST) mb_wait(&empty[slot], ((g / QNST) - 1) & 1u);
      float* dst = ring + slot * QSTAGE;
      const int k0 = ch * QKC;
      if (VEC) {
        // N % 4 == 0: every row chunk starts 16-byte aligned and the atom tail is a
        // whole number of float4 (3 (N - k0) floats, a multiple of 12)
#pragma unroll
        for (int u = 0; u < QVPT; ++u) {
          const int e = tid + u * QNT;
          const int row = e / QV4, c4 = e - row * QV4;
          const bool isf = row < QF;
          const int s = isf ? s_raw[row] : l0 + row - QF;
          const bool ok = ch < nch && (isf ? s >= 0 : s < L) && 3 * k0 + 4 * c4 + 4 <= 3 * n;
          const float* src = (isf ? fr : lr) + (ok ? ((int64_t)s * n + k0) * 3 + 4 * c4 : 0);
          cpa16(dst + row * QRS + 4 * c4, src, ok);
        }
      } else {
#pragma unroll 4
        for (int u = 0; u < QLPT; ++u) {
          const int e = tid + u * QNT;  // [0, 64 * 3 QKC)
          const int row = e / (3 * QKC), r = e - row * (3 * QKC);
          const bool isf = row < QF;
          const int s = isf ? s_raw[row] : l0 + row - QF;
          const bool ok = ch < nch && (isf ? s >= 0 : s < L) && k0 + r / 3 < n;
          const float* src = (isf ? fr : lr) + (ok ? ((int64_t)s * n + k0) * 3 + r : 0);
          cpa4(dst + row * QRS + r, src, ok);
        }
      }
      if (tid < QKC) {
        const bool ok = ch < nch && k0 + tid < n;
        cpa8(sW + slot * QKC + tid, w + (ok ? k0 + tid : 0), ok);
      }
      mb_cp_arrive(&full[slot]);
    };
    double c[6][3][2];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) c[i][j][0] = c[i][j][1] = 0.0;
#pragma unroll
    for (int st = 0; st < QNST - 1; ++st)
      if (st < nch) issue(st, (int)((gch + st) % QNST));
    // per-thread fragment offsets inside a stage (loop invariant)
    int offA[6], offB[3];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const int mt = wm * 6 + i;
      offA[i] = ((mt & 3) * 8 + gq) * QRS + 3 * tq + (mt >> 2);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) offB[i] = (QF + wn * 8 + gq) * QRS + 3 * tq + i;
    for (int ch = 0; ch < nch; ++ch) {
      const uint32_t g = gch + (uint32_t)ch;
      const int slot = (int)(g % QNST);
      if (ch + QNST - 1 < nch) issue(ch + QNST - 1, (int)((g + QNST - 1) % QNST));
      mb_wait(&full[slot], (g / QNST) & 1u);
      const float* sg = ring + slot * QSTAGE;
      const double* ww = sW + slot * QKC + tq;
#pragma unroll
      for (int s = 0; s < (wact ? QKC / 4 : 0); ++s) {
        const double wj = RAW ? 1.0 : ww[4 * s];
        double a[6], b[3];
#pragma unroll
        for (int i = 0; i < 6; ++i)
          a[i] = (UNC || RAW) ? (double)sg[offA[i] + 12 * s] : (double)sg[offA[i] + 12 * s] - fcA[i];
#pragma unroll
        for (int i = 0; i < 3; ++i)
          b[i] = RAW ? (double)sg[offB[i] + 12 * s] : wj * ((double)sg[offB[i] + 12 * s] - lcB[i]);
#pragma unroll
        for (int i = 0; i < 6; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) dmma884(c[i][j], a[i], b[j]);
      }
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[slot]);
    }
    gch += (uint32_t)nch;
    __syncthreads();  // every stage consumed: the accumulator staging below overlays the ring
    // stage accumulators: row (b, f) = mt * 8 + gq, column (g, l) = g QL + 8 wn + 2 tq + e
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int row = (wm * 6 + i) * 8 + gq, col = j * QL + wn * 8 + 2 * tq;
        sC[row * QCS + col] = c[i][j][0];
        sC[row * QCS + col + 1] = c[i][j][1];
      }
    __syncthreads();
    // fused fit of the in-window pairs (exact fp64)
    for (int p = tid; p < QF * QL; p += QNT) {
      const int f = p / QL, li = p - f * QL;
      const int t = s_t[f];
      const int l = l0 + li;
      if (t < 0 || l >= L) continue;
      const int slot = l - s_lo[f];
      if (slot < 0 || slot >= s_cnt[f]) continue;
      double S[9];
#pragma unroll
      for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int g = 0; g < 3; ++g) {
          S[b * 3 + g] = sC[(b * QF + f) * QCS + g * QL + li];
          if (RAW) {
            const double cxb = s_fc[f][b], clg = lc[3 * l + g];
            S[b * 3 + g] = wuni * S[b * 3 + g] - fwbar[3 * t + b] * clg - cxb * lwbar[3 * l + g] -
                           wuni * n * cxb * clg;
          } else if (UNC) {
            S[b * 3 + g] -= s_fc[f][b] * lwbar[3 * l + g];
          }
        }
      if (Sout) {  // covariance output only (dense; the close-structure path fits a subset later)
        double* o = Sout + ((int64_t)t * L + l) * 9;
#pragma unroll
        for (int e = 0; e < 9; ++e) o[e] = S[e];
        continue;
      }
      double q[4];
      bool ill = false;
      double msd = fit_fast(S, gx[t], ga[l], Rex ? q : nullptr, &ill);
      uint8_t fl = 0;
      if (ill) {
        double k4[4][4], V[4][4], ev[4];
        kearsley_from_S(S, gx[t], ga[l], k4);
        if (!jacobi4(k4, ev, V)) fl |= kFlagNoConverge;
        msd = ev[0];
        q[0] = V[0][0]; q[1] = V[1][0]; q[2] = V[2][0]; q[3] = V[3][0];
      }
      if (Dex) Dex[(int64_t)t * cap + slot] = msd;
      if (Dd) Dd[(int64_t)t * ldd + l] = (float)msd;
      if (Rex) {
        double r[9];
        quat_to_rot(q, r);
        double* o = Rex + ((int64_t)t * cap + slot) * 9;
#pragma unroll
        for (int e = 0; e < 9; ++e) o[e] = r[e];
      }
      if (fl && flags) flags[t] |= fl;
    }
    __syncthreads();  // sC overlays the ring of the next sub-tile
  }
}

cudaError_t launch_refine_dmma(const float* fr, const double* fc, const float* lr, const double* lc,
                               const double* lwbar, const double* w, const double* gx, const int* fmap,
                               const double* fwbar, double wuni, const double* ga, int T, int L, int n,
                               const int* perm, const int* lo, const int* cnt, int cap, double* Dex, double* Rex,
                               float* Dd, int64_t ldd, uint8_t* flags, cudaStream_t stream, double* Sout) {
  if (T <= 0 || L <= 0) return cudaSuccess;
  static bool attr = false;
  if (!attr) {
    for (const void* fn : {(const void*)refine_dmma_kernel<true, true>, (const void*)refine_dmma_kernel<false, true>,
                           (const void*)refine_dmma_kernel<true, false>, (const void*)refine_dmma_kernel<false, false>,
                           (const void*)refine_dmma_kernel<true, false, true>,
                           (const void*)refine_dmma_kernel<false, false, true>}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, QSMEM);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  const bool vec = n % 4 == 0 && (reinterpret_cast<uintptr_t>(fr) & 15) == 0 && (reinterpret_cast<uintptr_t>(lr) & 15) == 0;
  // x: sub-tile slots per group (typical window unions span 3-4 sub-tiles; wider
  // unions loop), y: frame groups (launch order keeps a group's sub-tiles adjacent)
  const int ngroups = (T + QF - 1) / QF;
  const int lsub = (L + QL - 1) / QL;
#define MC_RD_LAUNCH(V, U, R)                                                                                  \
  do {                                                                                                         \
  for (int g0 = 0; g0 < ngroups; g0 += 65535) {                                                                \
    const dim3 grid((unsigned)std::min(lo ? 4 : 8, lsub), (unsigned)std::min(65535, ngroups - g0));           \
    refine_dmma_kernel<V, U, R><<<grid, QNT, QSMEM, stream>>>(fr, fc, lr, lc, lwbar, w, gx, fmap, fwbar, wuni, ga, \
                                                              T, L, n, perm, lo, cnt, cap, Dex, Rex, Dd, ldd,   \
                                                              flags, g0, Sout);                                 \
  }                                                                                                            \
  } while (0)
  if (lwbar && fwbar && wuni > 0.0) {
    if (vec) MC_RD_LAUNCH(true, false, true); else MC_RD_LAUNCH(false, false, true);
  } else if (lwbar) {
    if (vec) MC_RD_LAUNCH(true, true, false); else MC_RD_LAUNCH(false, true, false);
  } else {
    if (vec) MC_RD_LAUNCH(true, false, false); else MC_RD_LAUNCH(false, false, false);
  }
#undef MC_RD_LAUNCH
  return cudaGetLastError();
}

}  // namespace mc
