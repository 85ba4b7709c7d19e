// K4 gradient contraction on the 5th-gen tensor cores, exact to ~2^-31 through
// int8 slices (Ozaki scheme): tcgen05.mma.kind::i8, int32 accumulation in TMEM.
//
// Same result as cv_grad_dmma_kernel (grad_dmma.cu):
//   ds_t,k = 2 w_k (sum_i cs_i xc_k - U^s_k) - w'_k corr^s_t,
//   U^s_k  = sum_{i in sig(t)} (cs_i Rhat_i) ac_{i,k}      (same for z),
// with U as a GEMM  C[r, k] = sum_kk A[r, kk] B[kk, k]:
//   r  = (frame f, s|z, axis b): 48 rows for a group of 8 frames (FORCE: r =
//        (frame f, axis b), 16 frames, coefficients -(V_s cs + V_z cz) of the
//        metadynamics bias force, SPEC bias_and_force / Eq. 1),
//   kk = (landmark l - wlo, axis g) over the group's significant union,
//   B  = CENTRED landmark coordinates ac (fp64 from the raw fp32 rows), k = atom.
// Both operands are split into 4 signed int8 digits with a power-of-two scale
// per A row (over kk) and per B column (per atom, over every landmark):
//   v = 2^e 2^-31 (d0 2^24 + d1 2^16 + d2 2^8 + d3),  d in [-128, 127],
// so sum_kk A B = 2^(eA + eB - 14) sum_{p,q} 2^(-8(p+q)) (D_p . D_q) and every
// digit product is an exact integer summed exactly in int32 (K <= 256 here).
// Levels p + q <= 3 are kept (10 of the 16 products; the dropped ones weigh
// <= 2^-32 of the leading term), combined in fp64 in the epilogue:
//   v = acc0 + fl32(acc1 2^-8 + acc2 2^-16 + acc3 2^-24).
// The B digits are prepared once per landmark set (ldig kernels below); the A
// digits per frame group in shared memory by two "prep" warps while the
// tensor cores work on the previous group.
//
// MMA shape: M = 128 atoms (TMEM lanes), K = 32 (one int8 k-step), and the A
// digits stacked along N: for B digit q one MMA with N = (4 - q) 48 reading
// A digits 0..3-q and accumulating into the TMEM columns of levels q..3, so a
// k-step is 4 MMAs (N = 192, 144, 96, 48) that cover exactly the 10 kept
// products.  Accumulators: 4 levels x 48 columns, double-buffered (384 of 512
// TMEM columns), so the epilogue of one atom tile overlaps the next tile's MMAs.
//
// Warp roles (384 threads, persistent over frame groups):
//   warp 0: TMA producer (B digits: 4 boxes of 128 atoms x 64 B per stage,
//           SWIZZLE_64B; frame rows of the epilogue: 1-D bulk copies)
//   warp 1: MMA issuer (one lane)         warps 2-3: A-digit prep + TMEM alloc
//   warps 4-11: epilogue (TMEM lane quarter = warp % 4, two row halves)
// Groups wider than WMAX landmarks (or with n % 4 != 0) are left to the DMMA
// kernel (launch_cv_grad_dmma with min_width).
#include <cstdio>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "launch.h"
#include "mc_math.cuh"

namespace mc {



namespace gi8 {
constexpr int R = 48;                    // GEMM rows per frame group
constexpr int NDIG = 4;                  // int8 digits per operand
constexpr int BMA = 128;                 // atoms per tile (TMEM lanes)
constexpr int SLAB = 64;                 // K bytes per pipeline stage (2 k-steps), SWIZZLE_64B rows
constexpr int KMAX = 256;                // K bytes of one group (its landmark union x 3)
// widest union handled here: 3 WMAX + 15 <= KMAX (the TMA K start 3 wlo is rounded down to 16 bytes:
// an unaligned inner box coordinate of a UINT8 map faults, tools/_diag/tma_u8_probe.cu)
constexpr int WMAX = (KMAX - 15) / 3;    // 80 landmarks
constexpr int NSLAB = KMAX / SLAB;       // 4
constexpr int L_STAGE = NDIG * BMA * SLAB;  // 32 KB
constexpr int L_DIG = BMA * SLAB;           // 8 KB per digit box
constexpr int C_SLAB = NDIG * R * SLAB;     // 12 KB: 192 A rows x 64 B
constexpr int C_BUF = NSLAB * C_SLAB;       // 48 KB
constexpr int EPI = 8;
constexpr int NT = 32 * (4 + EPI);
constexpr int ACC = NDIG * R;  // TMEM columns per accumulator buffer
constexpr int FVEC = 16;

template <int NCV>
struct Cfg;  // frames per group, B-digit pipeline stages, frame-row buffer bytes
template <>
struct Cfg<2> {
  static constexpr int DG = 8;
  static constexpr int STAGES = 3;
  static constexpr int X_BUF = DG * BMA * 12;
};
template <>
struct Cfg<1> {
  static constexpr int DG = 16;
  static constexpr int STAGES = 2;
  static constexpr int X_BUF = DG * BMA * 12;
};

template <int DG>
struct GHdr {
  int t[DG], raw[DG], ns[DG], flo[DG], fhi[DG];
  int cum[DG + 1];
  int wlo, koff, k0, nks, nslab, active;  // koff = 3 wlo - k0 in [0, 16)
  double cx[DG][3];
  double fv[DG][8];
  double dv[DG][2];
  double scp[R];  // sc_r 2^-eA_r
  double qs[R];   // 2^(31 - eA_r): quantisation scale
  float P[R];     // 2^eA_r
  float corr[R];
  unsigned long long rmax[R];
};

template <int NCV>
constexpr int smem_bytes() {
  return Cfg<NCV>::STAGES * L_STAGE + 2 * C_BUF + 2 * Cfg<NCV>::X_BUF + 2 * (int)sizeof(GHdr<Cfg<NCV>::DG>) +
         16 * 8 + 1024;
}

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
// K-major SWIZZLE_64B operand (64 B rows, 8-row groups 512 B apart), layout 4
__device__ __forceinline__ uint64_t desc64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}
// instruction descriptor: D = S32 (2), A = B = signed 8 bit (1), K-major, N >> 3, M >> 4
__host__ __device__ constexpr uint32_t idesc_i8(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BMA >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(reinterpret_cast<uint64_t>(bar))
               : "memory");
}
__device__ __forceinline__ void tld8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void prep_bar() { asm volatile("bar.sync 1, 64;" ::: "memory"); }

// byte offset of (row, kk) in a K-major SWIZZLE_64B operand made of 64-byte-K slabs
// of `rows` rows each (the pattern TMA writes: 16-byte chunk ^= (row % 8) >> 1)
__device__ __forceinline__ int swz64(int row, int kk, int slab_bytes) {
  return (kk >> 6) * slab_bytes + (row >> 3) * 512 + (row & 7) * 64 + (((((kk & 63) >> 4) ^ ((row & 7) >> 1)) & 3) << 4) +
         (kk & 15);
}

// power-of-two scale of a row / column with max |v| = mx: 2^e with mx 2^(7 - e) <= 127,
// so every value's 31-bit integer X = rint(v 2^(31 - e)) has |X| <= 127 2^24 + 1/2 and its
// balanced base-256 digits (d3, d2, d1 in [-128, 127], d0 = the rest) keep |d0| <= 127
__device__ __forceinline__ int digit_exp(double mx) {
  if (!(mx > 0.0) || !isfinite(mx)) return 0;
  int e;
  frexp(mx, &e);  // mx < 2^e
  if (ldexp(mx, 7 - e) > 127.0) ++e;
  return e;
}
__device__ __forceinline__ void digits4(double v, double qs, int8_t* d) {
  int X = __double2int_rn(v * qs);
#pragma unroll
  for (int p = 3; p > 0; --p) {
    const int lo = ((X + 128) & 255) - 128;
    d[p] = (int8_t)lo;
    X = (X - lo) >> 8;
  }
  d[0] = (int8_t)X;
}
}  // namespace gi8

// B digits of a landmark set: per-atom exponent eB[k] over every (landmark, axis)
// of the centred coordinates ac = lraw - lcen (fp64), then 4 digit planes
// dig[q][npad][kpad] (row = atom, K = (landmark, axis), zero padded).
__global__ void ldig_scale_kernel(const float* __restrict__ lraw, const double* __restrict__ lcen, int L, int n,
                                  int* __restrict__ eB) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= n) return;
  double mx = 0.0;
  for (int l = 0; l < L; ++l) {
    const float* p = lraw + ((int64_t)l * n + k) * 3;
#pragma unroll
    for (int g = 0; g < 3; ++g) mx = fmax(mx, fabs((double)p[g] - lcen[3 * l + g]));
  }
  eB[k] = gi8::digit_exp(mx);
}

// tile of 32 atoms x 64 landmarks: coalesced reads through shared memory, then one
// thread per (digit, atom) writes its 192-byte run of the row with 16-byte stores
__global__ void __launch_bounds__(256) ldig_kernel(const float* __restrict__ lraw, const double* __restrict__ lcen,
                                                   int L, int n, int npad, int kpad, const int* __restrict__ eB,
                                                   int8_t* __restrict__ dig) {
  __shared__ float sx[64][32 * 3 + 1];
  const int k0 = blockIdx.x * 32, l0 = blockIdx.y * 64;
  for (int e = threadIdx.x; e < 64 * 96; e += 256) {
    const int l = e / 96, r = e % 96;
    const int k = k0 + r / 3;
    sx[l][r] = (l0 + l < L && k < n) ? lraw[((int64_t)(l0 + l) * n + k0) * 3 + r] : 0.0f;
  }
  __syncthreads();
  if (threadIdx.x >= 128) return;
  const int q = threadIdx.x >> 5, kl = threadIdx.x & 31, k = k0 + kl;
  if (k >= n) return;
  const double qs = ldexp(1.0, 31 - eB[k]);
  const int nl = min(64, L - l0);
  int8_t* row = dig + ((int64_t)q * npad + k) * kpad + 3 * l0;
  alignas(16) int8_t buf[192];
  for (int l = 0; l < 64; ++l)
#pragma unroll
    for (int g = 0; g < 3; ++g) {
      int8_t d[4] = {0, 0, 0, 0};
      if (l < nl) gi8::digits4((double)sx[l][3 * kl + g] - lcen[3 * (l0 + l) + g], qs, d);
      buf[3 * l + g] = d[q];
    }
  if (nl == 64 && (kpad % 16) == 0) {
    for (int c = 0; c < 12; ++c) reinterpret_cast<int4*>(row)[c] = reinterpret_cast<const int4*>(buf)[c];
  } else {
    for (int c = 0; c < 3 * nl; ++c) row[c] = buf[c];
  }
}

template <typename OT, int NCV>
__global__ void __launch_bounds__(gi8::NT, 1)
cv_grad_i8_kernel(const __grid_constant__ CUtensorMap mapB, int T, int n, int npad, int cap,
                  const float* __restrict__ fraw, const double* __restrict__ fcen, const double* __restrict__ w,
                  const double* __restrict__ wa, const int* __restrict__ eB, const int* __restrict__ sig_idx,
                  const double* __restrict__ sig_coef, const int* __restrict__ nsig, const double* __restrict__ fvec,
                  const double* __restrict__ dV, const int* __restrict__ perm, const int* __restrict__ out_map,
                  OT* __restrict__ out0, OT* __restrict__ out1, int* __restrict__ wide_flag, int dbg) {
  using namespace gi8;
  constexpr int DG = Cfg<NCV>::DG;
  constexpr int STAGES = Cfg<NCV>::STAGES;
  constexpr int X_BUF = Cfg<NCV>::X_BUF;
  constexpr int EPR = 9 * NCV;  // coefficient entries per (frame, significant landmark)
  using Hdr = GHdr<DG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sL = sm;
  uint8_t* sC = sL + STAGES * L_STAGE;
  uint8_t* sX = sC + 2 * C_BUF;
  Hdr* hdr = reinterpret_cast<Hdr*>(sX + 2 * X_BUF);
  uint64_t* lfull = reinterpret_cast<uint64_t*>(hdr + 2);
  uint64_t* lempty = lfull + STAGES;
  uint64_t* cfull = lempty + STAGES;   // [2]
  uint64_t* cempty = cfull + 2;        // [2]
  uint64_t* tfull = cempty + 2;        // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint64_t* xfull = tempty + 2;        // [2]
  uint64_t* xempty = xfull + 2;        // [2]
  __shared__ uint32_t tmem_slot;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int groups = (T + DG - 1) / DG;
  const int ntile = (n + BMA - 1) / BMA;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
    for (int s = 0; s < STAGES; ++s) { mb_init(&lfull[s], 1); mb_init(&lempty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      mb_init(&cfull[b], 1);
      mb_init(&cempty[b], 1 + 1 + EPI);  // MMA commit + producer + epilogue warps
      mb_init(&tfull[b], 1);
      mb_init(&tempty[b], EPI);
      mb_init(&xfull[b], 1);
      mb_init(&xempty[b], EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_slot;

  if (warp == 2 || warp == 3) {
    // ------------------------------------------------------------ A-digit prep
    const int pt = tid - 64;
    int i = 0;
    for (int g = blockIdx.x; g < groups; g += gridDim.x, ++i) {
      const int cb = i & 1;
      Hdr& h = hdr[cb];
      uint8_t* C = sC + cb * C_BUF;
      mb_wait(&cempty[cb], ((i >> 1) & 1) ^ 1);
      if (pt < DG) {
        const int k = g * DG + pt;
        int t = -1, ns = 0;
        if (k < T) {
          t = perm ? perm[k] : k;
          ns = nsig[t];
        }
        h.t[pt] = t;
        h.raw[pt] = t < 0 ? -1 : (out_map ? out_map[t] : t);
        h.ns[pt] = t < 0 ? 0 : ns;
        h.flo[pt] = (t >= 0 && ns > 0) ? sig_idx[(int64_t)t * cap] : 0x7fffffff;
        h.fhi[pt] = (t >= 0 && ns > 0) ? sig_idx[(int64_t)t * cap + ns - 1] + 1 : -1;
        for (int a = 0; a < 3; ++a) h.cx[pt][a] = t < 0 ? 0.0 : fcen[3 * t + a];
        for (int e = 0; e < 8; ++e) h.fv[pt][e] = t < 0 ? 0.0 : fvec[(int64_t)t * FVEC + e];
        if (NCV == 1) {
          h.dv[pt][0] = t < 0 ? 0.0 : dV[2 * t];
          h.dv[pt][1] = t < 0 ? 0.0 : dV[2 * t + 1];
        }
      }
      prep_bar();
      if (pt == 0) {
        int a = 0x7fffffff, b = -1, tot = 0;
        for (int f = 0; f < DG; ++f) {
          a = min(a, h.flo[f]);
          b = max(b, h.fhi[f]);
          h.cum[f] = tot;
          tot += h.ns[f] * EPR;
        }
        h.cum[DG] = tot;
        const int width = b - a;
        h.active = (b >= 0 && width <= WMAX) ? 1 : 0;
        if (b >= 0 && width > WMAX && wide_flag) *wide_flag = 1;  // left to the DMMA kernel / caller
        h.wlo = a;
        h.koff = b >= 0 ? (3 * a) & 15 : 0;
        h.k0 = b >= 0 ? 3 * a - h.koff : 0;
        h.nks = b >= 0 ? (3 * width + h.koff + 31) / 32 : 0;
        h.nslab = (h.nks + 1) / 2;
        if ((dbg & 32) && g < 3)
          printf("prep blk %d g %d active %d wlo %d whi %d nks %d tot %d t0 %d raw0 %d ns0 %d\n", blockIdx.x, g,
                 h.active, a, b, h.nks, tot, h.t[0], h.raw[0], h.ns[0]);
      }
      prep_bar();
      if (!h.active) {
        if (pt == 0) mb_arrive(&cfull[cb]);
        continue;
      }
      const int nslab = h.nslab, wlo = h.wlo, koff = h.koff, tot = h.cum[DG];
      // zero the group's slabs and the row maxima
      for (int e = pt; e < nslab * C_SLAB / 16; e += 64) reinterpret_cast<int4*>(C)[e] = make_int4(0, 0, 0, 0);
      if (pt < R) h.rmax[pt] = 0ull;
      prep_bar();
      // coefficient of entry e: frame f, significant slot s, component j (row, axis g)
      auto entry = [&](int e, int& f, int& row, int& kk) -> double {
        f = 0;
#pragma unroll
        for (int q = 1; q < DG; ++q) f += e >= h.cum[q];
        const int el = e - h.cum[f];
        const int s = el / EPR, j = el % EPR;
        const int t = h.t[f];
        const int64_t base = (int64_t)t * cap + s;
        const int l = sig_idx[base];
        double v;
        if (NCV == 2) {
          v = sig_coef[base * 18 + j];
          row = f * 6 + (j / 9) * 3 + (j % 9) / 3;
        } else {
          v = -(h.dv[f][0] * sig_coef[base * 18 + j] + h.dv[f][1] * sig_coef[base * 18 + 9 + j]);
          row = f * 3 + j / 3;
        }
        kk = 3 * (l - wlo) + j % 3 + koff;
        return v;
      };
      for (int e = pt; e < tot; e += 64) {
        int f, row, kk;
        const double v = entry(e, f, row, kk);
        atomicMax(&h.rmax[row], (unsigned long long)__double_as_longlong(fabs(v)));
      }
      prep_bar();
      if (pt < R) {
        const int f = NCV == 2 ? pt / 6 : pt / 3;
        const int cv = NCV == 2 ? (pt % 6) / 3 : 0;
        const int b = pt % 3;
        const int e = digit_exp(__longlong_as_double((long long)h.rmax[pt]));
        double sc, corr;
        if (NCV == 2) {
          sc = h.fv[f][cv];
          corr = h.fv[f][2 + cv * 3 + b];
        } else {
          sc = -(h.dv[f][0] * h.fv[f][0] + h.dv[f][1] * h.fv[f][1]);
          corr = -(h.dv[f][0] * h.fv[f][2 + b] + h.dv[f][1] * h.fv[f][5 + b]);
        }
        h.scp[pt] = ldexp(sc, -e);
        h.qs[pt] = ldexp(1.0, 31 - e);
        h.P[pt] = ldexpf(1.0f, e);
        h.corr[pt] = (float)corr;
      }
      prep_bar();
      for (int e = pt; e < tot; e += 64) {
        int f, row, kk;
        const double v = entry(e, f, row, kk);
        int8_t d[4];
        digits4(v, h.qs[row], d);
#pragma unroll
        for (int p = 0; p < NDIG; ++p) C[swz64(p * R + row, kk, C_SLAB)] = (uint8_t)d[p];
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      prep_bar();
      if (pt == 0) mb_arrive(&cfull[cb]);
    }
  } else if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int i = 0;
      uint32_t it = 0, st = 0;
      for (int g = blockIdx.x; g < groups; g += gridDim.x, ++i) {
        const int cb = i & 1;
        const Hdr& h = hdr[cb];
        mb_wait(&cfull[cb], (i >> 1) & 1);
        if (h.active) {
          const int nslab = h.nslab, k0 = h.k0;
          int rows = 0;
          for (int f = 0; f < DG; ++f) rows += h.raw[f] >= 0;
          for (int tl = 0; tl < ntile; ++tl, ++it) {
            const int a0 = tl * BMA, nat = min(BMA, n - a0);
            const int xb = it & 1;
            mb_wait(&xempty[xb], ((it >> 1) & 1) ^ 1);
            uint8_t* X = sX + xb * X_BUF;
            if (dbg & 8) {
              mb_arrive(&xfull[xb]);
            } else {
              mb_expect(&xfull[xb], (uint32_t)(rows * 12 * nat));
              for (int f = 0; f < DG; ++f)
                if (h.raw[f] >= 0)
                  bulk_g2s(X + f * BMA * 12, fraw + ((int64_t)h.raw[f] * n + a0) * 3, (uint32_t)(12 * nat), &xfull[xb]);
            }
            for (int j = 0; j < nslab; ++j, ++st) {
              const int s = st % STAGES;
              mb_wait(&lempty[s], ((st / STAGES) & 1) ^ 1);
              uint8_t* dst = sL + s * L_STAGE;
              if (dbg & 4) {
                mb_arrive(&lfull[s]);
              } else {
                mb_expect(&lfull[s], (uint32_t)L_STAGE);
#pragma unroll
                for (int q = 0; q < NDIG; ++q) tma2d(&mapB, &lfull[s], dst + q * L_DIG, k0 + SLAB * j, q * npad + a0);
              }
            }
          }
        }
        mb_arrive(&cempty[cb]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    int i = 0;
    uint32_t it = 0, st = 0;
    constexpr uint32_t ID0 = idesc_i8(4 * R), ID1 = idesc_i8(3 * R), ID2 = idesc_i8(2 * R), ID3 = idesc_i8(R);
    for (int g = blockIdx.x; g < groups; g += gridDim.x, ++i) {
      const int cb = i & 1;
      const Hdr& h = hdr[cb];
      mb_wait(&cfull[cb], (i >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (!h.active) {
        if (lane == 0) mb_arrive(&cempty[cb]);
        __syncwarp();
        continue;
      }
      const int nslab = h.nslab, nks = h.nks;
      const uint32_t cbase = su32(sC + cb * C_BUF);
      for (int tl = 0; tl < ntile; ++tl, ++it) {
        const int ab = it & 1;
        mb_wait(&tempty[ab], ((it >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + (uint32_t)(ab * ACC);
        for (int j = 0; j < nslab; ++j, ++st) {
          const int s = st % STAGES;
          mb_wait(&lfull[s], (st / STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (lane == 0) {
            const uint32_t lb = su32(sL + s * L_STAGE);
            const uint32_t cs = cbase + (uint32_t)(j * C_SLAB);
#pragma unroll
            for (int kk = 0; kk < 2; ++kk) {
              if (2 * j + kk < nks && !(dbg & 1)) {
                const uint64_t bdesc = desc64(cs + 32 * kk);
                const uint32_t first = (j | kk) == 0 ? 0u : 1u;
                mma_i8(d, desc64(lb + 0 * L_DIG + 32 * kk), bdesc, ID0, first);
                mma_i8(d + R, desc64(lb + 1 * L_DIG + 32 * kk), bdesc, ID1, 1u);
                mma_i8(d + 2 * R, desc64(lb + 2 * L_DIG + 32 * kk), bdesc, ID2, 1u);
                mma_i8(d + 3 * R, desc64(lb + 3 * L_DIG + 32 * kk), bdesc, ID3, 1u);
              }
            }
            mma_commit(&lempty[s]);
            if (j == nslab - 1) mma_commit(&tfull[ab]);
          }
          __syncwarp();
        }
      }
      if (lane == 0) mma_commit(&cempty[cb]);
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int qd = warp & 3, half = (warp - 4) >> 2;
    constexpr int HR = R / 2;                 // 24 rows per half
    constexpr int FPH = DG / 2;               // frames per half
    constexpr int RPF = 3 * NCV;              // rows per frame
    int i = 0;
    uint32_t it = 0;
    for (int g = blockIdx.x; g < groups; g += gridDim.x, ++i) {
      const int cb = i & 1;
      const Hdr& h = hdr[cb];
      mb_wait(&cfull[cb], (i >> 1) & 1);
      if (h.active) {
        for (int tl = 0; tl < ntile; ++tl, ++it) {
          const int ab = it & 1;
          const int a0 = tl * BMA;
          const int al = qd * 32 + lane;
          const int a = a0 + al;
          const bool valid = a < n;
          // per-atom constants (the B column scale 2^eB and the weights)
          const int eb = valid ? eB[a] : 0;
          const double sxa = ldexp(1.0, 14 - eb);
          const double wk = valid ? w[a] : 0.0;
          const double wak = valid ? wa[a] : 0.0;
          mb_wait(&tfull[ab], (it >> 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          __syncwarp();  // tcgen05.ld is .sync.aligned: the whole warp, converged
          uint32_t acc[NDIG][HR];
          const uint32_t tb = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(ab * ACC + half * HR);
          if (!(dbg & 2)) {
#pragma unroll
            for (int l = 0; l < NDIG; ++l)
#pragma unroll
              for (int c = 0; c < HR / 8; ++c) tld8(tb + l * R + c * 8, &acc[l][c * 8]);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          } else {
#pragma unroll
            for (int l = 0; l < NDIG; ++l)
#pragma unroll
              for (int c = 0; c < HR; ++c) acc[l][c] = 0;
          }
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mb_arrive(&tempty[ab]);
          mb_wait(&xfull[ab], (it >> 1) & 1);
          if ((dbg & 32) && lane == 0 && warp == 4 && g < 3)
            printf("epi blk %d g %d tile %d acc0 %d %d P %g scp %g raw %d\n", blockIdx.x, g, tl, (int)acc[0][0],
                   (int)acc[1][0], h.P[0], h.scp[0], h.raw[0]);
          const float* X = reinterpret_cast<const float*>(sX + ab * X_BUF);
#pragma unroll
          for (int fl = 0; fl < FPH; ++fl) {
            const int f = half * FPH + fl;
            const int raw = h.raw[f];
            if (raw < 0) continue;  // warp-uniform
            double xc[3];
#pragma unroll
            for (int b = 0; b < 3; ++b) xc[b] = ((double)X[(f * BMA + al) * 3 + b] - h.cx[f][b]) * sxa;
#pragma unroll
            for (int cv = 0; cv < NCV; ++cv) {
              OT* dst = (cv ? out1 : out0) + ((int64_t)raw * n + a) * 3;
#pragma unroll
              for (int b = 0; b < 3; ++b) {
                const int rl = fl * RPF + cv * 3 + b;
                const int r = half * HR + rl;
                const float lo = fmaf((float)(int)acc[3][rl], 5.9604644775390625e-8f,
                                      fmaf((float)(int)acc[2][rl], 1.52587890625e-5f,
                                           (float)(int)acc[1][rl] * 3.90625e-3f));
                const double v = (double)(int)acc[0][rl] + (double)lo;
                // t = sc' xc' - v in units of 2^(eA_r + eB_k - 14)
                const double tt = fma(h.scp[r], xc[b], -v);
                const double scale = (double)h.P[r] * ldexp(2.0 * wk, eb - 14);
                if (valid) dst[b] = (OT)(tt * scale - wak * (double)h.corr[r]);
              }
            }
          }
          __syncwarp();
          if (lane == 0) mb_arrive(&xempty[ab]);
        }
      }
      __syncwarp();
      if (lane == 0) mb_arrive(&cempty[cb]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encode_i8() {
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

cudaError_t launch_ldig(const float* lraw, const double* lcen, int L, int n, int npad, int kpad, int* eB,
                        int8_t* dig, cudaStream_t stream) {
  if (L <= 0 || n <= 0) return cudaSuccess;
  if (npad < n || kpad < 3 * L || kpad % 16) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(dig, 0, (size_t)gi8::NDIG * npad * kpad, stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(eB, 0, (size_t)npad * sizeof(int), stream);
  if (e != cudaSuccess) return e;
  ldig_scale_kernel<<<(n + 127) / 128, 128, 0, stream>>>(lraw, lcen, L, n, eB);
  dim3 grid((n + 31) / 32, (L + 63) / 64);
  ldig_kernel<<<grid, 256, 0, stream>>>(lraw, lcen, L, n, npad, kpad, eB, dig);
  return cudaGetLastError();
}

// ncv = 2: ds (out0), dz (out1); ncv = 1: fused bias force F (out0) with dV [T, 2]
cudaError_t launch_cv_grad_i8(int T, int n, int cap, const float* fraw, const double* fcen, const float* lraw,
                              const double* lcen, const double* w, const double* wa, const int8_t* dig, const int* eB,
                              int npad, int kpad, const int* sig_idx, const double* sig_coef, const int* nsig,
                              const double* fvec, const double* dV, const int* perm, const int* out_map, void* out0,
                              void* out1, int out_f32, int ncv, int* wide_flag, cudaStream_t stream) {
  using namespace gi8;
  if (T <= 0 || n <= 0) return cudaSuccess;
  if (ncv != 1 && ncv != 2) return cudaErrorInvalidValue;
  const bool ok_i8 = n % 4 == 0 && (reinterpret_cast<uintptr_t>(fraw) & 15) == 0 && kpad % 16 == 0 && npad % BMA == 0;
  if (!ok_i8) {
    if (ncv != 2) return cudaErrorInvalidValue;  // the force path needs the tensor-core kernel
    return launch_cv_grad_dmma(T, n, cap, fraw, fcen, lraw, lcen, w, wa, sig_idx, sig_coef, nsig, fvec, perm, out_map,
                               out0, out1, out_f32, stream, -1);
  }
  auto enc = get_encode_i8();
  if (!enc) return cudaErrorInvalidValue;
  CUtensorMap map;
  cuuint64_t dims[2] = {(cuuint64_t)kpad, (cuuint64_t)NDIG * npad};
  cuuint64_t strides[1] = {(cuuint64_t)kpad};
  cuuint32_t box[2] = {(cuuint32_t)SLAB, (cuuint32_t)BMA};
  cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(dig), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int DG = ncv == 2 ? Cfg<2>::DG : Cfg<1>::DG;
  // diagnostic switches (MC_GI8_DBG bit mask; results invalid when set): 1 no MMAs,
  // 2 no TMEM loads, 4 no B-digit TMA, 8 no frame-row copies, 16 skip the DMMA fallback
  static const int dbg = [] {
    const char* e = getenv("MC_GI8_DBG");
    return e ? atoi(e) : 0;
  }();
  const int groups = (T + DG - 1) / DG;
  const int grid = groups < sms ? groups : sms;
#define MC_GI8(OTT, NC)                                                                                        \
  do {                                                                                                         \
    static bool attr = false;                                                                                  \
    if (!attr) {                                                                                               \
      cudaError_t e = cudaFuncSetAttribute(cv_grad_i8_kernel<OTT, NC>,                                         \
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<NC>());     \
      if (e != cudaSuccess) return e;                                                                          \
      attr = true;                                                                                             \
    }                                                                                                          \
    cv_grad_i8_kernel<OTT, NC><<<grid, NT, smem_bytes<NC>(), stream>>>(                                        \
        map, T, n, npad, cap, fraw, fcen, w, wa, eB, sig_idx, sig_coef, nsig, fvec, dV, perm, out_map,        \
        (OTT*)out0, (OTT*)out1, wide_flag, dbg);                                                                    \
  } while (0)
  if (ncv == 2) {
    if (out_f32) MC_GI8(float, 2); else MC_GI8(double, 2);
  } else {
    if (out_f32) MC_GI8(float, 1); else MC_GI8(double, 1);
  }
#undef MC_GI8
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || ncv != 2 || (dbg & 16)) return e;
  // groups wider than WMAX landmarks: the DMMA kernel (every other group returns at once)
  return launch_cv_grad_dmma(T, n, cap, fraw, fcen, lraw, lcen, w, wa, sig_idx, sig_coef, nsig, fvec, perm, out_map,
                             out0, out1, out_f32, stream, WMAX);
}

}  // namespace mc
