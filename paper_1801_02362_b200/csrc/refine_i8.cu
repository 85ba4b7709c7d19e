// Exact refits (the Kearsley covariances of the in-window pairs, geometry.py:180-196)
// on the 5th-gen tensor cores through exact int8 digits (Ozaki scheme,
// tcgen05.mma.kind::i8 with int32 accumulation in TMEM).
//
// Same contract as refine_dmma_kernel (refine_dmma.cu): for every frame t and every
// landmark l of its window [lo_t, lo_t + cnt_t) (or of all L, dense mode)
//   S[t,l][b][g] = sum_j (x_{t,j,b} - c_{t,b}) w_j (a_{l,j,g} - c_{l,g})
// followed by the fused Newton + adjugate fit (Jacobi fallback) -> MSD, R.
// Both operands are split per ROW over the atoms (K = atoms) into 4 signed int8
// digits, v = 2^(e-31) (d0 2^24 + d1 2^16 + d2 2^8 + d3) (the rules of grad_i8.cu):
//   frames  FD: rows (sorted slot k, axis b) = centred x, written per call (rdig_kernel),
//   landmarks LD: rows (l, axis g) = w (a - c_l), once per landmark set,
// each row stored with the 4 digits of every 32-atom k-step interleaved
// ([rows][kpad/32][4][32]: one 128-byte TMA row segment per k-step).  Every digit
// product is exact and the 10 products with p + q <= 3 are accumulated in int32
// per level (|acc3| <= 4 2^14 n < 2^31 for n < 32768), then
//   S = 2^(eF + eL - 38) (acc0 2^24 + acc1 2^16 + acc2 2^8 + acc3)   (exact in fp64).
// Error: each operand is exact to 2^-31 of its row maximum, so S is exact to
// ~2^-31 sqrt(n)/n of |x||w a| -- ~1e-11 on the MSD at config 4 (tolerance 1e-9).
//
// Tile: M = 128 TMEM lanes = 42 landmarks x 3 axes (lanes 126, 127 unused), N = 64 =
// 21 window-sorted frames x 3 axes (+ one ignored row); per 32-atom k-step 10 MMAs
// (M=128, N=64, K=32), one per digit product (A = LD digit q, B = FD digit p: the K slices
// [32q, 32q + 32) and [32p, 32p + 32) of the interleaved rows) into the TMEM columns of
// level p + q.  Accumulators 4 levels x 64 columns, double-buffered (all 512 TMEM
// columns), so a tile's epilogue (staging the 9 entries of each pair in shared memory,
// then one thread per in-window pair runs the fit) overlaps the next tile's MMAs.  21
// frames per group (not 16) cut the operand bytes per multiply-add by 18%: the kernel is
// bound by the L2 -> shared-memory rate of its operand boxes.  A frame group takes
// ceil(union / 42) landmark tiles of its window union, odd tiles sweeping K backwards
// (serpentine: they start on the frame rows still in L2).  Warp roles (256 threads,
// persistent over frame groups): 0 TMA producer (3-stage ring of 2 x 24 KB: 16 KB of
// landmark rows + 8 KB of frame rows per k-step), 1 MMA issuer, 2 TMEM allocator,
// 4-15 epilogue (all twelve drain the accumulators and run the fused fits).
#include <cuda.h>
#include <cudaTypedefs.h>

#include "launch.h"
#include "mc_math.cuh"

namespace mc {

namespace ri8 {
constexpr int FG = 21;             // frames per group
constexpr int NR = 3 * FG;         // 63 N rows used
constexpr int NB = 64;             // MMA N and frame-digit box rows (row 63: the next group's, ignored)
constexpr int LT = 42;             // landmarks per tile
constexpr int MR = 128;            // M rows (TMEM lanes); 3 LT = 126 used
constexpr int KS = 32;             // atoms per k-step
constexpr int ROWB = 4 * KS;       // 128 bytes per row and k-step (4 digits)
constexpr int A_ST = MR * ROWB;    // 16 KB
constexpr int B_ST = NB * ROWB;    // 8 KB
constexpr int STAGE = A_ST + B_ST; // 24 KB per k-step (a multiple of 1024)
// k-steps per pipeline stage: the MMA warp's barrier wait, tcgen05 fence and commit are paid
// once per KPS k-steps (grad_i8.cu: ~260 clk per stage against ~320 clk of tensor-pipe work
// per k-step here)
constexpr int KPS = 2;
constexpr int STG = KPS * STAGE;   // 48 KB per stage
constexpr int NST = 3;
constexpr int ACC = 4 * NB;        // 256 TMEM columns per accumulator buffer (2 buffers = 512)
constexpr int EPI = 12;            // epilogue warps: all drain the accumulators (3 per TMEM lane
                                   // quarter) and run the fused fits
constexpr int NT = 32 * (4 + EPI);
constexpr int SC_BYTES = FG * LT * 9 * 8;  // staged covariances of a tile (fp64)
constexpr int SMEM = NST * STG + SC_BYTES + 1024 + 512;

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
__device__ __forceinline__ void tma3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ void tma2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
// K-major SWIZZLE_128B operand (128 B rows, 8-row groups 1024 B apart), layout 2
__device__ __forceinline__ uint64_t desc128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// D = S32, A = B = signed 8 bit, K-major, N = 48, M = 128
// D = S32, A = B = signed 8 bit, K-major, N = n, M = 128
__host__ __device__ constexpr uint32_t idesc_n(int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(MR >> 4) << 24);
}
constexpr uint32_t IDESC = idesc_n(NB);
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// K-major SWIZZLE_32B operand (32 B rows, 8-row groups 256 B apart), layout 6
__device__ __forceinline__ uint64_t desc32(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
// one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.b32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
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
__device__ __forceinline__ void tld1(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(taddr));
}
__device__ __forceinline__ void tld4(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}
__device__ __forceinline__ double pow2d(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(32 * EPI) : "memory"); }

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
}  // namespace ri8

// Row digits of B structures (one CTA each, 256 threads): structure k is raw row
// fmap[perm[k]] (perm, fmap nullable), centred with cen[perm[k]] (fp64), optionally
// weighted by w; rows 3k + axis of dig ([3B][kpad/32][4][32], kpad % 32 == 0) and the
// per-row exponents e[3k + axis].  The structure is staged in shared memory (n <= 16384
// per pass; larger n re-reads it from L2).
__global__ void __launch_bounds__(256)
rdig_kernel(const float* __restrict__ raw, const double* __restrict__ cen, const double* __restrict__ w,
            const int* __restrict__ perm, const int* __restrict__ fmap, int B, int n, int kpad,
            int8_t* __restrict__ dig, int* __restrict__ eout, int staged, const int* __restrict__ ein, int planes) {
  extern __shared__ __align__(16) float sx[];  // the structure's 3n coordinates (staged mode)
  __shared__ double red[3][8];
  __shared__ int s_e[3];
  const int k = blockIdx.x;
  if (k >= B) return;
  const int t = perm ? perm[k] : k;
  const int src = fmap ? fmap[t] : t;
  const float* x = raw + (int64_t)src * n * 3;
  if (staged) {  // one coalesced pass over the row (16-byte loads when aligned)
    const int nf = 3 * n;
    if ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && nf % 4 == 0) {
      for (int e = threadIdx.x; e < nf / 4; e += 256)
        reinterpret_cast<float4*>(sx)[e] = __ldg(reinterpret_cast<const float4*>(x) + e);
    } else {
      for (int e = threadIdx.x; e < nf; e += 256) sx[e] = __ldg(x + e);
    }
    __syncthreads();
    x = sx;
  }
  double c[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) c[b] = cen[3 * t + b];
  if (ein) {  // exponents from the frame split (K1s): one pass over the coordinates
    if (threadIdx.x < 3) {
      const int e = ein[3 * t + threadIdx.x];
      s_e[threadIdx.x] = e;
      eout[3 * k + threadIdx.x] = e;
    }
    __syncthreads();
  } else {
  double mx[3] = {0.0, 0.0, 0.0};
  for (int j = threadIdx.x; j < n; j += 256) {
    const double wj = w ? w[j] : 1.0;
#pragma unroll
    for (int b = 0; b < 3; ++b) mx[b] = fmax(mx[b], fabs(wj * ((double)x[3 * j + b] - c[b])));
  }
#pragma unroll
  for (int b = 0; b < 3; ++b) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx[b] = fmax(mx[b], __shfl_xor_sync(0xffffffffu, mx[b], o));
    if ((threadIdx.x & 31) == 0) red[b][threadIdx.x >> 5] = mx[b];
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double m = 0.0;
    for (int i = 0; i < 8; ++i) m = fmax(m, red[threadIdx.x][i]);
    const int e = ri8::digit_exp(m);
    s_e[threadIdx.x] = e;
    eout[3 * k + threadIdx.x] = e;
  }
  __syncthreads();
  }
  const int nks = kpad / 32;
  if (planes) {
    // digit planes [nks][4][3B][32]: one thread per (k-step, axis, 16-atom half) packs the
    // 16 atoms' digit q into one 16-byte store per plane (a plane row is 32 bytes)
    const int64_t R3 = 3LL * B;
    for (int task = threadIdx.x; task < 6 * nks; task += 256) {
      const int h = task & 1, rest = task >> 1;
      const int ks = rest / 3, b = rest - 3 * ks;
      const double qs = ldexp(1.0, 31 - s_e[b]);
      uint32_t word[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int q = 0; q < 4; ++q) word[q][u] = 0u;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = 32 * ks + 16 * h + 4 * u + i;
          int8_t d[4] = {0, 0, 0, 0};
          if (j < n) ri8::digits4((w ? w[j] : 1.0) * ((double)x[3 * j + b] - c[b]), qs, d);
#pragma unroll
          for (int q = 0; q < 4; ++q) word[q][u] |= (uint32_t)(uint8_t)d[q] << (8 * i);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        reinterpret_cast<uint4*>(dig + (((int64_t)ks * 4 + q) * R3 + 3 * k + b) * 32)[h] =
            make_uint4(word[q][0], word[q][1], word[q][2], word[q][3]);
    }
    return;
  }
  // one thread per (k-step, axis, 4-atom quad): the 4 digits of 4 consecutive atoms packed
  // into one 32-bit word per digit plane, so 8 threads write a plane's 32 bytes
  for (int task = threadIdx.x; task < 24 * nks; task += 256) {
    const int qd = task & 7, rest = task >> 3;
    const int ks = rest / 3, b = rest - 3 * ks;
    const double qs = ldexp(1.0, 31 - s_e[b]);
    uint32_t word[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int j = 32 * ks + 4 * qd + i;
      int8_t d[4] = {0, 0, 0, 0};
      if (j < n) ri8::digits4((w ? w[j] : 1.0) * ((double)x[3 * j + b] - c[b]), qs, d);
#pragma unroll
      for (int q = 0; q < 4; ++q) word[q] |= (uint32_t)(uint8_t)d[q] << (8 * i);
    }
    // interleaved [3B][nks][4][32]: one 128-byte segment per row and k-step
    uint32_t* dst = reinterpret_cast<uint32_t*>(dig + ((int64_t)(3 * k + b) * nks + ks) * 128) + qd;
#pragma unroll
    for (int q = 0; q < 4; ++q) dst[8 * q] = word[q];
  }
}

// Frame digits in the plane layout, exponents known (from the uniform-weight frame split),
// w = 1: the common path of the windowed refits.  Same digits as rdig_kernel's plane branch,
// but the coordinates go through shared memory in chunks of RD_KC k-steps with coalesced
// 16-byte cp.async copies (double-buffered) instead of 16 scalar 12-byte-strided loads per
// thread (4x the L1 wavefronts of the bytes they use).
constexpr int RD_KC = 40;                  // k-steps per chunk: 1280 atoms, 15 KB, 240 tasks
constexpr int RD_CHF = 3 * 32 * RD_KC;     // floats per chunk
__global__ void __launch_bounds__(256)
rdig_planes_kernel(const float* __restrict__ raw, const double* __restrict__ cen, const int* __restrict__ perm,
                   const int* __restrict__ fmap, int B, int n, int kpad, int8_t* __restrict__ dig,
                   int* __restrict__ eout, const int* __restrict__ ein) {
  __shared__ __align__(16) float sx[2][RD_CHF];
  __shared__ int s_e[3];
  const int k = blockIdx.x;
  if (k >= B) return;
  const int t = perm ? perm[k] : k;
  const int src = fmap ? fmap[t] : t;
  const float* x = raw + (int64_t)src * n * 3;
  double c[3];
#pragma unroll
  for (int b = 0; b < 3; ++b) c[b] = cen[3 * t + b];
  if (threadIdx.x < 3) {
    const int e = ein[3 * t + threadIdx.x];
    s_e[threadIdx.x] = e;
    eout[3 * k + threadIdx.x] = e;
  }
  const int nks = kpad / 32;
  const int nch = (nks + RD_KC - 1) / RD_KC;
  auto issue = [&](int ci) {
    const int a0 = ci * 32 * RD_KC;
    const int cnt = min(32 * RD_KC, n - a0);  // atoms of the chunk (a multiple of 4, may be <= 0)
    const float4* g = reinterpret_cast<const float4*>(x + 3 * (int64_t)a0);
    const uint32_t d0 = ri8::su32(&sx[ci & 1][0]);
    for (int e = threadIdx.x; e < (3 * cnt) / 4; e += 256)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d0 + 16u * e), "l"(g + e) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0);
  const int64_t R3 = 3LL * B;
  for (int ci = 0; ci < nch; ++ci) {
    if (ci + 1 < nch) {
      issue(ci + 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const float* xs = sx[ci & 1];
    const int ks0 = ci * RD_KC, a0 = ks0 * 32;
    const int kc = min(RD_KC, nks - ks0);
    for (int task = threadIdx.x; task < 6 * kc; task += 256) {
      const int h = task & 1, rest = task >> 1;
      const int ksl = rest / 3, b = rest - 3 * ksl;
      const double qs = ldexp(1.0, 31 - s_e[b]);
      uint32_t word[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
#pragma unroll
        for (int q = 0; q < 4; ++q) word[q][u] = 0u;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int jl = 32 * ksl + 16 * h + 4 * u + i;
          int8_t d[4] = {0, 0, 0, 0};
          if (a0 + jl < n) ri8::digits4(1.0 * ((double)xs[3 * jl + b] - c[b]), qs, d);
#pragma unroll
          for (int q = 0; q < 4; ++q) word[q][u] |= (uint32_t)(uint8_t)d[q] << (8 * i);
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        reinterpret_cast<uint4*>(dig + (((int64_t)(ks0 + ksl) * 4 + q) * R3 + 3 * k + b) * 32)[h] =
            make_uint4(word[q][0], word[q][1], word[q][2], word[q][3]);
    }
    __syncthreads();  // the buffer is refilled by the chunk after next
  }
}

__global__ void __launch_bounds__(ri8::NT, 1)
refine_i8_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB, int T, int L,
                 int nks, const int* __restrict__ perm, const int* __restrict__ lo, const int* __restrict__ cnt,
                 const int* __restrict__ eF, const int* __restrict__ eL, const double* __restrict__ gx,
                 const double* __restrict__ ga, int cap, double* __restrict__ Dex, double* __restrict__ Rex,
                 float* __restrict__ Dd, int64_t ldd, uint8_t* __restrict__ flags, double* __restrict__ Sex,
                 const uint8_t* __restrict__ fitmask) {
  using namespace ri8;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sSt = sm;                                                  // [NST][KPS][A 16 KB | B 8 KB]
  double* sC = reinterpret_cast<double*>(sm + NST * STG);            // [FG][LT][9]
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + NST * STG + SC_BYTES);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;  // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  __shared__ uint32_t tmem_slot;
  __shared__ int s_t[FG], s_lo[FG], s_cnt[FG], s_eF[NR];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int groups = (T + FG - 1) / FG;
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
    for (int s = 0; s < NST; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mb_init(&tfull[b], 1); mb_init(&tempty[b], EPI); }
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

  // the window union of group g (every role computes it from global memory)
  auto union_of = [&](int g, int& wlo, int& whi) {
    wlo = L;
    whi = 0;
    for (int f = 0; f < FG; ++f) {
      const int k = g * FG + f;
      if (k >= T) break;
      const int t = perm ? perm[k] : k;
      const int a = lo ? lo[t] : 0, c = lo ? cnt[t] : L;
      if (c > 0) { wlo = min(wlo, a); whi = max(whi, a + c); }
    }
  };

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (one elect.sync lane issues)
    {
      uint32_t st = 0;
      for (int g = blockIdx.x; g < groups; g += gridDim.x) {
        int wlo, whi;
        union_of(g, wlo, whi);
        // serpentine k order: odd landmark tiles of a group sweep K backwards, so they start
        // on the frame rows the previous tile read last (still in L2) instead of re-reading
        // the group's frame rows from HBM in the same order
        for (int l0 = wlo, ti = 0; l0 < whi; l0 += LT, ++ti)
          for (int j = 0; j < nks; j += KPS, ++st) {
            const int s = st % NST;
            const int nk = min(KPS, nks - j);
            mb_wait(&empty[s], ((st / NST) & 1) ^ 1);
            if (elect_one()) {
              mb_expect(&full[s], (uint32_t)(nk * STAGE));
              for (int u = 0; u < nk; ++u) {
                const int ks = (ti & 1) ? nks - 1 - (j + u) : j + u;
                uint8_t* dst = sSt + s * STG + u * STAGE;
                tma2d(&mapA, &full[s], dst, ROWB * ks, 3 * l0);
                tma3d(&mapB, &full[s], dst + A_ST, 0, NR * g, 4 * ks);
              }
            }
            __syncwarp();
          }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    uint32_t st = 0, it = 0;
    const uint32_t sbase = su32(sSt);
    for (int g = blockIdx.x; g < groups; g += gridDim.x) {
      int wlo, whi;
      union_of(g, wlo, whi);
      for (int l0 = wlo; l0 < whi; l0 += LT, ++it) {
        const int ab = it & 1;
        mb_wait(&tempty[ab], ((it >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t d = tmem + (uint32_t)(ab * ACC);
        for (int j = 0; j < nks; j += KPS, ++st) {  // (the k order does not matter to the MMAs)
          const int s = st % NST;
          const int nk = min(KPS, nks - j);
          mb_wait(&full[s], (st / NST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          // one lane chosen by elect.sync issues (under `if (lane == 0)` ptxas wraps every
          // tcgen05.mma / commit in an ELECT ... BRA.U.ANY retry loop)
          if (elect_one()) {
            for (int u = 0; u < nk; ++u) {
              const uint32_t a = sbase + (uint32_t)(s * STG + u * STAGE), b = a + A_ST;
              // the 10 digit products with p + q <= 3 in 4 MMAs: the B tile holds the frame
              // digits plane by plane ([p][64 rows][32 B]), so for landmark digit q ONE MMA with
              // N = (4 - q) 64 reads frame digits 0..3-q and writes the TMEM columns of levels
              // q..3 (kind::i8 with N <= 64 is issue-bound at ~45 clk per MMA, N = 256 runs at
              // N/2 clk: tools/_diag/i8_probe.cu)
              const uint64_t bd = desc32(b), ad = desc128(a);
              mma_i8(d, ad, bd, idesc_n(4 * NB), (j + u) > 0 ? 1u : 0u);
              mma_i8(d + (uint32_t)NB, ad + (KS >> 4), bd, idesc_n(3 * NB), 1u);
              mma_i8(d + (uint32_t)(2 * NB), ad + 2 * (KS >> 4), bd, idesc_n(2 * NB), 1u);
              mma_i8(d + (uint32_t)(3 * NB), ad + 3 * (KS >> 4), bd, idesc_n(NB), 1u);
            }
            mma_commit(&empty[s]);
            if (j + KPS >= nks) mma_commit(&tfull[ab]);
          }
          __syncwarp();
        }
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int r = (warp & 3) * 32 + lane;  // TMEM lane = landmark row 3 l' + g of the tile
    const int lp = r / 3, gg = r - 3 * (r / 3);
    const int et = tid - 128;
    uint32_t it = 0;
    for (int g = blockIdx.x; g < groups; g += gridDim.x) {
      int wlo, whi;
      union_of(g, wlo, whi);
      if (et < FG) {
        const int k = g * FG + et;
        const int t = k < T ? (perm ? perm[k] : k) : -1;
        s_t[et] = t;
        s_lo[et] = (t >= 0 && lo) ? lo[t] : 0;
        s_cnt[et] = t < 0 ? 0 : (lo ? cnt[t] : L);
      }
      if (et < NR) s_eF[et] = (g * NR + et < 3 * T) ? eF[g * NR + et] : 0;
      epi_bar();
      for (int l0 = wlo; l0 < whi; l0 += LT, ++it) {
        const int ab = it & 1;
        const int l = l0 + lp;
        const bool lok = r < 3 * LT && l < L;
        const int el = lok ? eL[3 * l + gg] : 0;
        {  // the accumulator drain: every epilogue warp (TMEM lane quarter = warp % 4), the
           // 7 three-frame column chunks dealt round-robin over the quarter's 3 warps (with only
           // warps 4-7 draining, one warp per scheduler converted all 63 columns serially)
        mb_wait(&tfull[ab], (it >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        __syncwarp();
        const uint32_t tb = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(ab * ACC);
#pragma unroll 1
        for (int fc = (warp - 4) >> 2; fc < FG / 3; fc += EPI / 4) {  // 3 frames (9 columns) at a time
          uint32_t acc[4][9];
#pragma unroll
          for (int lvl = 0; lvl < 4; ++lvl) {
            tld8(tb + NB * lvl + 9 * fc, &acc[lvl][0]);
            tld1(tb + NB * lvl + 9 * fc + 8, &acc[lvl][8]);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (lok) {
#pragma unroll
            for (int c = 0; c < 9; ++c) {
              const int f = 3 * fc + c / 3, b = c % 3;
              const double v = (double)(int)acc[0][c] * 16777216.0 + (double)(int)acc[1][c] * 65536.0 +
                               (double)(int)acc[2][c] * 256.0 + (double)(int)acc[3][c];
              sC[(f * LT + lp) * 9 + 3 * b + gg] = v * pow2d(s_eF[3 * f + b] + el - 38);
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mb_arrive(&tempty[ab]);
        }
        epi_bar();
        // fused fit of the in-window pairs (exact fp64), all epilogue warps
        for (int pi = et; pi < FG * LT; pi += 32 * EPI) {
          const int f = pi / LT, li = pi - f * LT;
          const int t = s_t[f], ll = l0 + li;
          if (t < 0 || ll >= L || ll >= whi) continue;
          const int slot = ll - s_lo[f];
          if (slot < 0 || slot >= s_cnt[f]) continue;
          const double* S = sC + (f * LT + li) * 9;
          if (Sex) {  // close-structure replay: the covariances of every window pair (Eq. 5 rows)
            double* so = Sex + ((int64_t)t * cap + slot) * 9;
#pragma unroll
            for (int e = 0; e < 9; ++e) so[e] = S[e];
          }
          if (fitmask && !fitmask[t]) continue;  // fits only on the refresh rows
          double q[4];
          bool ill = false;
          double msd = fit_fast(S, gx[t], ga[ll], Rex ? q : nullptr, &ill);
          uint8_t fl = 0;
          if (ill) {
            double k4[4][4], V[4][4], ev[4];
            kearsley_from_S(S, gx[t], ga[ll], k4);
            if (!jacobi4(k4, ev, V)) fl |= kFlagNoConverge;
            msd = ev[0];
            q[0] = V[0][0]; q[1] = V[1][0]; q[2] = V[2][0]; q[3] = V[3][0];
          }
          if (Dex) Dex[(int64_t)t * cap + slot] = msd;
          if (Dd) Dd[(int64_t)t * ldd + ll] = (float)msd;
          if (Rex) {
            double rr[9];
            quat_to_rot(q, rr);
            double* o = Rex + ((int64_t)t * cap + slot) * 9;
#pragma unroll
            for (int e = 0; e < 9; ++e) o[e] = rr[e];
          }
          if (fl && flags) flags[t] |= fl;
        }
        epi_bar();  // sC is rewritten by the next tile
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encode_ri8() {
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

// frame digits in planes [nks][4][rows][32 B]: a 3-D map (32 B, rows, plane) whose box
// (32, box_rows, 4) lands in shared memory as 4 digit planes of box_rows 32-byte rows
bool make_dig_planes_map(CUtensorMap* m, const int8_t* dig, int64_t rows, int kpad, int box_rows) {
  auto enc = get_encode_ri8();
  if (!enc) return false;
  cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)(4 * (kpad / 32))};
  cuuint64_t strides[2] = {32, (cuuint64_t)(32 * rows)};
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 4};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(dig), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_dig_map(CUtensorMap* m, const int8_t* dig, int64_t rows, int kpad, int box_rows) {
  auto enc = get_encode_ri8();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)4 * kpad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)4 * kpad};
  cuuint32_t box[2] = {(cuuint32_t)ri8::ROWB, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(dig), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

cudaError_t launch_rdig(const float* raw, const double* cen, const double* w, const int* perm, const int* fmap, int B,
                        int n, int kpad, int8_t* dig, int* e, cudaStream_t stream, const int* ein, int planes) {
  if (B <= 0 || n <= 0) return cudaSuccess;
  if (kpad % 32 || kpad < n) return cudaErrorInvalidValue;
  // stage the structure in shared memory when it fits (n <= 16384: 192 KB)
  const int staged = 0;  // staging a 120 KB row in shared memory (1 CTA / SM) measured slower than two L2-served passes
  const int smem = staged ? 12 * n : 0;
  static bool attr = false;
  if (!attr) {
    cudaError_t e2 = cudaFuncSetAttribute(rdig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 16384);
    if (e2 != cudaSuccess) return e2;
    attr = true;
  }
  if (planes && !w && ein && n % 4 == 0 && (reinterpret_cast<uintptr_t>(raw) & 15) == 0) {
    rdig_planes_kernel<<<B, 256, 0, stream>>>(raw, cen, perm, fmap, B, n, kpad, dig, e, ein);
    return cudaGetLastError();
  }
  rdig_kernel<<<B, 256, smem, stream>>>(raw, cen, w, perm, fmap, B, n, kpad, dig, e, staged, w ? nullptr : ein,
                                        planes);
  return cudaGetLastError();
}

cudaError_t launch_refine_i8(const int8_t* ldig, const int* eL, const int8_t* fdig, const int* eF, int T, int L, int n,
                             int kpad, const int* perm, const int* lo, const int* cnt, const double* gx,
                             const double* ga, int cap, double* Dex, double* Rex, float* Dd, int64_t ldd,
                             uint8_t* flags, cudaStream_t stream, double* Sex, const uint8_t* fitmask) {
  using namespace ri8;
  if (T <= 0 || L <= 0) return cudaSuccess;
  if (kpad % 32 || kpad < n || n >= 32768) return cudaErrorInvalidValue;
  CUtensorMap ma, mb;
  if (!make_dig_map(&ma, ldig, 3LL * L, kpad, MR) || !make_dig_planes_map(&mb, fdig, 3LL * T, kpad, NB))
    return cudaErrorInvalidValue;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(refine_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int groups = (T + FG - 1) / FG;
  const int grid = groups < sms ? groups : sms;
  refine_i8_kernel<<<grid, NT, SMEM, stream>>>(ma, mb, T, L, kpad / 32, perm, lo, cnt, eF, eL, gx, ga, cap, Dex, Rex,
                                               Dd, ldd, flags, Sex, fitmask);
  return cudaGetLastError();
}

}  // namespace mc
