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
// digit product is an exact integer summed exactly in int32 (K <= 384 here).
// Levels p + q <= 3 are kept (10 of the 16 products; the dropped ones weigh
// <= 2^-32 of the leading term), combined in fp64 in the epilogue:
//   v = acc0 + fl32(acc1 2^-8 + acc2 2^-16 + acc3 2^-24).
//
// Two kernels per call:
//  * cstack_prep_kernel (one CTA per frame group): the group's A digits as the
//    exact shared-memory image the MMA reads (K-major, SWIZZLE_32B, one 6 KB
//    block of 192 rows x 32 B per k-step) plus a header (frames, union start,
//    per-row constants), written to a caller workspace;
//  * cv_grad_i8_kernel (persistent, one CTA per SM): per group the header and
//    image are bulk-copied into shared memory once; per atom tile of 128 the B
//    digits stream through a 3-stage ring of 2 x 16 KB TMA boxes (two k-steps
//    per stage; a box = 128 atoms x one 128-byte row = the 4 digits of one
//    32-byte k-step, SWIZZLE_128B, so digit q
//    is the K slice [32q, 32q + 32) of the row and the TMA moves 128-byte row
//    segments, not 32-byte ones); per k-step 4 MMAs with M = 128 atoms (TMEM
//    lanes), K = 32, and the A digits stacked along N: for B digit q one MMA
//    with N = (4 - q) 48 reading A digits 0..3-q into the TMEM columns of levels
//    q..3 -- exactly the 10 kept products.  Accumulators: 4 levels x 48 columns,
//    double-buffered (384 of 512 TMEM columns), so the epilogue of one atom
//    tile overlaps the next tile's MMAs.
// Warp roles (640 threads): 0 TMA producer (header/image, B digits); 1 MMA
// issuer (the warp converged, one elect.sync lane issues); 2 TMEM allocator +
// producer of the frame rows and per-atom constants (1-D bulk copies);
// 4-19 epilogue (TMEM lane quarter = warp % 4, 12 rows = 2 frames (or 4 in
// FORCE mode) per warp).  Groups whose union is wider than WMAX landmarks (or
// n % 4 != 0) are left to the DMMA kernel (launch_cv_grad_dmma, min_width).
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "launch.h"
#include "mc_math.cuh"

namespace mc {

namespace gi8 {
constexpr int R = 48;                 // GEMM rows per frame group
constexpr int NDIG = 4;               // int8 digits per operand
constexpr int BMA = 128;              // atoms per tile (TMEM lanes)
constexpr int KS = 32;                // K bytes per MMA k-step (= per pipeline stage), SWIZZLE_32B rows
constexpr int NKS_MAX = 12;           // k-steps of one group (K <= 384 bytes)
// widest union handled here: 3 WMAX + 31 <= 32 NKS_MAX (the group's K start 3 wlo is
// rounded down to the 32-byte k-step of the digit layout)
constexpr int WMAX = (KS * NKS_MAX - 31) / 3;  // 117 landmarks
constexpr int L_STAGE = NDIG * BMA * KS;       // 16 KB: 128 atom rows x (4 digits x 32 B)
constexpr int C_KS = NDIG * R * KS;            // 6 KB: 192 A rows x 32 B per k-step
constexpr int C_IMG = NKS_MAX * C_KS;          // 72 KB
constexpr int EPI = 16;                        // epilogue warps (4 per TMEM lane quarter)
constexpr int NT = 32 * (4 + EPI);
constexpr int ACC = NDIG * R;  // TMEM columns per accumulator buffer
constexpr int FVEC = 16;
constexpr int RPW = R / 4;     // rows per epilogue warp (12)

// k-steps per pipeline stage: the MMA thread's barrier wait, tcgen05 fence and commit cost
// ~260 clk per stage (clock64 accounting, tools/_diag/r02_s4_gi8_prof.sh) against ~260 clk of
// tensor-pipe work per k-step, so they are paid once per KPS k-steps
constexpr int KPS = 2;
// per-atom constants of a tile (eB int32, w fp64, w' fp64), bulk-copied behind the tile's
// frame rows so the epilogue reads them from shared memory (as global loads their L2 latency
// was exposed once per tile: the 16 epilogue warps run the tile phases in lockstep)
constexpr int XC_BYTES = BMA * (4 + 8 + 8);
template <int NCV>
struct Cfg;  // frames per group, B-digit pipeline stages (of KPS k-steps), frame-row buffer bytes
template <>
struct Cfg<2> {
  static constexpr int DG = 8;
  static constexpr int NST = 3;
  static constexpr int NST_W = 4;  // stages of the streamed-A (wide) kernel
  static constexpr int X_BUF = DG * BMA * 12 + XC_BYTES;
};
template <>
struct Cfg<1> {
  static constexpr int DG = 16;
  static constexpr int NST = 3;
  static constexpr int NST_W = 3;
  static constexpr int X_BUF = DG * BMA * 12 + XC_BYTES;
};

struct RowC {
  double scp;  // sc_r 2^-eA_r (the sum-of-coefficients term in the row's digit units)
  float P;     // 2^eA_r
  float corr;  // the w' correction sum of the row
};

template <int DG>
struct __align__(16) GHdr {
  int t[DG], raw[DG];
  int wlo, koff, k0, nks, active, pad_[3];
  long long img, pad2_;  // wide groups: byte offset of the group's image in the wide workspace
  double cx[DG][3];
  RowC rc[R];
};

// wide groups (union wider than WMAX landmarks): the A digits are not resident; each
// pipeline stage carries the B box and the group's A block of that k-step
constexpr int W_STAGE = L_STAGE + C_KS;  // 22 KB
template <int NCV, bool WIDE = false>
constexpr int smem_bytes() {
  return (WIDE ? Cfg<NCV>::NST_W * KPS * W_STAGE : Cfg<NCV>::NST * KPS * L_STAGE + C_IMG) + 2 * Cfg<NCV>::X_BUF +
         (int)sizeof(GHdr<Cfg<NCV>::DG>) + 32 * 8 + 1024;
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
// L2 eviction policies: the landmark digits are re-read by ~100 frame groups and must
// survive the ~47 GB of frame rows and gradient rows that stream through L2 once
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                      uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, "
      "%3}], [%4], %5;" ::"r"(su32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(su32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                              uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar)), "l"(policy)
      : "memory");
}
// 2^e as an exact fp64 / fp32 (no ldexp: its generic path is a loop of doublings)
__device__ __forceinline__ double pow2d(int e) { return __longlong_as_double((long long)(e + 1023) << 52); }
__device__ __forceinline__ void store_stream(float* p, float v) { __stcs(p, v); }
__device__ __forceinline__ void store_stream(double* p, double v) { __stcs(p, v); }
// K-major SWIZZLE_128B operand (128 B rows, 8-row groups 1024 B apart), layout 2
__device__ __forceinline__ uint64_t desc128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// K-major SWIZZLE_32B operand (32 B rows, 8-row groups 256 B apart), layout 6
__device__ __forceinline__ uint64_t desc32(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
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
__device__ __forceinline__ void tld4(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}

// Shared-state-space loads for the epilogue.  The header and the frame rows are read
// through these (not through generic pointers) so the compiler knows they cannot alias the
// global gradient stores and may schedule the loads of later rows above earlier stores
// (with generic loads every row was a serial load -> fp64 chain -> store sequence).  They are
// plain (non-volatile) asm: the address operand must derive from a token produced by an
// asm volatile AFTER the barrier wait that makes the data visible (shared_token).
__device__ __forceinline__ uint32_t shared_token(const void* p) {
  uint32_t t;
  asm volatile("mov.b32 %0, %1;" : "=r"(t) : "r"(su32(p)));
  return t;
}
__device__ __forceinline__ int lds_i32(uint32_t a) {
  int v;
  asm("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float lds_f32(uint32_t a) {
  float v;
  asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ RowC lds_rowc(uint32_t a) {
  uint32_t x, y, z, u;
  asm("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(u) : "r"(a));
  RowC r;
  r.scp = __hiloint2double((int)y, (int)x);
  r.P = __uint_as_float(z);
  r.corr = __uint_as_float(u);
  return r;
}

// byte offset of (row, kk) in a K-major SWIZZLE_32B operand made of 32-byte-K blocks of
// `rows` rows each (the pattern TMA writes: 16-byte chunk ^= (row % 8) >> 2)
__device__ __forceinline__ int swz32(int row, int kk, int block_bytes) {
  return (kk >> 5) * block_bytes + (row >> 3) * 256 + (row & 7) * 32 + (((((kk & 31) >> 4) ^ ((row & 7) >> 2)) & 1) << 4) +
         (kk & 15);
}

// power-of-two scale of a row / column with max |v| = mx: 2^e with mx 2^(7 - e) <= 127,
// so every value's 31-bit integer X = rint(v 2^(31 - e)) has |X| <= 127 2^24 and its
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
static_assert(smem_bytes<1, true>() <= 227 * 1024 && smem_bytes<2, true>() <= 227 * 1024 &&
              smem_bytes<1>() <= 227 * 1024 && smem_bytes<2>() <= 227 * 1024, "shared memory per CTA");
}  // namespace gi8

// B digits of a landmark set: per-atom exponent eB[k] over every (landmark, axis)
// of the centred coordinates ac = lraw - lcen (fp64), then the digits interleaved per
// 32-byte k-step: dig[npad][kpad / 32][4][32] (row = atom, K = (landmark, axis), zero
// padded), so one atom's 4 digits of a k-step are one 128-byte segment.
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

// tile of 32 atoms x 64 landmarks (192 K bytes = 6 k-steps): coalesced reads through
// shared memory, then one thread per (atom, k-step) writes its 128-byte segment
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
  if (threadIdx.x >= 192) return;
  const int kl = threadIdx.x & 31, c = threadIdx.x >> 5, k = k0 + kl;  // atom, k-step of the tile
  const int kb0 = 3 * l0 + 32 * c;                                   // first K byte of the k-step
  if (k >= n || kb0 >= kpad) return;
  const double qs = ldexp(1.0, 31 - eB[k]);
  alignas(16) int8_t buf[128];
  for (int j = 0; j < 32; ++j) {
    const int kk = 32 * c + j, l = kk / 3, g = kk % 3;
    int8_t d[4] = {0, 0, 0, 0};
    if (l0 + l < L) gi8::digits4((double)sx[l][3 * kl + g] - lcen[3 * (l0 + l) + g], qs, d);
#pragma unroll
    for (int q = 0; q < 4; ++q) buf[32 * q + j] = d[q];
  }
  int4* dst = reinterpret_cast<int4*>(dig + (int64_t)k * 4 * kpad + 4 * kb0);
#pragma unroll
  for (int e = 0; e < 8; ++e) dst[e] = reinterpret_cast<const int4*>(buf)[e];
}

// A digits of one frame group (one CTA per group): the SWIZZLE_32B shared-memory image
// of the 192 stacked digit rows (digit p of GEMM row r = row p * 48 + r) per k-step, and
// the group header.  NCV = 2: rows (f, s|z, b) with coefficients cs_i Rhat_i / cz_i Rhat_i
// (sig_coef [.., 0:9 | 9:18]); NCV = 1: rows (f, b) with -(V_s cs_i + V_z cz_i) Rhat_i.
template <int NCV>
__global__ void __launch_bounds__(128)
cstack_prep_kernel(int T, int cap, const double* __restrict__ fcen, const int* __restrict__ sig_idx,
                   const double* __restrict__ sig_coef, const int* __restrict__ nsig, const double* __restrict__ fvec,
                   const double* __restrict__ dV, const int* __restrict__ perm, const int* __restrict__ out_map,
                   gi8::GHdr<gi8::Cfg<NCV>::DG>* __restrict__ hdrs, uint8_t* __restrict__ cimg,
                   int* __restrict__ wide_flag) {
  using namespace gi8;
  constexpr int DG = Cfg<NCV>::DG;
  constexpr int EPR = 9 * NCV;  // coefficient entries per (frame, significant landmark)
  extern __shared__ __align__(16) uint8_t img[];  // [NKS_MAX][192 rows x 32 B]
  __shared__ GHdr<DG> h;
  __shared__ int s_ns[DG], s_flo[DG], s_fhi[DG], s_cum[DG + 1];
  __shared__ double s_fv[DG][8], s_dv[DG][2];
  __shared__ unsigned long long s_rmax[R];
  __shared__ double s_qs[R];
  const int g = blockIdx.x, tid = threadIdx.x;
  if (tid < DG) {
    const int k = g * DG + tid;
    int t = -1, ns = 0;
    if (k < T) {
      t = perm ? perm[k] : k;
      ns = nsig[t];
    }
    h.t[tid] = t;
    h.raw[tid] = t < 0 ? -1 : (out_map ? out_map[t] : t);
    s_ns[tid] = t < 0 ? 0 : ns;
    s_flo[tid] = (t >= 0 && ns > 0) ? sig_idx[(int64_t)t * cap] : 0x7fffffff;
    s_fhi[tid] = (t >= 0 && ns > 0) ? sig_idx[(int64_t)t * cap + ns - 1] + 1 : -1;
    for (int a = 0; a < 3; ++a) h.cx[tid][a] = t < 0 ? 0.0 : fcen[3 * t + a];
    for (int e = 0; e < 8; ++e) s_fv[tid][e] = t < 0 ? 0.0 : fvec[(int64_t)t * FVEC + e];
    s_dv[tid][0] = (NCV == 1 && t >= 0) ? dV[2 * t] : 0.0;
    s_dv[tid][1] = (NCV == 1 && t >= 0) ? dV[2 * t + 1] : 0.0;
  }
  if (tid < R) s_rmax[tid] = 0ull;
  __syncthreads();
  if (tid == 0) {
    int a = 0x7fffffff, b = -1, tot = 0;
    for (int f = 0; f < DG; ++f) {
      a = min(a, s_flo[f]);
      b = max(b, s_fhi[f]);
      s_cum[f] = tot;
      tot += s_ns[f] * EPR;
    }
    s_cum[DG] = tot;
    const int width = b - a;
    h.active = (b >= 0 && width <= WMAX) ? 1 : 0;
    if (b >= 0 && width > WMAX && wide_flag) atomicOr(wide_flag, 1);  // left to the DMMA kernel / caller
    h.wlo = b >= 0 ? a : 0;
    h.koff = b >= 0 ? (3 * a) & 31 : 0;
    h.k0 = b >= 0 ? 3 * a - h.koff : 0;
    h.nks = h.active ? (3 * width + h.koff + KS - 1) / KS : 0;
    h.pad_[0] = h.pad_[1] = h.pad_[2] = 0;
    h.img = h.pad2_ = 0;
  }
  __syncthreads();
  const int nks = h.nks, wlo = h.wlo, koff = h.koff, tot = s_cum[DG];
  if (h.active) {
    for (int e = tid; e < nks * C_KS / 16; e += 128) reinterpret_cast<int4*>(img)[e] = make_int4(0, 0, 0, 0);
    auto entry = [&](int e, int& row, int& kk) -> double {
      int f = 0;
#pragma unroll
      for (int q = 1; q < DG; ++q) f += e >= s_cum[q];
      const int el = e - s_cum[f];
      const int s = el / EPR, j = el % EPR;
      const int64_t base = (int64_t)h.t[f] * cap + s;
      const int l = sig_idx[base];
      double v;
      if (NCV == 2) {
        v = sig_coef[base * 18 + j];
        row = f * 6 + (j / 9) * 3 + (j % 9) / 3;
      } else {
        v = -(s_dv[f][0] * sig_coef[base * 18 + j] + s_dv[f][1] * sig_coef[base * 18 + 9 + j]);
        row = f * 3 + j / 3;
      }
      kk = 3 * (l - wlo) + j % 3 + koff;
      return v;
    };
    for (int e = tid; e < tot; e += 128) {
      int row, kk;
      const double v = entry(e, row, kk);
      atomicMax(&s_rmax[row], (unsigned long long)__double_as_longlong(fabs(v)));
    }
    __syncthreads();
    if (tid < R) s_qs[tid] = ldexp(1.0, 31 - digit_exp(__longlong_as_double((long long)s_rmax[tid])));
    __syncthreads();
    for (int e = tid; e < tot; e += 128) {
      int row, kk;
      const double v = entry(e, row, kk);
      int8_t d[4];
      digits4(v, s_qs[row], d);
#pragma unroll
      for (int p = 0; p < NDIG; ++p) img[swz32(p * R + row, kk, C_KS)] = (uint8_t)d[p];
    }
  }
  if (tid < R) {
    const int f = NCV == 2 ? tid / 6 : tid / 3;
    const int cv = NCV == 2 ? (tid % 6) / 3 : 0;
    const int b = tid % 3;
    const int e = h.active ? digit_exp(__longlong_as_double((long long)s_rmax[tid])) : 0;
    double sc, corr;
    if (NCV == 2) {
      sc = s_fv[f][cv];
      corr = s_fv[f][2 + cv * 3 + b];
    } else {
      sc = -(s_dv[f][0] * s_fv[f][0] + s_dv[f][1] * s_fv[f][1]);
      corr = -(s_dv[f][0] * s_fv[f][2 + b] + s_dv[f][1] * s_fv[f][5 + b]);
    }
    h.rc[tid].scp = ldexp(sc, -e);
    h.rc[tid].P = ldexpf(1.0f, e);
    h.rc[tid].corr = (float)corr;
  }
  __syncthreads();
  // write out: header (16-byte words) and the used k-steps of the image
  const int4* hs = reinterpret_cast<const int4*>(&h);
  int4* hd = reinterpret_cast<int4*>(hdrs + g);
  for (int e = tid; e < (int)(sizeof(GHdr<DG>) / 16); e += 128) hd[e] = hs[e];
  int4* cd = reinterpret_cast<int4*>(cimg + (int64_t)g * C_IMG);
  for (int e = tid; e < nks * C_KS / 16; e += 128) cd[e] = reinterpret_cast<const int4*>(img)[e];
}

// Wide-group plan (one thread per frame group): bytes of the group's A image when its
// significant union is wider than WMAX landmarks (the narrow kernel skips those), else 0.
template <int NCV>
__global__ void grad_i8_plan_kernel(int T, int cap, const int* __restrict__ sig_idx, const int* __restrict__ nsig,
                                    const int* __restrict__ perm, long long* __restrict__ bytes) {
  using namespace gi8;
  constexpr int DG = Cfg<NCV>::DG;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (T + DG - 1) / DG) return;
  int a = 0x7fffffff, b = -1;
  for (int f = 0; f < DG; ++f) {
    const int k = g * DG + f;
    if (k >= T) break;
    const int t = perm ? perm[k] : k;
    const int ns = nsig[t];
    if (ns <= 0) continue;
    a = min(a, sig_idx[(int64_t)t * cap]);
    b = max(b, sig_idx[(int64_t)t * cap + ns - 1] + 1);
  }
  long long by = 0;
  if (b >= 0 && b - a > WMAX) {
    const int koff = (3 * a) & 31;
    by = (long long)((3 * (b - a) + koff + KS - 1) / KS) * C_KS;
  }
  bytes[g] = by;
}

// A digits of one WIDE frame group (one CTA per listed group): as cstack_prep_kernel, but
// the image (nks > NKS_MAX k-steps) is built NKS_MAX k-steps at a time in shared memory
// and copied to the wide workspace at wide_off[i]; header hdrs[i] (compact order).
template <int NCV>
__global__ void __launch_bounds__(128)
cstack_prep_wide_kernel(int T, int cap, const double* __restrict__ fcen, const int* __restrict__ sig_idx,
                        const double* __restrict__ sig_coef, const int* __restrict__ nsig,
                        const double* __restrict__ fvec, const double* __restrict__ dV, const int* __restrict__ perm,
                        const int* __restrict__ out_map, const int* __restrict__ wide_ids,
                        const long long* __restrict__ wide_off, gi8::GHdr<gi8::Cfg<NCV>::DG>* __restrict__ hdrs,
                        uint8_t* __restrict__ wimg) {
  using namespace gi8;
  constexpr int DG = Cfg<NCV>::DG;
  constexpr int EPR = 9 * NCV;
  extern __shared__ __align__(16) uint8_t img[];  // [NKS_MAX][192 rows x 32 B]
  __shared__ GHdr<DG> h;
  __shared__ int s_ns[DG], s_cum[DG + 1], s_pa[DG], s_pb[DG], s_ccum[DG + 1];
  __shared__ double s_fv[DG][8], s_dv[DG][2];
  __shared__ unsigned long long s_rmax[R];
  __shared__ double s_qs[R];
  const int g = wide_ids[blockIdx.x], tid = threadIdx.x;
  if (tid < DG) {
    const int k = g * DG + tid;
    int t = -1, ns = 0;
    if (k < T) {
      t = perm ? perm[k] : k;
      ns = nsig[t];
    }
    h.t[tid] = t;
    h.raw[tid] = t < 0 ? -1 : (out_map ? out_map[t] : t);
    s_ns[tid] = t < 0 ? 0 : ns;
    for (int a = 0; a < 3; ++a) h.cx[tid][a] = t < 0 ? 0.0 : fcen[3 * t + a];
    for (int e = 0; e < 8; ++e) s_fv[tid][e] = t < 0 ? 0.0 : fvec[(int64_t)t * FVEC + e];
    s_dv[tid][0] = (NCV == 1 && t >= 0) ? dV[2 * t] : 0.0;
    s_dv[tid][1] = (NCV == 1 && t >= 0) ? dV[2 * t + 1] : 0.0;
  }
  if (tid < R) s_rmax[tid] = 0ull;
  __syncthreads();
  if (tid == 0) {
    int a = 0x7fffffff, b = -1, tot = 0;
    for (int f = 0; f < DG; ++f) {
      if (s_ns[f] > 0) {
        a = min(a, sig_idx[(int64_t)h.t[f] * cap]);
        b = max(b, sig_idx[(int64_t)h.t[f] * cap + s_ns[f] - 1] + 1);
      }
      s_cum[f] = tot;
      tot += s_ns[f] * EPR;
    }
    s_cum[DG] = tot;
    h.active = 1;
    h.wlo = a;
    h.koff = (3 * a) & 31;
    h.k0 = 3 * a - h.koff;
    h.nks = (3 * (b - a) + h.koff + KS - 1) / KS;
    h.pad_[0] = h.pad_[1] = h.pad_[2] = 0;
    h.img = wide_off[blockIdx.x];
    h.pad2_ = 0;
  }
  __syncthreads();
  const int nks = h.nks, wlo = h.wlo, koff = h.koff;
  // entry e of the frame-major list restricted to sig positions [pa_f, pb_f) (cum: prefix)
  auto entry = [&](int e, const int* pa, const int* cum, int& row, int& kk) -> double {
    int f = 0;
#pragma unroll
    for (int q = 1; q < DG; ++q) f += e >= cum[q];
    const int el = e - cum[f];
    const int s = pa[f] + el / EPR, j = el % EPR;
    const int64_t base = (int64_t)h.t[f] * cap + s;
    const int l = sig_idx[base];
    double v;
    if (NCV == 2) {
      v = sig_coef[base * 18 + j];
      row = f * 6 + (j / 9) * 3 + (j % 9) / 3;
    } else {
      v = -(s_dv[f][0] * sig_coef[base * 18 + j] + s_dv[f][1] * sig_coef[base * 18 + 9 + j]);
      row = f * 3 + j / 3;
    }
    kk = 3 * (l - wlo) + j % 3 + koff;
    return v;
  };
  if (tid < DG) s_pa[tid] = 0;
  __syncthreads();
  for (int e = tid; e < s_cum[DG]; e += 128) {
    int row, kk;
    const double v = entry(e, s_pa, s_cum, row, kk);
    atomicMax(&s_rmax[row], (unsigned long long)__double_as_longlong(fabs(v)));
  }
  __syncthreads();
  if (tid < R) s_qs[tid] = ldexp(1.0, 31 - digit_exp(__longlong_as_double((long long)s_rmax[tid])));
  uint8_t* dst0 = wimg + h.img;
  for (int c0 = 0; c0 < nks; c0 += NKS_MAX) {
    const int nc = min(NKS_MAX, nks - c0);
    const int k_lo = KS * c0, k_hi = KS * (c0 + nc);  // this chunk's K bytes
    for (int e = tid; e < nc * C_KS / 16; e += 128) reinterpret_cast<int4*>(img)[e] = make_int4(0, 0, 0, 0);
    if (tid < DG) {
      // sig positions whose landmark touches [k_lo, k_hi): 3 (l - wlo) + koff + 2 >= k_lo and
      // 3 (l - wlo) + koff < k_hi (the ascending list, binary searches)
      const int64_t base = (int64_t)max(h.t[tid], 0) * cap;
      const int ns = s_ns[tid];
      const int lmin = wlo + max(0, (k_lo - koff - 2 + 2) / 3), lmax = wlo + (k_hi - koff + 2) / 3;  // [lmin, lmax)
      int lo = 0, hi = ns;
      while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (sig_idx[base + m] < lmin) lo = m + 1; else hi = m;
      }
      const int pa = lo;
      hi = ns;
      while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (sig_idx[base + m] < lmax) lo = m + 1; else hi = m;
      }
      s_pa[tid] = pa;
      s_pb[tid] = lo;
    }
    __syncthreads();
    if (tid == 0) {
      int tot = 0;
      for (int f = 0; f < DG; ++f) {
        s_ccum[f] = tot;
        tot += (s_pb[f] - s_pa[f]) * EPR;
      }
      s_ccum[DG] = tot;
    }
    __syncthreads();
    for (int e = tid; e < s_ccum[DG]; e += 128) {
      int row, kk;
      const double v = entry(e, s_pa, s_ccum, row, kk);
      if (kk < k_lo || kk >= k_hi) continue;
      int8_t d[4];
      digits4(v, s_qs[row], d);
#pragma unroll
      for (int p = 0; p < NDIG; ++p) img[swz32(p * R + row, kk - k_lo, C_KS)] = (uint8_t)d[p];
    }
    __syncthreads();
    int4* cd = reinterpret_cast<int4*>(dst0 + (int64_t)c0 * C_KS);
    for (int e = tid; e < nc * C_KS / 16; e += 128) cd[e] = reinterpret_cast<const int4*>(img)[e];
    __syncthreads();
  }
  if (tid < R) {
    const int f = NCV == 2 ? tid / 6 : tid / 3;
    const int cv = NCV == 2 ? (tid % 6) / 3 : 0;
    const int b = tid % 3;
    const int e = digit_exp(__longlong_as_double((long long)s_rmax[tid]));
    double sc, corr;
    if (NCV == 2) {
      sc = s_fv[f][cv];
      corr = s_fv[f][2 + cv * 3 + b];
    } else {
      sc = -(s_dv[f][0] * s_fv[f][0] + s_dv[f][1] * s_fv[f][1]);
      corr = -(s_dv[f][0] * s_fv[f][2 + b] + s_dv[f][1] * s_fv[f][5 + b]);
    }
    h.rc[tid].scp = ldexp(sc, -e);
    h.rc[tid].P = ldexpf(1.0f, e);
    h.rc[tid].corr = (float)corr;
  }
  __syncthreads();
  const int4* hs = reinterpret_cast<const int4*>(&h);
  int4* hd = reinterpret_cast<int4*>(hdrs + blockIdx.x);
  for (int e = tid; e < (int)(sizeof(GHdr<DG>) / 16); e += 128) hd[e] = hs[e];
}

// diagnostic switch (env MC_GI8_EXP, results invalid): bit 0 = the epilogue only drains the
// accumulators (TMEM loads, no recombination or stores) -- the MMA / TMA-side time; bit 1 =
// no MMAs issued (commits only) -- the operand-delivery time; bit 2 = no B-digit boxes loaded
// (the producer only arrives) -- the MMA + epilogue time without L2 -> shared-memory delivery
__constant__ int c_gi8_exp = 0;

// -DMC_GI8_PROF (diagnostic build, tools/_diag/r02_s4_gi8_prof.sh): clock64 accounting of
// block 0's producer / MMA / frame-row / epilogue (warp 4) threads, printed by the launcher
#ifdef MC_GI8_PROF
__device__ unsigned long long g_gi8_prof[32];
#define GP_DECL unsigned long long gp_t = clock64(), gp_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}
#define GP_LAP(i)                               \
  do {                                          \
    const unsigned long long gp_n = clock64();  \
    gp_acc[i] += gp_n - gp_t;                   \
    gp_t = gp_n;                                \
  } while (0)
#define GP_CNT(i) (++gp_acc[i])
#define GP_FLUSH(base, cond)                                                    \
  do {                                                                          \
    if (blockIdx.x == 0 && (cond))                                              \
      for (int gp_i = 0; gp_i < 8; ++gp_i) atomicAdd(&g_gi8_prof[(base) + gp_i], gp_acc[gp_i]); \
  } while (0)
#else
#define GP_DECL
#define GP_LAP(i)
#define GP_CNT(i)
#define GP_FLUSH(base, cond)
#endif

template <typename OT, int NCV, bool WIDE>
__global__ void __launch_bounds__(gi8::NT, 1)
cv_grad_i8_kernel(const __grid_constant__ CUtensorMap mapB, int T, int n, int npad, const float* __restrict__ fraw,
                  const double* __restrict__ w, const double* __restrict__ wa, const int* __restrict__ eB,
                  const gi8::GHdr<gi8::Cfg<NCV>::DG>* __restrict__ hdrs, const uint8_t* __restrict__ cimg,
                  OT* __restrict__ out0, OT* __restrict__ out1) {
  using namespace gi8;
  constexpr int DG = Cfg<NCV>::DG;
  constexpr int NST = WIDE ? Cfg<NCV>::NST_W : Cfg<NCV>::NST;
  constexpr int SUB = WIDE ? W_STAGE : L_STAGE;  // bytes of one k-step (WIDE: B box + the k-step's A block)
  constexpr int STG = KPS * SUB;                 // stage bytes
  constexpr int X_BUF = Cfg<NCV>::X_BUF;
  using Hdr = GHdr<DG>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sL = sm;                  // [NST][KPS][128 atoms][4 digits x 32 B] (SWIZZLE_128B) [+ A block]
  uint8_t* sC = sL + NST * STG;      // [NKS_MAX][192 rows x 32 B] (narrow groups only)
  uint8_t* sX = sC + (WIDE ? 0 : C_IMG);  // [2][DG][128 atoms x 3] fp32
  Hdr* hdr = reinterpret_cast<Hdr*>(sX + 2 * X_BUF);
  uint64_t* lfull = reinterpret_cast<uint64_t*>(hdr + 1);
  uint64_t* lempty = lfull + NST;
  uint64_t* cfull = lempty + NST;
  uint64_t* cempty = cfull + 1;
  uint64_t* tfull = cempty + 1;   // [2]
  uint64_t* tempty = tfull + 2;   // [2]
  uint64_t* xfull = tempty + 2;   // [2]
  uint64_t* xempty = xfull + 2;   // [2]
  __shared__ uint32_t tmem_slot;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int groups = WIDE ? T : (T + DG - 1) / DG;  // WIDE: T = the number of listed groups
  const int ntile = (n + BMA - 1) / BMA;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
    for (int s = 0; s < NST; ++s) { mb_init(&lfull[s], 1); mb_init(&lempty[s], 1); }
    mb_init(cfull, 1);
    mb_init(cempty, 1 + 1 + EPI);  // MMA commit + frame-row producer + epilogue warps
    for (int b = 0; b < 2; ++b) {
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

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    // (the warp walks the loops converged, one elect.sync lane issues the copies)
    {
      int i = 0;
      uint32_t st = 0;
      const uint64_t keep = policy_evict_last();
      GP_DECL;
      for (int g = blockIdx.x; g < groups; g += gridDim.x, ++i) {
        const Hdr* hg = hdrs + g;
        const int active = hg->active, nks = hg->nks, k0 = hg->k0;
        GP_LAP(0);
        mb_wait(cempty, (i & 1) ^ 1);  // the previous group's MMAs, frame rows and epilogue are done
        GP_LAP(1);
        if (elect_one()) {
          mb_expect(cfull, (uint32_t)(sizeof(Hdr) + ((active && !WIDE) ? nks * C_KS : 0)));
          bulk_g2s(hdr, hg, (uint32_t)sizeof(Hdr), cfull);
          if (active && !WIDE) bulk_g2s(sC, cimg + (int64_t)g * C_IMG, (uint32_t)(nks * C_KS), cfull);
        }
        __syncwarp();
        if (!active) continue;
        const uint8_t* aimg = WIDE ? cimg + hg->img : nullptr;
        for (int tl = 0; tl < ntile; ++tl) {
          const int a0 = tl * BMA;
          for (int j = 0; j < nks; j += KPS, ++st) {
            const int s = st % NST;
            const int nk = min(KPS, nks - j);
            GP_LAP(0);
            mb_wait(&lempty[s], ((st / NST) & 1) ^ 1);
            GP_LAP(2);
            if (elect_one()) {
              if (c_gi8_exp & 4) {  // diagnostic: no operand delivery (the MMAs read stale stages)
                mb_arrive(&lfull[s]);
              } else {
                mb_expect(&lfull[s], (uint32_t)(nk * SUB));
                for (int u = 0; u < nk; ++u) {
                  uint8_t* dst = sL + s * STG + u * SUB;
                  tma2d(&mapB, &lfull[s], dst, 4 * (k0 + KS * (j + u)), a0, keep);
                  if (WIDE) bulk_g2s(dst + L_STAGE, aimg + (int64_t)(j + u) * C_KS, (uint32_t)C_KS, &lfull[s]);
                }
              }
            }
            __syncwarp();
          }
        }
      }
      GP_LAP(0);
      GP_FLUSH(0, lane == 0);
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp walks the loop converged and one lane chosen by elect.sync issues: under
    // `if (lane == 0)` ptxas wraps every tcgen05.mma / commit in an ELECT ... BRA.U.ANY retry
    // loop (it cannot prove a single active thread), ~85 clk of issue path per MMA against
    // ~65 clk of tensor-pipe work.
    int i = 0;
    uint32_t it = 0, st = 0;
    constexpr uint32_t ID0 = idesc_i8(4 * R), ID1 = idesc_i8(3 * R), ID2 = idesc_i8(2 * R), ID3 = idesc_i8(R);
    const uint32_t cbase = su32(sC), lbase = su32(sL);
    const bool no_mma = c_gi8_exp & 2;
    GP_DECL;
    for (int g = blockIdx.x; g < groups; g += gridDim.x, ++i) {
      GP_LAP(0);
      mb_wait(cfull, i & 1);
      GP_LAP(1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int active = hdr->active, nks = hdr->nks;
      if (active) {
        for (int tl = 0; tl < ntile; ++tl, ++it) {
          const int ab = it & 1;
          GP_LAP(0);
          mb_wait(&tempty[ab], ((it >> 1) & 1) ^ 1);
          GP_LAP(2);
          GP_CNT(6);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t d = tmem + (uint32_t)(ab * ACC);
          for (int j = 0; j < nks; j += KPS, ++st) {
            const int s = st % NST;
            const int nk = min(KPS, nks - j);
            GP_LAP(0);
            mb_wait(&lfull[s], (st / NST) & 1);
            GP_LAP(3);
            GP_CNT(7);
            asm volatile("tcgen05.fence::after_thread_sync;");
            if (elect_one()) {
              if (!no_mma) {
                for (int u = 0; u < nk; ++u) {
                  const uint32_t lb = lbase + (uint32_t)(s * STG + u * SUB);
                  const uint64_t bdesc = desc32(WIDE ? lb + (uint32_t)L_STAGE : cbase + (uint32_t)((j + u) * C_KS));
                  const uint64_t adesc = desc128(lb);  // digit q: the K slice [32 q, 32 q + 32) of the 128-byte rows
                  mma_i8(d, adesc, bdesc, ID0, (j + u) == 0 ? 0u : 1u);
                  mma_i8(d + R, adesc + (KS >> 4), bdesc, ID1, 1u);
                  mma_i8(d + 2 * R, adesc + 2 * (KS >> 4), bdesc, ID2, 1u);
                  mma_i8(d + 3 * R, adesc + 3 * (KS >> 4), bdesc, ID3, 1u);
                }
              }
              mma_commit(&lempty[s]);
              if (j + KPS >= nks) mma_commit(&tfull[ab]);
            }
            __syncwarp();
            GP_LAP(4);
          }
        }
      }
      if (elect_one()) {
        if (active) mma_commit(cempty);  // arrives once the group's MMAs have read the image
        else mb_arrive(cempty);
      }
      __syncwarp();
    }
    GP_LAP(0);
    GP_FLUSH(8, lane == 0);
  } else if (warp == 2) {
    // ------------------------------------------------------------ frame-row producer
    if (lane == 0) {
      int i = 0;
      uint32_t it = 0;
      const uint64_t once = policy_evict_first();
      GP_DECL;
      for (int g = blockIdx.x; g < groups; g += gridDim.x, ++i) {
        GP_LAP(0);
        mb_wait(cfull, i & 1);
        GP_LAP(1);
        if (hdr->active) {
          int rows = 0, raw[DG];
#pragma unroll
          for (int f = 0; f < DG; ++f) {
            raw[f] = hdr->raw[f];
            rows += raw[f] >= 0;
          }
          for (int tl = 0; tl < ntile; ++tl, ++it) {
            const int a0 = tl * BMA, nat = min(BMA, n - a0);
            const int xb = it & 1;
            GP_LAP(0);
            mb_wait(&xempty[xb], ((it >> 1) & 1) ^ 1);
            GP_LAP(2);
            mb_expect(&xfull[xb], (uint32_t)((rows * 12 + 20) * nat));
            uint8_t* X = sX + xb * X_BUF;
            uint8_t* XC = X + DG * BMA * 12;
            bulk_g2s(XC, eB + a0, (uint32_t)(4 * nat), &xfull[xb]);
            bulk_g2s(XC + 4 * BMA, w + a0, (uint32_t)(8 * nat), &xfull[xb]);
            bulk_g2s(XC + 12 * BMA, wa + a0, (uint32_t)(8 * nat), &xfull[xb]);
#pragma unroll
            for (int f = 0; f < DG; ++f)
              if (raw[f] >= 0)
                bulk_g2s_hint(X + f * BMA * 12, fraw + ((int64_t)raw[f] * n + a0) * 3, (uint32_t)(12 * nat), &xfull[xb],
                              once);
          }
        }
        mb_arrive(cempty);
      }
      GP_LAP(0);
      GP_FLUSH(16, true);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ epilogue
    const int qd = warp & 3, part = (warp - 4) >> 2;  // TMEM lane quarter, row block of 12
    constexpr int FPW = RPW / (3 * NCV);            // frames per warp (2, or 4 in FORCE mode)
    int i = 0;
    uint32_t it = 0;
    GP_DECL;
    for (int g = blockIdx.x; g < groups; g += gridDim.x, ++i) {
      GP_LAP(0);
      mb_wait(cfull, i & 1);
      GP_LAP(1);
      const uint32_t hs = shared_token(hdr);  // the group's header, shared state space
      if (hdr->active) {
        for (int tl = 0; tl < ntile; ++tl, ++it) {
          const int ab = it & 1;
          const int al = qd * 32 + lane;
          const int a = tl * BMA + al;
          const bool valid = a < n;
          // the tile's frame rows and per-atom constants (the B column scale 2^eB and the
          // weights) are in shared memory well before its accumulators are complete
          GP_LAP(0);
          mb_wait(&xfull[ab], (it >> 1) & 1);
          GP_LAP(4);
          const uint32_t xs0 = shared_token(sX + ab * X_BUF);
          const uint32_t xcs = xs0 + (uint32_t)(DG * BMA * 12);
          const int eb = valid ? lds_i32(xcs + 4 * al) : 0;
          const double sxa = pow2d(14 - eb);
          const double q2w = valid ? 2.0 * lds_f64(xcs + 4 * BMA + 8 * al) * pow2d(eb - 14) : 0.0;
          const double wak = valid ? lds_f64(xcs + 12 * BMA + 8 * al) : 0.0;
          const float q2wf = (float)q2w, wakf = (float)wak;
          GP_LAP(0);
          mb_wait(&tfull[ab], (it >> 1) & 1);
          GP_LAP(2);
          asm volatile("tcgen05.fence::after_thread_sync;");
          __syncwarp();  // tcgen05.ld is .sync.aligned: the whole warp, converged
          uint32_t acc[NDIG][RPW];
          const uint32_t tb = tmem + ((uint32_t)(qd * 32) << 16) + (uint32_t)(ab * ACC + part * RPW);
#pragma unroll
          for (int l = 0; l < NDIG; ++l) {
            tld8(tb + l * R, &acc[l][0]);
            tld4(tb + l * R + 8, &acc[l][8]);
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mb_arrive(&tempty[ab]);
          GP_LAP(3);
          if (c_gi8_exp & 1) {
            __syncwarp();
            if (lane == 0) mb_arrive(&xempty[ab]);
            continue;
          }
          const uint32_t xs = xs0 + (uint32_t)(al * 12);
#pragma unroll
          for (int fl = 0; fl < FPW; ++fl) {
            const int f = part * FPW + fl;
            const int raw = lds_i32(hs + (uint32_t)(offsetof(Hdr, raw) + 4 * f));
            if (raw < 0) continue;  // warp-uniform
            double xc[3];
#pragma unroll
            for (int b = 0; b < 3; ++b)
              xc[b] = ((double)lds_f32(xs + (uint32_t)((f * BMA * 3 + b) * 4)) -
                       lds_f64(hs + (uint32_t)(offsetof(Hdr, cx) + 8 * (3 * f + b)))) * sxa;
#pragma unroll
            for (int cv = 0; cv < NCV; ++cv) {
              OT* dst = (cv ? out1 : out0) + ((int64_t)raw * n + a) * 3;
#pragma unroll
              for (int b = 0; b < 3; ++b) {
                const int rl = fl * 3 * NCV + cv * 3 + b;
                const RowC rc = lds_rowc(hs + (uint32_t)(offsetof(Hdr, rc) + 16 * (part * RPW + rl)));
                const float lo = fmaf((float)(int)acc[3][rl], 5.9604644775390625e-8f,
                                      fmaf((float)(int)acc[2][rl], 1.52587890625e-5f,
                                           (float)(int)acc[1][rl] * 3.90625e-3f));
                if constexpr (sizeof(OT) == 4) {
                  // fp32 outputs: only the cancelling step sc' xc' - acc0 in fp64 (3 fp64-pipe
                  // ops per output instead of 9); t1 and lo are then both far below 2^31 units and
                  // the rest is fp32 (relative error ~2^-23 of the result, the output's own rounding)
                  const double t1 = fma(rc.scp, xc[b], -(double)(int)acc[0][rl]);
                  const float tt = (float)t1 - lo;
                  if (valid) store_stream(dst + b, (OT)fmaf(tt, rc.P * q2wf, -wakf * rc.corr));
                } else {
                  const double v = (double)(int)acc[0][rl] + (double)lo;
                  // t = sc' xc' - v in units of 2^(eA_r + eB_k - 14)
                  const double tt = fma(rc.scp, xc[b], -v);
                  if (valid) store_stream(dst + b, (OT)(tt * (double)rc.P * q2w - wak * (double)rc.corr));
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) mb_arrive(&xempty[ab]);
          GP_LAP(5);
        }
      }
      __syncwarp();
      if (lane == 0) mb_arrive(cempty);
    }
    GP_LAP(0);
    GP_FLUSH(24, warp == 4 && lane == 0);
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
bool make_ldig_map(CUtensorMap* map, const int8_t* dig, int npad, int kpad) {
  using namespace gi8;
  auto enc = get_encode_i8();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)NDIG * kpad, (cuuint64_t)npad};
  cuuint64_t strides[1] = {(cuuint64_t)NDIG * kpad};
  cuuint32_t box[2] = {(cuuint32_t)(NDIG * KS), (cuuint32_t)BMA};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<int8_t*>(dig), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count_i8() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}
}  // namespace

cudaError_t launch_ldig(const float* lraw, const double* lcen, int L, int n, int npad, int kpad, int* eB,
                        int8_t* dig, cudaStream_t stream) {
  if (L <= 0 || n <= 0) return cudaSuccess;
  if (npad < n || kpad < 3 * L || kpad % 32) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(dig, 0, (size_t)gi8::NDIG * npad * kpad, stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(eB, 0, (size_t)npad * sizeof(int), stream);
  if (e != cudaSuccess) return e;
  ldig_scale_kernel<<<(n + 127) / 128, 128, 0, stream>>>(lraw, lcen, L, n, eB);
  dim3 grid((n + 31) / 32, (L + 63) / 64);
  ldig_kernel<<<grid, 256, 0, stream>>>(lraw, lcen, L, n, npad, kpad, eB, dig);
  return cudaGetLastError();
}

size_t grad_i8_workspace(int T, int ncv) {
  using namespace gi8;
  const int DG = ncv == 2 ? Cfg<2>::DG : Cfg<1>::DG;
  const size_t groups = (size_t)((T + DG - 1) / DG);
  const size_t hb = ncv == 2 ? sizeof(GHdr<Cfg<2>::DG>) : sizeof(GHdr<Cfg<1>::DG>);
  return groups * (hb + C_IMG) + 256;
}

// ncv = 2: ds (out0), dz (out1); ncv = 1: fused bias force F (out0) with dV [T, 2]
cudaError_t launch_cv_grad_i8(int T, int n, int cap, const float* fraw, const double* fcen, const float* lraw,
                              const double* lcen, const double* w, const double* wa, const int8_t* dig, const int* eB,
                              int npad, int kpad, const int* sig_idx, const double* sig_coef, const int* nsig,
                              const double* fvec, const double* dV, const int* perm, const int* out_map, void* out0,
                              void* out1, int out_f32, int ncv, int* wide_flag, void* ws, size_t ws_bytes,
                              cudaStream_t stream) {
  using namespace gi8;
  if (T <= 0 || n <= 0) return cudaSuccess;
  if (ncv != 1 && ncv != 2) return cudaErrorInvalidValue;
  const bool ok_i8 = n % 4 == 0 && (reinterpret_cast<uintptr_t>(fraw) & 15) == 0 && kpad % 32 == 0 &&
                     npad % BMA == 0 && ws && ws_bytes >= grad_i8_workspace(T, ncv);
  if (!ok_i8) {
    if (ncv != 2) return cudaErrorInvalidValue;  // the force path needs the tensor-core kernel
    return launch_cv_grad_dmma(T, n, cap, fraw, fcen, lraw, lcen, w, wa, sig_idx, sig_coef, nsig, fvec, perm, out_map,
                               out0, out1, out_f32, stream, -1);
  }
  // diagnostic switch (MC_GI8_DBG bit 16: skip the DMMA pass of the wide groups)
  static const int dbg = [] {
    const char* e = getenv("MC_GI8_DBG");
    return e ? atoi(e) : 0;
  }();
  static const bool exp_set = [] {
    const char* e = getenv("MC_GI8_EXP");
    if (!e) return true;
    const int v = atoi(e);
    return cudaMemcpyToSymbol(c_gi8_exp, &v, sizeof(int)) == cudaSuccess;
  }();
  (void)exp_set;
  CUtensorMap map;
  if (!make_ldig_map(&map, dig, npad, kpad)) return cudaErrorInvalidValue;
  const int sms = sm_count_i8();
  const int DG = ncv == 2 ? Cfg<2>::DG : Cfg<1>::DG;
  const int groups = (T + DG - 1) / DG;
  const int grid = groups < sms ? groups : sms;
  uint8_t* wsb = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws) + 255) & ~uintptr_t(255));
#define MC_GI8(OTT, NC)                                                                                          \
  do {                                                                                                           \
    using H = GHdr<Cfg<NC>::DG>;                                                                                 \
    H* hdrs = reinterpret_cast<H*>(wsb);                                                                         \
    uint8_t* cimg = wsb + (size_t)groups * sizeof(H);                                                            \
    static bool attr = false;                                                                                    \
    if (!attr) {                                                                                                 \
      cudaError_t e = cudaFuncSetAttribute(cv_grad_i8_kernel<OTT, NC, false>,                                    \
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<NC>());       \
      if (e == cudaSuccess)                                                                                      \
        e = cudaFuncSetAttribute(cstack_prep_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, C_IMG);    \
      if (e != cudaSuccess) return e;                                                                            \
      attr = true;                                                                                               \
    }                                                                                                            \
    cstack_prep_kernel<NC><<<groups, 128, C_IMG, stream>>>(T, cap, fcen, sig_idx, sig_coef, nsig, fvec, dV,      \
                                                           perm, out_map, hdrs, cimg, wide_flag);                \
    cv_grad_i8_kernel<OTT, NC, false><<<grid, NT, smem_bytes<NC>(), stream>>>(map, T, n, npad, fraw, w, wa, eB,  \
                                                                              hdrs,                              \
                                                                       cimg, (OTT*)out0, (OTT*)out1);            \
  } while (0)
  if (ncv == 2) {
    if (out_f32) MC_GI8(float, 2); else MC_GI8(double, 2);
  } else {
    if (out_f32) MC_GI8(float, 1); else MC_GI8(double, 1);
  }
#undef MC_GI8
#ifdef MC_GI8_PROF
  {
    unsigned long long h[32];
    cudaStreamSynchronize(stream);
    cudaMemcpyFromSymbol(h, g_gi8_prof, sizeof(h));
    fprintf(stderr, "gi8prof producer: other %llu wait_cempty %llu wait_lempty %llu\n", h[0], h[1], h[2]);
    fprintf(stderr, "gi8prof mma: other %llu wait_cfull %llu wait_tempty %llu wait_lfull %llu issue %llu tiles %llu ksteps %llu\n",
            h[8], h[9], h[10], h[11], h[12], h[14], h[15]);
    fprintf(stderr, "gi8prof rows: other %llu wait_cfull %llu wait_xempty %llu\n", h[16], h[17], h[18]);
    fprintf(stderr, "gi8prof epi: other %llu wait_cfull %llu wait_tfull %llu tmem_ld %llu wait_xfull %llu math_store %llu\n",
            h[24], h[25], h[26], h[27], h[28], h[29]);
    memset(h, 0, sizeof(h));
    cudaMemcpyToSymbol(g_gi8_prof, h, sizeof(h));
  }
#endif
  cudaError_t e = cudaGetLastError();
  // ncv = 2 with wide_flag: the caller runs the wide groups on launch_cv_grad_i8_wide
  if (e != cudaSuccess || ncv != 2 || (dbg & 16) || wide_flag) return e;
  // groups wider than WMAX landmarks: the DMMA kernel (every other group returns at once)
  return launch_cv_grad_dmma(T, n, cap, fraw, fcen, lraw, lcen, w, wa, sig_idx, sig_coef, nsig, fvec, perm, out_map,
                             out0, out1, out_f32, stream, WMAX);
}

cudaError_t launch_grad_i8_plan(int T, int cap, int ncv, const int* sig_idx, const int* nsig, const int* perm,
                                long long* bytes, cudaStream_t stream) {
  using namespace gi8;
  if (T <= 0) return cudaSuccess;
  const int DG = ncv == 2 ? Cfg<2>::DG : Cfg<1>::DG;
  const int groups = (T + DG - 1) / DG;
  if (ncv == 2)
    grad_i8_plan_kernel<2><<<(groups + 127) / 128, 128, 0, stream>>>(T, cap, sig_idx, nsig, perm, bytes);
  else
    grad_i8_plan_kernel<1><<<(groups + 127) / 128, 128, 0, stream>>>(T, cap, sig_idx, nsig, perm, bytes);
  return cudaGetLastError();
}

size_t grad_i8_wide_header_bytes(int nwide, int ncv) {
  using namespace gi8;
  const size_t hb = ncv == 2 ? sizeof(GHdr<Cfg<2>::DG>) : sizeof(GHdr<Cfg<1>::DG>);
  return (size_t)nwide * hb + 256;
}

// the wide groups (listed in wide_ids, their images at byte offsets wide_off of wimg):
// A images built in chunks, then the streamed-A kernel over the listed groups
cudaError_t launch_cv_grad_i8_wide(int T, int n, int cap, const float* fraw, const double* fcen, const double* w,
                                   const double* wa, const int8_t* dig, const int* eB, int npad, int kpad,
                                   const int* sig_idx, const double* sig_coef, const int* nsig, const double* fvec,
                                   const double* dV, const int* perm, const int* out_map, void* out0, void* out1,
                                   int out_f32, int ncv, const int* wide_ids, int nwide, const long long* wide_off,
                                   void* hws, void* wimg, cudaStream_t stream) {
  using namespace gi8;
  if (T <= 0 || nwide <= 0) return cudaSuccess;
  if ((ncv != 1 && ncv != 2) || n % 4 != 0 || (reinterpret_cast<uintptr_t>(fraw) & 15) || kpad % 32 ||
      npad % BMA || !hws || !wimg)
    return cudaErrorInvalidValue;
  CUtensorMap map;
  if (!make_ldig_map(&map, dig, npad, kpad)) return cudaErrorInvalidValue;
  const int sms = sm_count_i8();
  const int grid = nwide < sms ? nwide : sms;
  uint8_t* hb = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(hws) + 255) & ~uintptr_t(255));
#define MC_GI8W(OTT, NC)                                                                                         \
  do {                                                                                                           \
    using H = GHdr<Cfg<NC>::DG>;                                                                                 \
    H* hdrs = reinterpret_cast<H*>(hb);                                                                          \
    static bool attr = false;                                                                                    \
    if (!attr) {                                                                                                 \
      cudaError_t e = cudaFuncSetAttribute(cv_grad_i8_kernel<OTT, NC, true>,                                     \
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes<NC, true>()); \
      if (e == cudaSuccess)                                                                                      \
        e = cudaFuncSetAttribute(cstack_prep_wide_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                                 C_IMG);                                                                         \
      if (e != cudaSuccess) return e;                                                                            \
      attr = true;                                                                                               \
    }                                                                                                            \
    cstack_prep_wide_kernel<NC><<<nwide, 128, C_IMG, stream>>>(T, cap, fcen, sig_idx, sig_coef, nsig, fvec, dV,  \
                                                               perm, out_map, wide_ids, wide_off, hdrs,          \
                                                               (uint8_t*)wimg);                                  \
    cv_grad_i8_kernel<OTT, NC, true><<<grid, NT, smem_bytes<NC, true>(), stream>>>(                              \
        map, nwide, n, npad, fraw, w, wa, eB, hdrs, (const uint8_t*)wimg, (OTT*)out0, (OTT*)out1);               \
  } while (0)
  if (ncv == 2) {
    if (out_f32) MC_GI8W(float, 2); else MC_GI8W(double, 2);
  } else {
    if (out_f32) MC_GI8W(float, 1); else MC_GI8W(double, 1);
  }
#undef MC_GI8W
  return cudaGetLastError();
}

}  // namespace mc
