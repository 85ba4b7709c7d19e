// K2+K3 on CTA pairs: tcgen05.mma.cta_group::2 (M = 256 frames per pair).
//
// Same math and accumulator layout as msd_tf32_kernel (tf32_gemm.cu): for
// every frame axis b a TMEM accumulator [frames x 144] with columns
// (g, l) = 48 g + l, 3 axes x 3 split terms = 9 MMAs per 8-atom k-step.
// What changes is the operand traffic per SM: a cluster of two CTAs on one
// TPC computes a 256-frame x 48-landmark tile; each CTA stages only its own
// 128 frame rows (A) and HALF of the 144 landmark rows (B: CTA0 holds
// (g=0, l 0..47) + (g=1, l 0..23), CTA1 (g=1, l 24..47) + (g=2, l 0..47)),
// so per MMA each SM's shared memory supplies 4 KB of A + 2.25 KB of B
// instead of 4 + 4.5 KB, and each SM pulls 57 KB instead of 66 KB per stage
// from L2.  The leader CTA (rank 0) issues the MMAs for the pair; TMA loads
// of both CTAs complete on the leader's full barrier (cta_group::2 TMA with
// the peer-masked barrier address); MMA commits multicast to both CTAs'
// empty / tmem-full barriers; both epilogues report to the leader's
// tmem-empty barrier.  Each CTA reads its own 128 TMEM lanes in the
// epilogue exactly like the 1-CTA kernel.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "mc_math.cuh"
#include "tc_epilogue.cuh"

namespace mc {

namespace g2 {
constexpr int BM = 128;            // frame rows per CTA (256 per pair)
constexpr int BL = 48;             // landmarks per tile
constexpr int BN = 3 * BL;         // 144 accumulator columns per frame axis
constexpr int BNH = BN / 2;        // 72 landmark rows staged per CTA
constexpr int BOX = 24;            // landmark rows per TMA box (3 boxes per CTA per hi|lo)
constexpr int ROWB = 64;           // bytes per operand row per stage (SWIZZLE_64B): 16 tf32 / 32 f16 atoms
constexpr int STAGES = 3;
constexpr int A_BYTES = BM * ROWB;          // 8 KB
constexpr int B_BYTES = BNH * ROWB;         // 4.5 KB
constexpr int BOX_BYTES = BOX * ROWB;       // 1.5 KB
constexpr int STAGE_BYTES = 6 * A_BYTES + 2 * B_BYTES;  // 57 KB
// F16 interleaved hi|lo 128 B rows (SWIZZLE_128B): 3 A planes x 16 KB + 72 B rows
constexpr int A2_BYTES = BM * 128;
constexpr int BOX2_BYTES = BOX * 128;
static_assert(3 * A2_BYTES + 3 * BOX2_BYTES == STAGE_BYTES, "both formats stage 57 KB");
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr int TMEM_COLS = 512;
// warps 4.. are the epilogue: two per TMEM lane quarter, each finishing half
// of the 8-landmark column chunks, so the latency-bound fp64 Newton runs on
// two warps per SM sub-partition and the accumulator is released sooner
constexpr int EPI_WARPS = 8;
constexpr int NT = 32 * (4 + EPI_WARPS);
template <bool F16>
__host__ __device__ constexpr uint32_t idesc() {  // D = F32, A = B = TF32 (2) or F16 (0), K-major, N >> 3, M >> 4
  return (1u << 4) | ((F16 ? 0u : 2u) << 7) | ((F16 ? 0u : 2u) << 10) | ((uint32_t)(BN >> 3) << 17) |
         ((uint32_t)((2 * BM) >> 4) << 24);
}
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;  // clears the CTA-rank bit: the pair leader's smem window
}  // namespace g2

namespace {
__device__ __forceinline__ uint32_t s32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s32(b)), "r"(c));
}

// bounded wait: a protocol bug traps (clean context error) instead of hanging the GPU.
// CTA-scope acquire for barriers completed by TMA / tcgen05.commit (an
// .acquire.cluster poll invalidates the L1 on every try, CCTL.IVALL in SASS);
// cluster scope only where a peer thread's generic writes must be observed.
template <bool CLUSTER = false>
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t it = 0;; ++it) {
    if (CLUSTER)
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(s32(b)), "r"(parity)
          : "memory");
    else
      asm volatile(
          "{\n\t.reg .pred p;\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
          "selp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(done)
          : "r"(s32(b)), "r"(parity)
          : "memory");
    if (done) return;
    if (it > (1u << 28)) __trap();
  }
}

__device__ __forceinline__ void bar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s32(b)), "r"(bytes) : "memory");
}

// arrive on CTA `to`'s barrier at the same smem offset
__device__ __forceinline__ void bar_arrive_remote(uint64_t* b, uint32_t to) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(s32(b)), "r"(to));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

__device__ __forceinline__ void tma2_load(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];" ::"r"(s32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(s32(bar) & g2::PEER_MASK)
      : "memory");
}

__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

template <bool F16>
__device__ __forceinline__ void mma2(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  if (F16)
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(g2::idesc<true>()), "r"(acc));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(g2::idesc<false>()), "r"(acc));
}

__device__ __forceinline__ void commit2_both(uint64_t* bar) {
  const uint16_t mask = 0x3;
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          s32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void tmem_ld8_(uint32_t taddr, float v[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tile2_coords(int tile, int ntm, int ntl, int& tm, int& tl) {
  constexpr int GROUP_M = 2;
  const int gsize = GROUP_M * ntl;
  const int g = tile / gsize;
  const int r = tile - g * gsize;
  const int gm = min(GROUP_M, ntm - g * GROUP_M);
  tl = r / gm;
  tm = g * GROUP_M + (r - tl * gm);
}

}  // namespace

template <bool F16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(g2::NT, 1)
msd_tf32_2sm_kernel(const __grid_constant__ CUtensorMap mfh, const __grid_constant__ CUtensorMap mfl,
                    const __grid_constant__ CUtensorMap mlh, const __grid_constant__ CUtensorMap mll,
                    const double* __restrict__ gx, const double* __restrict__ ga, const double* __restrict__ fsc,
                    const double* __restrict__ lsc, int T, int L, int kpad, float* __restrict__ D, int64_t ldd) {
  using namespace g2;
  constexpr int KB = ROWB / (F16 ? 2 : 4);  // atoms per stage
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int ntm = (T + 2 * BM - 1) / (2 * BM), ntl = (L + BL - 1) / BL;
  const int ntiles = ntm * ntl;
  const int nkb = kpad / KB;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mfh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mfl)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mlh)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mll)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { bar_init(&full[s], 1); bar_init(&empty[s], 1); }
    bar_init(tfull, 1);
    bar_init(tempty, 2 * EPI_WARPS);  // epilogue warps of both CTAs (used on the leader)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(s32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cid; tile < ntiles; tile += ncl) {
        int tm, tl;
        tile2_coords(tile, ntm, ntl, tm, tl);
        const int t0 = tm * 2 * BM + (int)rank * BM, l0 = tl * BL;
        for (int kb = 0; kb < nkb; ++kb) {
          bar_wait(&empty[stage], phase ^ 1);
          uint8_t* st = smem + stage * STAGE_BYTES;
          if (rank == 0) bar_expect_tx(&full[stage], 2 * STAGE_BYTES);
          if constexpr (F16) {
            const int c0 = kb * 64;
#pragma unroll
            for (int p = 0; p < 3; ++p) tma2_load(&mfh, &full[stage], st + p * A2_BYTES, c0, p * T + t0);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
              const int r = (int)rank * BNH + q * BOX;
              const int g = r / BL, l = r - g * BL;
              tma2_load(&mlh, &full[stage], st + 3 * A2_BYTES + q * BOX2_BYTES, c0, g * L + l0 + l);
            }
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          const int k0 = kb * KB;
#pragma unroll
          for (int p = 0; p < 3; ++p) {
            tma2_load(&mfh, &full[stage], st + (2 * p) * A_BYTES, k0, p * T + t0);
            tma2_load(&mfl, &full[stage], st + (2 * p + 1) * A_BYTES, k0, p * T + t0);
          }
          uint8_t* bh = st + 6 * A_BYTES;
          uint8_t* bl = bh + B_BYTES;
          // rows of the stacked [g][l] operand held by this CTA: 72 rank..72 rank + 71
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const int r = (int)rank * BNH + q * BOX;  // row in [0, 144)
            const int g = r / BL, l = r - g * BL;
            tma2_load(&mlh, &full[stage], bh + q * BOX_BYTES, k0, g * L + l0 + l);
            tma2_load(&mll, &full[stage], bl + q * BOX_BYTES, k0, g * L + l0 + l);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = cid; tile < ntiles; tile += ncl, ++it) {
        bar_wait<true>(tempty, (it & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (int kb = 0; kb < nkb; ++kb) {
          bar_wait(&full[stage], phase);
          asm volatile("tcgen05.fence::after_thread_sync;");
          if (lane == 0) {
            const uint32_t st = s32(smem + stage * STAGE_BYTES);
            if constexpr (F16) {
              const uint32_t bb = st + 3 * A2_BYTES;
#pragma unroll
              for (int k = 0; k < 2; ++k) {
                const uint32_t koff = k * 32;
                const uint64_t dbh = desc_sw128(bb + koff);
                const uint64_t dbl = desc_sw128(bb + 64 + koff);
#pragma unroll
                for (int term = 0; term < 3; ++term) {
#pragma unroll
                  for (int p = 0; p < 3; ++p) {
                    const uint64_t a = desc_sw128(st + p * A2_BYTES + (term == 2 ? 64 : 0) + koff);
                    mma2<F16>(tmem_base + p * BN, a, term == 1 ? dbl : dbh, (term | kb | k) != 0 ? 1u : 0u);
                  }
                }
              }
            } else {
            const uint32_t bh = st + 6 * A_BYTES, bl = bh + B_BYTES;
#pragma unroll
            for (int k = 0; k < ROWB / 32; ++k) {
              const uint32_t koff = k * 32;
              const uint64_t dbh = desc_sw64(bh + koff);
              const uint64_t dbl = desc_sw64(bl + koff);
              // term-major: consecutive MMAs hit different accumulators
#pragma unroll
              for (int term = 0; term < 3; ++term) {
#pragma unroll
                for (int p = 0; p < 3; ++p) {
                  const uint32_t d = tmem_base + p * BN;
                  const uint64_t a = desc_sw64(st + (2 * p + (term == 2 ? 1 : 0)) * A_BYTES + koff);
                  mma2<F16>(d, a, term == 1 ? dbl : dbh, (term | kb | k) != 0 ? 1u : 0u);
                }
              }
            }
            }
            commit2_both(&empty[stage]);
            if (kb == nkb - 1) commit2_both(tfull);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int row = q * 32 + lane;
    int it = 0;
    for (int tile = cid; tile < ntiles; tile += ncl, ++it) {
      int tm, tl;
      tile2_coords(tile, ntm, ntl, tm, tl);
      const int t = tm * 2 * BM + (int)rank * BM + row;
      const int l0 = tl * BL;
      bar_wait(tfull, it & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const double gxt = t < T ? gx[t] : 0.0;
      const double fst = (F16 && t < T) ? fsc[t] : 1.0;
      const uint32_t lane_base = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = half; c < BL / 8; c += EPI_WARPS / 4) {
        float v[9][8];
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
          for (int g = 0; g < 3; ++g) tmem_ld8_(lane_base + p * BN + g * BL + c * 8, v[p * 3 + g]);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (t < T) {
          float out[8];
          msd8_estimate(v, gxt, ga, fst, F16 ? lsc : nullptr, l0 + c * 8, L, out);
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
      if (lane == 0) bar_arrive_remote(tempty, 0);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync();
  if (warp == 2) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(g2::TMEM_COLS));
  }
}

bool make_operand_map(CUtensorMap* m, const void* base, int esz, int64_t rows, int64_t row_elems, int box_rows,
                      bool sw128);

template <bool F16>
static cudaError_t launch_gemm2(const void* fh, const void* fl, const void* lh, const void* ll, const double* gx,
                                const double* ga, const double* fsc, const double* lsc, int T, int L, int kpad,
                                float* D, int64_t ldd, int grid, cudaStream_t stream) {
  using namespace g2;
  if (T <= 0 || L <= 0) return cudaSuccess;
  constexpr int esz = F16 ? 2 : 4;
  if (kpad % (ROWB / esz)) return cudaErrorInvalidValue;
  CUtensorMap mfh, mfl, mlh, mll;
  if (F16) {
    if (!make_operand_map(&mfh, fh, esz, 3LL * T, 2LL * kpad, BM, true) ||
        !make_operand_map(&mlh, lh, esz, 3LL * L, 2LL * kpad, BOX, true))
      return cudaErrorInvalidValue;
    mfl = mfh;
    mll = mlh;
  } else if (!make_operand_map(&mfh, fh, esz, 3LL * T, kpad, BM, false) ||
             !make_operand_map(&mfl, fl, esz, 3LL * T, kpad, BM, false) ||
             !make_operand_map(&mlh, lh, esz, 3LL * L, kpad, BOX, false) ||
             !make_operand_map(&mll, ll, esz, 3LL * L, kpad, BOX, false)) {
    return cudaErrorInvalidValue;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e =
        cudaFuncSetAttribute(msd_tf32_2sm_kernel<F16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int ntiles = ((T + 2 * BM - 1) / (2 * BM)) * ((L + BL - 1) / BL);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int clusters = grid > 0 ? grid / 2 : nsm / 2;
  if (clusters > ntiles) clusters = ntiles;
  if (clusters < 1) clusters = 1;
  msd_tf32_2sm_kernel<F16><<<2 * clusters, NT, SMEM_BYTES, stream>>>(mfh, mfl, mlh, mll, gx, ga, fsc, lsc, T, L,
                                                                     kpad, D, ldd);
  return cudaGetLastError();
}

cudaError_t launch_msd_tf32_2sm(const float* fh, const float* fl, const float* lh, const float* ll, const double* gx,
                                const double* ga, int T, int L, int kpad, float* D, int64_t ldd, int grid,
                                cudaStream_t stream) {
  return launch_gemm2<false>(fh, fl, lh, ll, gx, ga, nullptr, nullptr, T, L, kpad, D, ldd, grid, stream);
}

cudaError_t launch_msd_f16_2sm(const void* fhl, const void* lhl, const double* fsc, const double* lsc,
                               const double* gx, const double* ga, int T, int L, int kpad, float* D, int64_t ldd,
                               int grid, cudaStream_t stream) {
  return launch_gemm2<true>(fhl, nullptr, lhl, nullptr, gx, ga, fsc, lsc, T, L, kpad, D, ldd, grid, stream);
}

}  // namespace mc
