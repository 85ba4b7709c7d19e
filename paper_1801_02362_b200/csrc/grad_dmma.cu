// K4 gradient pass of the fp32-coordinate path on the fp64 tensor cores.
//
// Same result as cv_grad_block_kernel<OT, false> (grad_block.cu):
//   ds_t,k = 2 w_k (sum_i cs_i x_k - U^s_k) - w'_k corr^s_t,
//   U^s_k  = sum_{i in sig(t)} (cs_i Rhat_i) a_{i,k}          (same for z),
// but the contraction U is issued as a real fp64 GEMM on DMMA
// (mma.sync m8n8k4 f64, exact fp64 products and sums):
//   C[r, k] = sum_kk A[r, kk] B[kk, k],   r = (frame f, s|z, axis b)  (48 rows
//   for a group of 8 sorted frames), kk = (landmark l - wlo, axis g) over the
//   group's window union, B[kk, k] = centred landmark coordinate a_{l,k,g}.
// The vector kernel re-reads all 18 coefficients of a (frame, landmark) from
// shared memory for every atom; here one A fragment (1 double per lane) feeds
// 4 DMMAs and one B fragment 6, so the fp64 pipe rather than shared memory
// sets the pace.  Coefficients are staged once per CTA (all atoms of a group when
// there are enough groups); the raw fp32 landmark coordinates stream through a
// 3-stage ring of 1-D TMA bulk copies (8 landmarks x 256 atoms per stage) and are
// converted when a B fragment is read (once per 6 DMMAs).  B holds raw, not
// centred, coordinates: the centroid term sum_kk A[r, kk] lc[kk] is one scalar
// per GEMM row, subtracted in the epilogue (no fp64 add beside the DMMAs).
#include <algorithm>
#include <type_traits>

#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int DG = 8;              // frames per group
constexpr int DR = 6 * DG;         // 48 GEMM rows
constexpr int DWMAX = 96;          // landmarks per staged window chunk
constexpr int DKMAX = 3 * DWMAX;   // 288 kk columns
constexpr int AST = 292;           // sA row stride (doubles): 4 mod 16 -> conflict-free 8x4 fragments
constexpr int DNA = 256;           // atoms per sub-tile (8 warps x 32)
constexpr int DKC = 24;            // kk rows per B chunk (8 landmarks)
constexpr int LROW = 3 * DNA + 8;  // raw floats per staged landmark row (+8: bank shift between landmarks)
constexpr int NST = 3;             // cp.async ring stages
constexpr int MAXWC = 127;         // window chunks with per-chunk list ranges (union <= 12192 landmarks)
#ifndef MC_GD_WAT
#define MC_GD_WAT 16
#endif
constexpr int WAT = MC_GD_WAT;     // atoms per warp (n-tiles of 8)
constexpr int NJ = WAT / 8;
constexpr int DNT = 32 * (DNA / WAT);  // 16 warps: more warps in flight to hide the fragment-load latency
constexpr int CHL = DKC / 3;       // landmarks per chunk
constexpr int LPT = CHL * DNA * 3 / DNT;  // raw floats per thread per chunk
constexpr int XPT = DG * DNA * 3 / DNT;  // frame floats per thread per sub-tile
constexpr int DSMEM = DR * AST * (int)sizeof(double) + DKMAX * (int)sizeof(double) +
                      NST * CHL * LROW * (int)sizeof(float) + DG * 3 * DNA * (int)sizeof(float) +
                      2 * DNA * (int)sizeof(double) + (2 * NST + 1) * (int)sizeof(uint64_t);

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d), "l"(src), "r"(ok ? 4 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(c));
}
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
          smem_addr(b)),
      "r"(parity)
      : "memory");
}
// 1-D bulk copy global -> shared completing on an mbarrier (TMA engine)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
}  // namespace

__device__ __forceinline__ void cp_async16(float* dst, const float* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

// VEC: N % 4 == 0 and 16-byte aligned inputs -> 16-byte copies of whole float4
// (3 * (atoms) floats per row chunk is then a multiple of 4 at every boundary)
template <typename OT, bool VEC>
__global__ void __launch_bounds__(DNT, 1)
cv_grad_dmma_kernel(int T, int n, int cap, const float* __restrict__ fraw, const double* __restrict__ fcen,
                    const float* __restrict__ lraw, const double* __restrict__ lcen, const double* __restrict__ w,
                    const double* __restrict__ wa, const int* __restrict__ sig_idx,
                    const double* __restrict__ sig_coef, const int* __restrict__ nsig,
                    const double* __restrict__ fvec, const int* __restrict__ perm, const int* __restrict__ out_map,
                    OT* __restrict__ ds, OT* __restrict__ dz, int apb, int min_width, int i8_dg) {
  extern __shared__ __align__(16) double dsm[];
  double* sA = dsm;                                       // [DR][AST] coefficients
  double* sLc = dsm + DR * AST;                           // [DKMAX] landmark centroid per kk
  float* sR = reinterpret_cast<float*>(sLc + DKMAX);      // [NST][CHL][LROW] raw landmark floats
  float* sX = sR + NST * CHL * LROW;                      // [DG][3 DNA] raw frame floats of the sub-tile
  // VEC: warp-decoupled ring -- thread 0 issues 1-D TMA bulk copies completing on
  // full[slot]; each warp releases a slot on empty[slot]; no CTA barrier per chunk
  double* sWW = reinterpret_cast<double*>(sX + DG * 3 * DNA);  // VEC: [2][DNA] w, w_align of the sub-tile
  uint64_t* full = reinterpret_cast<uint64_t*>(sWW + 2 * DNA);
  uint64_t* empty = full + NST;
  uint64_t* xfull = empty + NST;
  __shared__ int s_t[DG], s_raw[DG], s_ns[DG], s_flo[DG], s_fhi[DG], s_mine[DG];
  __shared__ double s_fc[DG][3], s_fv[DG][8];
  __shared__ int s_wlo, s_whi;
  __shared__ double s_bias[DR];
  __shared__ double s_rcx[DR], s_rsc[DR], s_rcorr[DR];
  __shared__ unsigned long long s_rptr[DR];
  __shared__ int s_rx[DR];
  __shared__ int s_cum[DG + 1];
  // s_beg[f][c]: first position of frame f's (ascending) significant list inside
  // window chunk c = [wlo + c DWMAX, ..); a restage reads only its chunk's entries
  __shared__ int s_beg[DG][MAXWC + 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gq = lane >> 2, tq = lane & 3;  // mma groupID / threadID_in_group
  if (tid < DG) {
    const int k = blockIdx.x * DG + tid;
    int t = -1, ns = 0;
    if (k < T) {
      t = perm ? perm[k] : k;
      ns = nsig[t];
    }
    s_t[tid] = t;
    s_raw[tid] = (t >= 0 && out_map) ? out_map[t] : t;  // caller's row: raw coordinates and gradients
    s_ns[tid] = ns;
    s_flo[tid] = (t >= 0 && ns > 0) ? sig_idx[(int64_t)t * cap] : 0x7fffffff;
    s_fhi[tid] = (t >= 0 && ns > 0) ? sig_idx[(int64_t)t * cap + ns - 1] + 1 : -1;
    // min_width >= 0: this call completes only the frames of the int8 kernel's WIDE groups
    // (i8_dg sorted frames each, union wider than min_width landmarks; grad_i8.cu did the rest)
    int mine = 1;
    if (min_width >= 0 && k < T) {
      const int k0 = (k / i8_dg) * i8_dg, k1 = min(T, k0 + i8_dg);
      int a = 0x7fffffff, b = -1;
      for (int kk = k0; kk < k1; ++kk) {
        const int tt = perm ? perm[kk] : kk;
        const int nn = nsig[tt];
        if (nn <= 0) continue;
        a = min(a, sig_idx[(int64_t)tt * cap]);
        b = max(b, sig_idx[(int64_t)tt * cap + nn - 1] + 1);
      }
      mine = b >= 0 && b - a > min_width;
    }
    s_mine[tid] = mine;
    if (t >= 0) {
      for (int a = 0; a < 3; ++a) s_fc[tid][a] = fcen[3 * t + a];
      const double* fv = fvec + (int64_t)t * 16;
      for (int e = 0; e < 8; ++e) s_fv[tid][e] = fv[e];  // sumcs, sumcz, corr_s[3], corr_z[3]
    }
  }
  __syncthreads();
  if (tid < DR) {  // epilogue row table: r = (frame f, s|z, axis b)
    const int f = tid / 6, sz = (tid % 6) / 3, b = tid % 3;
    const int t = s_t[f];
    s_rptr[tid] = (t < 0 || !s_mine[f])
                      ? 0ull
                      : reinterpret_cast<unsigned long long>((sz ? dz : ds) + (int64_t)s_raw[f] * n * 3 + b);
    s_rcx[tid] = t < 0 ? 0.0 : s_fc[f][b];
    s_rsc[tid] = t < 0 ? 0.0 : s_fv[f][sz];
    s_rcorr[tid] = t < 0 ? 0.0 : s_fv[f][2 + sz * 3 + b];
    s_rx[tid] = f * 3 * DNA + b;
    s_bias[tid] = 0.0;  // stays 0 when the group has no significant landmark (sharded: empty windows)
  }
  if (tid == 0) {
    int a = 0x7fffffff, b = -1, any = 0;
    for (int f = 0; f < DG; ++f) {
      a = min(a, s_flo[f]);
      b = max(b, s_fhi[f]);
      any |= s_mine[f] && s_t[f] >= 0;
    }
    s_wlo = a;
    s_whi = any ? b : -1;  // no frame of this call here: nothing to write
  }
  if (VEC) {
    if (tid == 0) {
      for (int i = 0; i < NST; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], DNT / 32); }
      mb_init(xfull, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // stale ring rows are multiplied by zero coefficients: make them finite once
    for (int e = tid; e < NST * CHL * LROW; e += DNT) sR[e] = 0.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const int wlo = s_wlo, whi = s_whi;
  // no significant landmark in the whole group (landmark-sharded evaluation: frames whose
  // window lies on other shards): nothing to contract and nothing to write -- those rows
  // belong to (and are completed by) other ranks
  if (whi < 0) return;

  const bool restage = whi - wlo > DWMAX;
  const int nwc = whi > wlo ? (whi - wlo + DWMAX - 1) / DWMAX : 0;
  const bool ranged = nwc <= MAXWC;  // else: each restage filters the whole list
  if (ranged) {
    for (int i = tid; i < DG * (MAXWC + 1); i += DNT) (&s_beg[0][0])[i] = 0;
    __syncthreads();
    for (int f = 0; f < DG; ++f) {
      const int t = s_t[f], ns = s_ns[f];
      if (t < 0 || ns <= 0) continue;  // block-uniform
      const int* idx = sig_idx + (int64_t)t * cap;
      for (int e = tid; e < ns; e += DNT) {
        const int c = (idx[e] - wlo) / DWMAX;
        const int cprev = e == 0 ? -1 : (idx[e - 1] - wlo) / DWMAX;
        for (int q = cprev + 1; q <= c; ++q) s_beg[f][q] = e;
        if (e == ns - 1)
          for (int q = c + 1; q <= nwc; ++q) s_beg[f][q] = ns;
      }
    }
    __syncthreads();
  }
  uint32_t gch = 0, xphase = 0;  // VEC: chunks consumed by this CTA (ring position / parity)
  bool staged = false;
  const int katom0 = blockIdx.y * apb;
  const int katom1 = min(n, katom0 + apb);
  // VEC producer (thread 0): walks the chunk sequence (atom sub-tile a0, window
  // chunk w0, landmark chunk ch) in consumption order, up to NST - 1 chunks ahead,
  // across w0 and a0 boundaries -- the next block's first chunks are in flight
  // during this block's epilogue or coefficient restaging.
  int pa0 = katom0, pch = 0, pw0 = wlo, pwn = min(DWMAX, whi - wlo);
  uint32_t gprod = 0, plimit = 0;
  auto produce_next = [&]() {
    const uint32_t g = gprod++;
    const int slot = (int)(g % NST);
    if (g >= (uint32_t)NST) mb_wait(&empty[slot], ((g / NST) - 1) & 1u);
    const int natp = min(DNA, n - pa0);
    const int q1 = min(CHL, pwn - pch * CHL);
    mb_expect(&full[slot], (uint32_t)(q1 * 12 * natp));
    float* dst = sR + slot * CHL * LROW;
    for (int q = 0; q < q1; ++q)
      bulk_g2s(dst + q * LROW, lraw + ((int64_t)(pw0 + pch * CHL + q) * n + pa0) * 3, 12 * natp, &full[slot]);
    if (++pch * CHL >= pwn) {
      pch = 0;
      pw0 += DWMAX;
      if (pw0 >= whi) {
        pw0 = wlo;
        pa0 += DNA;
      }
      pwn = min(DWMAX, whi - pw0);
    }
  };
  if (VEC && tid == 0 && whi > wlo) {
    uint32_t per_a0 = 0;
    for (int w0 = wlo; w0 < whi; w0 += DWMAX) per_a0 += (uint32_t)((3 * min(DWMAX, whi - w0) + DKC - 1) / DKC);
    plimit = (uint32_t)((katom1 - katom0 + DNA - 1) / DNA) * per_a0;
    while (gprod < plimit && gprod < (uint32_t)(NST - 1)) produce_next();
  }
  for (int a0 = katom0; a0 < katom1; a0 += DNA) {
    // the epilogue's frame coordinates: issued now, long complete by the time
    // the contraction below has finished
    const int nat = min(DNA, n - a0);  // valid atoms of this sub-tile
    if (VEC) {
      if (tid == 0) {
        int rows = 0;
        for (int f = 0; f < DG; ++f) rows += s_raw[f] >= 0;
        mb_expect(xfull, (uint32_t)(rows * 12 * nat + 16 * nat));
        for (int f = 0; f < DG; ++f)
          if (s_raw[f] >= 0) bulk_g2s(sX + f * 3 * DNA, fraw + ((int64_t)s_raw[f] * n + a0) * 3, 12 * nat, xfull);
        // the epilogue's atom weights ride on the same barrier (no global loads there)
        bulk_g2s(sWW, w + a0, 8 * nat, xfull);
        bulk_g2s(sWW + DNA, wa + a0, 8 * nat, xfull);
      }
    } else {
#pragma unroll 4
      for (int u = 0; u < XPT; ++u) {
        const int e = tid + u * DNT;  // [0, DG * 3 DNA)
        const int f = e / (3 * DNA), r = e - f * (3 * DNA);
        const int t = s_raw[f];
        const bool ok = t >= 0 && a0 + r / 3 < n;
        cp_async4(sX + e, fraw + ((int64_t)(ok ? t : 0) * n + (ok ? a0 : 0)) * 3 + (ok ? r : 0), ok);
      }
    }
    if (!VEC) cp_commit();
    double c[6][NJ][2];
#pragma unroll
    for (int m = 0; m < 6; ++m)
#pragma unroll
      for (int j = 0; j < NJ; ++j) c[m][j][0] = c[m][j][1] = 0.0;
    for (int w0 = wlo; w0 < whi; w0 += DWMAX) {
      const int wn = min(DWMAX, whi - w0);
      const int nch = (3 * wn + DKC - 1) / DKC;
      if (restage || !staged) {  // block-uniform
        staged = true;
        __syncthreads();
        for (int e = tid; e < DR * AST; e += DNT) sA[e] = 0.0;
        for (int e = tid; e < DKMAX; e += DNT) sLc[e] = e < 3 * wn ? lcen[3 * w0 + e] : 0.0;
        __syncthreads();
        // coefficient scatter of this window chunk, all frames at once (independent
        // loads in flight); entries of the chunk only when the list ranges are known
        const int wc = (w0 - wlo) / DWMAX;
        if (tid == 0) {
          int tot = 0;
          for (int f = 0; f < DG; ++f) {
            s_cum[f] = tot;
            if (s_t[f] >= 0) tot += 18 * (ranged ? s_beg[f][wc + 1] - s_beg[f][wc] : s_ns[f]);
          }
          s_cum[DG] = tot;
        }
        __syncthreads();
        const int tot = s_cum[DG];
#pragma unroll 4
        for (int e = tid; e < tot; e += DNT) {
          int f = 0;
#pragma unroll
          for (int q = 1; q < DG; ++q) f += e >= s_cum[q];
          const int t = s_t[f], el = e - s_cum[f];
          const int s = el / 18 + (ranged ? s_beg[f][wc] : 0), e18 = el % 18;
          const int l = sig_idx[(int64_t)t * cap + s] - w0;
          const double v = sig_coef[((int64_t)t * cap + s) * 18 + e18];
          if (l >= 0 && l < wn) {
            const int sz = e18 / 9, b = (e18 % 9) / 3, g = e18 % 3;
            sA[(f * 6 + sz * 3 + b) * AST + l * 3 + g] = v;
          }
        }
        __syncthreads();
        // centroid term of the contraction (B holds raw coordinates):
        // bias_r = sum_kk A[r, kk] lc[kk], subtracted in the epilogue
        for (int r = warp; r < DR; r += DNT / 32) {
          double acc = 0.0;
          for (int kk = lane; kk < 3 * wn; kk += 32) acc += sA[r * AST + kk] * sLc[kk];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (lane == 0) s_bias[r] = (w0 == wlo ? 0.0 : s_bias[r]) + acc;
        }
      }
      // loop-invariant fragment offsets: B element (kk = 4 s + tq -> landmark q, axis g)
      int offB[DKC / 4];
#pragma unroll
      for (int s = 0; s < DKC / 4; ++s) {
        const int kc = s * 4 + tq;
        offB[s] = (kc / 3) * LROW + (warp * WAT + gq) * 3 + kc % 3;
      }
      const double* aRow = sA + gq * AST + tq;
      if constexpr (VEC) {
        const bool wact = a0 + warp * WAT < n;
        for (int ch = 0; ch < nch; ++ch) {
          const uint32_t g = gch + (uint32_t)ch;
          if (tid == 0)
            while (gprod < plimit && gprod < g + (uint32_t)NST) produce_next();
          const int slot = (int)(g % NST);
          mb_wait(&full[slot], (g / NST) & 1u);
          const float* rb = sR + slot * CHL * LROW;
          const double* ak = aRow + ch * DKC;
          // KS k-steps of 4 kk; full chunks take the KS = 6 path, a partial last
          // chunk only the k-steps that hold window landmarks
          auto contract = [&](auto ks) {
            constexpr int KS = decltype(ks)::value;
#pragma unroll
            for (int s = 0; s < KS; ++s) {
              double a[6], b[NJ];
#pragma unroll
              for (int m = 0; m < 6; ++m) a[m] = ak[m * 8 * AST + 4 * s];
#pragma unroll
              for (int j = 0; j < NJ; ++j) b[j] = (double)rb[offB[s] + j * 24];
#pragma unroll
              for (int m = 0; m < 6; ++m)
#pragma unroll
                for (int j = 0; j < NJ; ++j) dmma(c[m][j], a[m], b[j]);
            }
          };
          // warps whose atoms all lie past n skip the contraction
          const int ksteps = wact ? (3 * min(CHL, wn - ch * CHL) + 3) / 4 : 0;
          static_assert(DKC / 4 == 6, "k-step dispatch below assumes 6 k-steps per chunk");
          switch (ksteps) {
            case 6: contract(std::integral_constant<int, 6>{}); break;
            case 5: contract(std::integral_constant<int, 5>{}); break;
            case 4: contract(std::integral_constant<int, 4>{}); break;
            case 3: contract(std::integral_constant<int, 3>{}); break;
            case 2: contract(std::integral_constant<int, 2>{}); break;
            case 1: contract(std::integral_constant<int, 1>{}); break;
            default: break;
          }
          __syncwarp();
          if (lane == 0) mb_arrive(&empty[slot]);
        }
        gch += (uint32_t)nch;
        __syncthreads();  // sA may be restaged for the next window chunk
        continue;
      }
      // stage chunk ch (landmarks w0 + CHL ch .., atoms a0 .. a0 + DNA) into ring slot `slot`;
      // out-of-range elements are zero-filled (their coefficients are zero too)
      auto issue = [&](int ch, int slot) {
        float* dst = sR + slot * CHL * LROW;
#pragma unroll 4
        for (int u = 0; u < LPT; ++u) {
          const int e = tid + u * DNT;  // [0, CHL * 3 DNA)
          const int q = e / (3 * DNA), r = e - q * (3 * DNA);
          const int li = w0 + ch * CHL + q;
          const bool ok = ch < nch && li < w0 + wn && a0 + r / 3 < n;
          cp_async4(dst + q * LROW + r, lraw + ((int64_t)(ok ? li : 0) * n + (ok ? a0 : 0)) * 3 + (ok ? r : 0), ok);
        }
        cp_commit();
      };
#pragma unroll
      for (int st = 0; st < NST - 1; ++st) issue(st, st);
      int slot = 0, fill = NST - 1;
      for (int ch = 0; ch < nch; ++ch) {
        cp_wait<NST - 2>();
        __syncthreads();
        issue(ch + NST - 1, fill);
        fill = fill + 1 == NST ? 0 : fill + 1;
        const float* rb = sR + slot * CHL * LROW;
        const double* ak = aRow + ch * DKC;
#pragma unroll
        for (int s = 0; s < DKC / 4; ++s) {
          double a[6], b[NJ];
#pragma unroll
          for (int m = 0; m < 6; ++m) a[m] = ak[m * 8 * AST + 4 * s];
#pragma unroll
          for (int j = 0; j < NJ; ++j) b[j] = (double)rb[offB[s] + j * 24];
#pragma unroll
          for (int m = 0; m < 6; ++m)
#pragma unroll
            for (int j = 0; j < NJ; ++j) dmma(c[m][j], a[m], b[j]);
        }
        slot = slot + 1 == NST ? 0 : slot + 1;
      }
      cp_wait<0>();
      __syncthreads();
    }
    // epilogue: each accumulator element is one (frame, s|z, axis, atom) output.
    // Loads of a half (3 row tiles x 8 atoms) are batched ahead of its stores.
    double wk[NJ][2], wak[NJ][2];
    if (VEC) {
      mb_wait(xfull, xphase);
      xphase ^= 1u;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int al = warp * WAT + j * 8 + 2 * tq + e;
          wk[j][e] = a0 + al < n ? sWW[al] : 0.0;
          wak[j][e] = a0 + al < n ? sWW[DNA + al] : 0.0;
        }
    } else {
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int k = a0 + warp * WAT + j * 8 + 2 * tq + e;
          wk[j][e] = k < n ? w[k] : 0.0;
          wak[j][e] = k < n ? wa[k] : 0.0;
        }
      cp_wait<0>();
      __syncthreads();
    }
    // per GEMM row r: output row pointer (ds or dz of frame f, axis b; null for an
    // absent frame), centroid, sums and the sX offset, tabulated once per CTA
    const bool full = a0 + DNA <= n;  // block-uniform: no per-atom bound checks
#pragma unroll
    for (int m = 0; m < 6; ++m) {
      const int r = m * 8 + gq;
      OT* __restrict__ rp = reinterpret_cast<OT*>(s_rptr[r]);
      if (!rp) continue;
      const double cx = s_rcx[r], sc = s_rsc[r], corr = s_rcorr[r], bias = s_bias[r];
      const float* xs = sX + s_rx[r];
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int al = warp * WAT + j * 8 + 2 * tq + e;
          if (!full && a0 + al >= n) continue;
          const double x = (double)xs[3 * al] - cx;
          rp[(int64_t)(a0 + al) * 3] = (OT)(2.0 * wk[j][e] * (sc * x - (c[m][j][e] - bias)) - wak[j][e] * corr);
        }
    }
    __syncthreads();  // sX is refilled by the next sub-tile
  }
}

cudaError_t launch_cv_grad_dmma(int T, int n, int cap, const float* fraw, const double* fcen, const float* lraw,
                                const double* lcen, const double* w, const double* wa, const int* sig_idx,
                                const double* sig_coef, const int* nsig, const double* fvec, const int* perm,
                                const int* out_map, void* ds, void* dz, int out_f32, cudaStream_t stream,
                                int min_width, int i8_dg) {
  if (T <= 0 || n <= 0) return cudaSuccess;
  // atoms per CTA: all of them when there are enough frame groups to fill the
  // machine (the coefficient staging is then paid once per group), else split
  // the atoms over grid.y until ~4 CTAs per SM exist
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int groups = (T + DG - 1) / DG;
  const int tiles = (n + DNA - 1) / DNA;
  const int nyb = std::max(1, std::min(tiles, (4 * sms + groups - 1) / groups));
  const int apb = ((tiles + nyb - 1) / nyb) * DNA;
  dim3 grid(groups, (n + apb - 1) / apb);
  static bool attr = false;
  if (!attr) {
    for (const void* fn : {(const void*)cv_grad_dmma_kernel<float, true>, (const void*)cv_grad_dmma_kernel<float, false>,
                           (const void*)cv_grad_dmma_kernel<double, true>, (const void*)cv_grad_dmma_kernel<double, false>}) {
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, DSMEM);
      if (e != cudaSuccess) return e;
    }
    attr = true;
  }
  const bool vec = n % 4 == 0 && (reinterpret_cast<uintptr_t>(fraw) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(lraw) & 15) == 0;
#define MC_GD_LAUNCH(OTT, V)                                                                                         \
  cv_grad_dmma_kernel<OTT, V><<<grid, DNT, DSMEM, stream>>>(T, n, cap, fraw, fcen, lraw, lcen, w, wa, sig_idx,     \
                                                            sig_coef, nsig, fvec, perm, out_map, (OTT*)ds,     \
                                                            (OTT*)dz, apb, min_width, i8_dg > 0 ? i8_dg : DG)
  if (out_f32) {
    if (vec) MC_GD_LAUNCH(float, true); else MC_GD_LAUNCH(float, false);
  } else {
    if (vec) MC_GD_LAUNCH(double, true); else MC_GD_LAUNCH(double, false);
  }
#undef MC_GD_LAUNCH
  return cudaGetLastError();
}

}  // namespace mc
