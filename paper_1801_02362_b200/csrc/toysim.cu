// Toy MD driver on the device (SPEC [MODULE] toysim): overdamped
// Langevin (Euler-Maruyama) on a bead chain, the path CV s (and z) evaluated every
// step in the original mode (Alg. 1: exact fits to every reference) or the
// close-structure mode (Alg. 2: one exact x<->y fit per step, the reference set
// refitted only when D(x, y) > eps, Eq. 5/6 otherwise), metadynamics hills on s
// (Eq. 1, direct summation), and the bias force -dV/ds ds/dx.
//
// B200 design: the whole trajectory runs inside ONE launch, one CTA per walker
// (independent walkers = independent CTAs, no inter-CTA traffic); the walker's
// state (positions, close structure, saved rotations, hills, counters) lives in
// shared memory / registers for all steps and is written back at the end, so a
// step costs no launch and no host round trip (the sequential chain of a toy MD
// is latency-bound; a launch per step would cost more than the step).  Chunked
// runs (step0 > 0) continue from the state arrays.  Every reduction runs in a
// fixed order (warp 0 shuffles, per-bead force terms summed in a fixed order), so
// identical seeds give bit-identical runs.
//
// Fits mirror the reference kearsley_fit (geometry.py:227-263): the 4x4 Kearsley
// matrix from S and its cyclic Jacobi spectrum (geometry.py:106-153); the Eq. 6
// dR_xy term uses the contracted closed form of pathcv.cu (dk_contract).
//
// Random numbers: Philox4x32-10 keyed by the run seed, counter (bead, step lo,
// step hi, walker); three normals per bead and step by Box-Muller (the oracle,
// oracle/toysim.py, draws the identical integers).
#include "launch.h"
#include "mc_math.cuh"

namespace mc {

namespace {
constexpr int TNT = 128;
constexpr int TMAXN = 64;
constexpr int TMAXL = 128;
}  // namespace

__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c[0], hi0 = __umulhi(0xD2511F53u, c[0]);
    const uint32_t lo1 = 0xCD9E8D57u * c[2], hi1 = __umulhi(0xCD9E8D57u, c[2]);
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

// three N(0, 1) numbers for (walker, step, bead)
__device__ __forceinline__ void toy_normals(unsigned long long seed, int walker, long long step, int bead, double z[3]) {
  uint32_t c[4] = {(uint32_t)bead, (uint32_t)(step & 0xffffffffLL), (uint32_t)((unsigned long long)step >> 32),
                   (uint32_t)walker};
  philox4x32_10(c, (uint32_t)(seed & 0xffffffffULL), (uint32_t)(seed >> 32));
  const double s32 = 2.3283064365386963e-10;  // 2^-32
  const double u0 = ((double)c[0] + 0.5) * s32, u1 = ((double)c[1] + 0.5) * s32;
  const double u2 = ((double)c[2] + 0.5) * s32, u3 = ((double)c[3] + 0.5) * s32;
  const double twopi = 6.283185307179586;
  const double r0 = sqrt(-2.0 * log(u0)), r1 = sqrt(-2.0 * log(u2));
  z[0] = r0 * cos(twopi * u1);
  z[1] = r0 * sin(twopi * u1);
  z[2] = r1 * cos(twopi * u3);
}

// bonded force on bead k (harmonic bonds, harmonic angles in theta); terms in a fixed
// order: bond (k-1,k), bond (k,k+1), angles with vertex k-1, k, k+1
__device__ void toy_bonded_force(const double* x, int n, int k, const ToyParams& P, double F[3]) {
  F[0] = F[1] = F[2] = 0.0;
  auto bond = [&](int i, int j) {  // force on i from bond (i, j): +k (d - r0) r / d, r = x_j - x_i
    const double r[3] = {x[3 * j] - x[3 * i], x[3 * j + 1] - x[3 * i + 1], x[3 * j + 2] - x[3 * i + 2]};
    const double d = sqrt(r[0] * r[0] + r[1] * r[1] + r[2] * r[2]);
    const double f = P.bond_k * (d - P.bond_r0) / d;
    F[0] += f * r[0];
    F[1] += f * r[1];
    F[2] += f * r[2];
  };
  if (k > 0) bond(k, k - 1);
  if (k + 1 < n) bond(k, k + 1);
  // angle (a, v, b) with vertex v: force on `who` (0: end a, 1: vertex, 2: end b)
  auto angle = [&](int v, int who) {
    const int a = v - 1, b = v + 1;
    const double u[3] = {x[3 * a] - x[3 * v], x[3 * a + 1] - x[3 * v + 1], x[3 * a + 2] - x[3 * v + 2]};
    const double w[3] = {x[3 * b] - x[3 * v], x[3 * b + 1] - x[3 * v + 1], x[3 * b + 2] - x[3 * v + 2]};
    const double nu = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
    const double nw = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    double c = (u[0] * w[0] + u[1] * w[1] + u[2] * w[2]) / (nu * nw);
    c = fmin(1.0, fmax(-1.0, c));
    const double th = acos(c);
    const double sn = fmax(sqrt(fmax(0.0, 1.0 - c * c)), 1e-12);
    const double pre = P.angle_k * (th - P.theta0) / sn;  // F_end = pre * dcos/d(end)
    double fa[3], fb[3];
#pragma unroll
    for (int e = 0; e < 3; ++e) {
      fa[e] = pre * (w[e] / (nu * nw) - c * u[e] / (nu * nu));
      fb[e] = pre * (u[e] / (nu * nw) - c * w[e] / (nw * nw));
    }
#pragma unroll
    for (int e = 0; e < 3; ++e) F[e] += who == 0 ? fa[e] : (who == 2 ? fb[e] : -(fa[e] + fb[e]));
  };
  if (k - 1 >= 1 && k - 1 <= n - 2) angle(k - 1, 2);
  if (k >= 1 && k <= n - 2) angle(k, 1);
  if (k + 1 >= 1 && k + 1 <= n - 2) angle(k + 1, 0);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void __launch_bounds__(TNT, 3)
toysim_kernel(ToyParams P, const double* __restrict__ refs, const double* __restrict__ refg,
              const double* __restrict__ refmom, const double* __restrict__ q, const double* __restrict__ w,
              const double* __restrict__ wa, double* __restrict__ xs, double* __restrict__ ys,
              double* __restrict__ rays, int* __restrict__ hasy, double* __restrict__ hills,
              int* __restrict__ nhills, long long* __restrict__ counters, double* __restrict__ cv,
              uint8_t* __restrict__ rlog, double* __restrict__ traj, uint8_t* __restrict__ flags,
              uint8_t* __restrict__ act, long long* __restrict__ nl_last) {
  const int wk = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = P.n, L = P.L;
  __shared__ double sx[TMAXN * 3], sxn[TMAXN * 3], sxc[TMAXN * 3], sy[TMAXN * 3], sg[2][TMAXN * 3];
  __shared__ double sw[TMAXN], swa[TMAXN];
  __shared__ double sRay[TMAXL * 9], sRh[TMAXL * 9], sS[TMAXL * 9], sD[TMAXL], scs[TMAXL], scz[TMAXL];
  extern __shared__ double sPart[];  // [L + 1][36]: per-reference Eq. 6 terms, then their sums
  __shared__ double s_gx, s_dxy, s_rxy[9], s_eig[4], s_V[16], s_v[2][4], s_sum[2], s_gsum[6];
  __shared__ double s_s, s_z, s_bias, s_dvds;
  __shared__ int s_refresh, s_hasy, s_nh;
  // neighbour list (SPEC neighbourlist): the members (s_act), the last update step
  __shared__ uint8_t s_act[TMAXL];
  __shared__ long long s_nl_last;
  const bool nl = P.nl_m > 0;
  __shared__ unsigned s_flags;
  for (int e = tid; e < 3 * n; e += TNT) {
    sx[e] = xs[(int64_t)wk * 3 * n + e];
    sy[e] = ys[(int64_t)wk * 3 * n + e];
  }
  for (int j = tid; j < n; j += TNT) { sw[j] = w[j]; swa[j] = wa[j]; }
  if (P.mode == 2)
    for (int e = tid; e < 9 * L; e += TNT) sRay[e] = rays[(int64_t)wk * 9 * L + e];
  if (nl)
    for (int i = tid; i < L; i += TNT) s_act[i] = act[(int64_t)wk * L + i];
  if (tid == 0) {
    s_nl_last = nl ? nl_last[wk] : -1;
    s_hasy = hasy[wk];
    s_nh = nhills[wk];
    s_flags = 0u;
  }
  long long c_exp = 0, c_cheap = 0, c_reas = 0;
  __syncthreads();
  for (int it = 0; it < P.steps; ++it) {
    const long long t = P.step0 + it;
    if (P.traj_stride > 0 && t % P.traj_stride == 0) {
      const int64_t slot = (int64_t)(it / P.traj_stride);
      const int64_t nsl = (P.steps + P.traj_stride - 1) / P.traj_stride;
      for (int e = tid; e < 3 * n; e += TNT) traj[((int64_t)wk * nsl + slot) * 3 * n + e] = sx[e];
    }
    if (P.mode != 0) {
      // A: centre (alignment-weighted centroid, geometry.py:67-76), Gx
      if (warp == 0) {
        double c[3] = {0.0, 0.0, 0.0};
        for (int j = lane; j < n; j += 32)
#pragma unroll
          for (int a = 0; a < 3; ++a) c[a] = fma(swa[j], sx[3 * j + a], c[a]);
#pragma unroll
        for (int a = 0; a < 3; ++a) c[a] = warp_sum_d(c[a]);
        double g = 0.0;
        for (int j = lane; j < n; j += 32) {
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            const double v = sx[3 * j + a] - c[a];
            sxc[3 * j + a] = v;
            g = fma(sw[j] * v, v, g);
          }
        }
        g = warp_sum_d(g);
        if (lane == 0) s_gx = g;
      }
      __syncthreads();
      // B: the x<->y fit (close mode; Alg. 2 lines 2-4), refresh decision (strict '>')
      if (P.mode == 2) {
        if (s_hasy) {
          if (warp == 0) {
            double S[9], gy = 0.0;
#pragma unroll
            for (int e = 0; e < 9; ++e) S[e] = 0.0;
            for (int j = lane; j < n; j += 32) {
#pragma unroll
              for (int b = 0; b < 3; ++b)
#pragma unroll
                for (int g = 0; g < 3; ++g) S[3 * b + g] = fma(sw[j] * sxc[3 * j + b], sy[3 * j + g], S[3 * b + g]);
#pragma unroll
              for (int a = 0; a < 3; ++a) gy = fma(sw[j] * sy[3 * j + a], sy[3 * j + a], gy);
            }
#pragma unroll
            for (int e = 0; e < 9; ++e) S[e] = warp_sum_d(S[e]);
            gy = warp_sum_d(gy);
            if (lane == 0) {
              double K[4][4], eig[4], V[4][4];
              kearsley_from_S(S, s_gx, gy, K);
              if (!jacobi4(K, eig, V)) s_flags |= kFlagNoConverge;
              double q0[4] = {V[0][0], V[1][0], V[2][0], V[3][0]};
              quat_to_rot(q0, s_rxy);
#pragma unroll
              for (int e = 0; e < 4; ++e) s_eig[e] = eig[e];
#pragma unroll
              for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) s_V[4 * r + cc] = V[r][cc];
              s_dxy = eig[0];
              s_refresh = eig[0] > P.eps ? 1 : 0;
            }
          }
        } else if (tid == 0) {
          s_refresh = 1;  // first step: no close structure yet
          s_dxy = 0.0;
        }
      } else if (tid == 0) {
        s_refresh = 1;
        s_dxy = 0.0;
      }
      __syncthreads();
      const bool exact = s_refresh != 0;
      // neighbour list: update on the first step and whenever t - last >= stride
      // (maybe_update); the references evaluated: all (no list, an update, or a close-mode
      // reassignment refitting every saved rotation), else only the list members
      const bool update = nl && (s_nl_last < 0 || t - s_nl_last >= P.nl_stride);
      const bool every = !nl || update || (P.mode == 2 && exact);
      // C: one thread per reference: covariance, then the exact fit (Eq. 3) or Eq. 5
      for (int i = tid; i < L; i += TNT) {
        if (!every && !s_act[i]) {
          sD[i] = INFINITY;  // not evaluated this step (outside the list)
          continue;
        }
        const double* a = refs + (int64_t)i * n * 3;
        double S[9];
#pragma unroll
        for (int e = 0; e < 9; ++e) S[e] = 0.0;
        for (int j = 0; j < n; ++j) {
          const double wj = sw[j];
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const double xb = wj * sxc[3 * j + b];
#pragma unroll
            for (int g = 0; g < 3; ++g) S[3 * b + g] = fma(xb, a[3 * j + g], S[3 * b + g]);
          }
        }
#pragma unroll
        for (int e = 0; e < 9; ++e) sS[9 * i + e] = S[e];
        if (exact) {
          double K[4][4], eig[4], V[4][4], R[9];
          kearsley_from_S(S, s_gx, refg[i], K);
          if (!jacobi4(K, eig, V)) atomicOr(&s_flags, (unsigned)kFlagNoConverge);
          const double q0[4] = {V[0][0], V[1][0], V[2][0], V[3][0]};
          quat_to_rot(q0, R);
          sD[i] = eig[0];
#pragma unroll
          for (int e = 0; e < 9; ++e) sRh[9 * i + e] = R[e];
          if (P.mode == 2)
#pragma unroll
            for (int e = 0; e < 9; ++e) sRay[9 * i + e] = R[e];  // y <- x: R_{a_i y} = R_{a_i x}
        } else {
          double Rh[9], dot = 0.0;
#pragma unroll
          for (int r = 0; r < 3; ++r)
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)
              Rh[3 * r + cc] = s_rxy[3 * r] * sRay[9 * i + cc] + s_rxy[3 * r + 1] * sRay[9 * i + 3 + cc] +
                               s_rxy[3 * r + 2] * sRay[9 * i + 6 + cc];
#pragma unroll
          for (int e = 0; e < 9; ++e) {
            sRh[9 * i + e] = Rh[e];
            dot = fma(Rh[e], S[e], dot);
          }
          sD[i] = s_gx + refg[i] - 2.0 * dot;
        }
      }
      __syncthreads();
      if (update) {
        // the M smallest distances, ties by lower index (rank = #{j: D_j < D_i or
        // D_j == D_i and j < i}); the members are a set (ascending-index order)
        for (int i = tid; i < L; i += TNT) {
          const double di = sD[i];
          int rank = 0;
          for (int j = 0; j < L; ++j) rank += (sD[j] < di || (sD[j] == di && j < i)) ? 1 : 0;
          s_act[i] = rank < P.nl_m ? 1 : 0;
        }
        if (tid == 0) s_nl_last = t;
        __syncthreads();
      }
      // D: property map (Eq. 2 with the min-D shift) and z, coefficients (warp 0), over the
      // list members only when a neighbour list is on
      if (warp == 0) {
        double dmin = INFINITY;
        for (int i = lane; i < L; i += 32)
          if (!nl || s_act[i]) dmin = fmin(dmin, sD[i]);
        dmin = warp_min_d(dmin);
        double zs = 0.0, qs = 0.0;
        for (int i = lane; i < L; i += 32) {
          if (nl && !s_act[i]) continue;
          const double e = exp(-P.lam * (sD[i] - dmin));
          zs += e;
          qs = fma(q[i], e, qs);
        }
        zs = warp_sum_d(zs);
        qs = warp_sum_d(qs);
        const double sval = qs / zs, zval = dmin - log(zs) / P.lam;
        double ss = 0.0, sz = 0.0;
        for (int i = lane; i < L; i += 32) {
          const bool on = !nl || s_act[i];
          const double p = on ? exp(-P.lam * (sD[i] - dmin)) / zs : 0.0;
          scs[i] = on ? -P.lam * p * (q[i] - sval) : 0.0;
          scz[i] = p;
          ss += scs[i];
          sz += p;
        }
        ss = warp_sum_d(ss);
        sz = warp_sum_d(sz);
        if (lane == 0) {
          s_s = sval;
          s_z = zval;
          s_sum[0] = ss;
          s_sum[1] = sz;
          if (!isfinite(sval) || !isfinite(zval)) s_flags |= kFlagNonFinite;
        }
      }
      __syncthreads();
      // E: Eq. 6 dR_xy term (non-refresh steps): M = -2 [sum c_i S_i R_i^T - R_xy sum c_i R_i A_i R_i^T],
      // g = <M, dR/dq>, v = sum_m (q_m . g) / (l0 - lm) q_m.  Per-reference terms in
      // parallel (thread i -> sPart[i][36]), summed in index order by warp 0 below.
      if (!exact) {
        for (int i = tid; i < L; i += TNT) {
          if (nl && !s_act[i]) {  // outside the list: no Eq. 6 term
            for (int e = 0; e < 36; ++e) sPart[36 * i + e] = 0.0;
            continue;
          }
          const double* Si = sS + 9 * i;
          const double* Ri = sRay + 9 * i;
          const double* m = refmom + 6 * (int64_t)i;
          const double A[9] = {m[0], m[1], m[2], m[1], m[3], m[4], m[2], m[4], m[5]};
          double SR[9], RA[9], RAR[9];
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              SR[3 * a + b] = Si[3 * a] * Ri[3 * b] + Si[3 * a + 1] * Ri[3 * b + 1] + Si[3 * a + 2] * Ri[3 * b + 2];
              RA[3 * a + b] = Ri[3 * a] * A[b] + Ri[3 * a + 1] * A[3 + b] + Ri[3 * a + 2] * A[6 + b];
            }
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
              RAR[3 * a + b] = RA[3 * a] * Ri[3 * b] + RA[3 * a + 1] * Ri[3 * b + 1] + RA[3 * a + 2] * Ri[3 * b + 2];
          double* pp = sPart + 36 * i;
#pragma unroll
          for (int e = 0; e < 9; ++e) {
            pp[e] = scs[i] * SR[e];
            pp[9 + e] = scs[i] * RAR[e];
            pp[18 + e] = scz[i] * SR[e];
            pp[27 + e] = scz[i] * RAR[e];
          }
        }
      }
      if (warp == 1) {
        // hills deposited so far (Eq. 1, direct summation): V(s) and dV/ds
        double V = 0.0, dv = 0.0;
        const double inv = 1.0 / (P.hill_sigma * P.hill_sigma);
        for (int h = lane; h < s_nh; h += 32) {
          const double d = s_s - hills[(int64_t)wk * P.max_hills + h];
          const double e = P.hill_h * exp(-0.5 * d * d * inv);
          V += e;
          dv -= e * d * inv;
        }
        V = warp_sum_d(V);
        dv = warp_sum_d(dv);
        if (lane == 0) {
          s_bias = V;
          s_dvds = dv;
        }
      }
      __syncthreads();
      if (!exact && warp == 0) {
        double acc0 = 0.0, acc1 = 0.0;  // entries lane and 32 + lane (< 36)
        for (int i = 0; i < L; ++i) {
          acc0 += sPart[36 * i + lane];
          if (lane < 4) acc1 += sPart[36 * i + 32 + lane];
        }
        sPart[36 * L + lane] = acc0;
        if (lane < 4) sPart[36 * L + 32 + lane] = acc1;
        __syncwarp();
        if (lane < 2) {
          const int c = lane;
          const double* SR = sPart + 36 * L + 18 * c;
          const double* RAR = SR + 9;
          double J[4][9];
          const double q0[4] = {s_V[0], s_V[4], s_V[8], s_V[12]};
          rot_quat_jacobian(q0, J);
          double M[9];
#pragma unroll
          for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              const double xr = s_rxy[3 * a] * RAR[b] + s_rxy[3 * a + 1] * RAR[3 + b] + s_rxy[3 * a + 2] * RAR[6 + b];
              M[3 * a + b] = -2.0 * (SR[3 * a + b] - xr);
            }
          double g[4];
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 9; ++k) acc += M[k] * J[cc][k];
            g[cc] = acc;
          }
          double v[4] = {0.0, 0.0, 0.0, 0.0};
          for (int m = 1; m < 4; ++m) {
            const double h = (s_V[m] * g[0] + s_V[4 + m] * g[1] + s_V[8 + m] * g[2] + s_V[12 + m] * g[3]) /
                             (s_eig[0] - s_eig[m]);
#pragma unroll
            for (int r = 0; r < 4; ++r) v[r] += h * s_V[4 * r + m];
          }
#pragma unroll
          for (int r = 0; r < 4; ++r) s_v[c][r] = v[r];
        }
      }
      __syncthreads();
      // F: centred gradients of s and z per atom (exact rows: envelope form 2w(x - R a);
      // approx rows add the dR_xy term), then the raw-coordinate centring correction
      for (int k = tid; k < n; k += TNT) {
        double us[3] = {0.0, 0.0, 0.0}, uz[3] = {0.0, 0.0, 0.0};
        for (int i = 0; i < L; ++i) {
          if (nl && !s_act[i]) continue;
          const double* a = refs + ((int64_t)i * n + k) * 3;
          const double* Rh = sRh + 9 * i;
#pragma unroll
          for (int b = 0; b < 3; ++b) {
            const double ra = Rh[3 * b] * a[0] + Rh[3 * b + 1] * a[1] + Rh[3 * b + 2] * a[2];
            us[b] = fma(scs[i], ra, us[b]);
            uz[b] = fma(scz[i], ra, uz[b]);
          }
        }
        const double wk2 = 2.0 * sw[k];
        double gs[3], gz[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          gs[b] = wk2 * (s_sum[0] * sxc[3 * k + b] - us[b]);
          gz[b] = wk2 * (s_sum[1] * sxc[3 * k + b] - uz[b]);
        }
        if (!exact) {
          const double q0[4] = {s_V[0], s_V[4], s_V[8], s_V[12]};
          const double xk[3] = {sxc[3 * k], sxc[3 * k + 1], sxc[3 * k + 2]};
          const double yk[3] = {sy[3 * k], sy[3 * k + 1], sy[3 * k + 2]};
          double d[3];
          dk_contract(s_v[0], q0, sw[k], xk, yk, d);
#pragma unroll
          for (int b = 0; b < 3; ++b) gs[b] += d[b];
          dk_contract(s_v[1], q0, sw[k], xk, yk, d);
#pragma unroll
          for (int b = 0; b < 3; ++b) gz[b] += d[b];
        }
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          sg[0][3 * k + b] = gs[b];
          sg[1][3 * k + b] = gz[b];
        }
      }
      __syncthreads();
      if (warp == 0) {
        double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        for (int j = lane; j < n; j += 32)
#pragma unroll
          for (int e = 0; e < 3; ++e) {
            acc[e] += sg[0][3 * j + e];
            acc[3 + e] += sg[1][3 * j + e];
          }
#pragma unroll
        for (int e = 0; e < 6; ++e) acc[e] = warp_sum_d(acc[e]);
        if (lane < 6) s_gsum[lane] = acc[lane];
      }
      __syncthreads();
      for (int e = tid; e < 3 * n; e += TNT) {
        const int j = e / 3, b = e - 3 * j;
        sg[0][e] -= swa[j] * s_gsum[b];
        sg[1][e] -= swa[j] * s_gsum[3 + b];
      }
      if (tid == 0) {
        const int64_t o = (int64_t)wk * P.steps + it;
        cv[4 * o] = s_s;
        cv[4 * o + 1] = s_z;
        cv[4 * o + 2] = s_bias;
        cv[4 * o + 3] = s_dxy;
        rlog[o] = (P.mode == 2 && exact) ? 1 : 0;
        // counters (SPEC msd-engine): original = L exact per step; close = 1 (x<->y) + L on
        // reassignment, else L cheap; with a neighbour list M instead of L except on update
        // steps (SPEC neighbourlist: an update evaluates all N)
        const long long nev = every ? L : P.nl_m;
        if (P.mode == 1) {
          c_exp += nev;
        } else {
          c_exp += 1;
          if (exact) { c_exp += L; c_reas += 1; } else { c_cheap += nev; }
        }
      }
      __syncthreads();
      if (P.mode == 2 && exact) {  // Alg. 2: y <- x (centred)
        for (int e = tid; e < 3 * n; e += TNT) sy[e] = sxc[e];
        if (tid == 0) s_hasy = 1;
      }
    }
    // G: forces and the Euler-Maruyama step x += mob F + sqrt(2 kT mob) xi
    for (int k = tid; k < n; k += TNT) {
      double F[3], z[3];
      toy_bonded_force(sx, n, k, P, F);
      if (P.mode != 0)
#pragma unroll
        for (int b = 0; b < 3; ++b) F[b] -= s_dvds * sg[0][3 * k + b];  // F_bias = -dV/ds ds/dx
      toy_normals(P.seed, wk, t, k, z);
#pragma unroll
      for (int b = 0; b < 3; ++b) sxn[3 * k + b] = sx[3 * k + b] + P.mob * F[b] + P.noise * z[b];
    }
    __syncthreads();
    for (int e = tid; e < 3 * n; e += TNT) sx[e] = sxn[e];
    // H: deposit a hill at this step's s every tau_G steps (after its force used the old ones)
    if (tid == 0 && P.mode != 0 && P.tau_g > 0 && t % P.tau_g == 0) {
      if (s_nh < P.max_hills) hills[(int64_t)wk * P.max_hills + s_nh++] = s_s;
      else s_flags |= kFlagSigOverflow;
    }
    __syncthreads();
  }
  for (int e = tid; e < 3 * n; e += TNT) {
    xs[(int64_t)wk * 3 * n + e] = sx[e];
    ys[(int64_t)wk * 3 * n + e] = sy[e];
  }
  if (P.mode == 2)
    for (int e = tid; e < 9 * L; e += TNT) rays[(int64_t)wk * 9 * L + e] = sRay[e];
  if (nl)
    for (int i = tid; i < L; i += TNT) act[(int64_t)wk * L + i] = s_act[i];
  if (tid == 0) {
    if (nl) nl_last[wk] = s_nl_last;
    hasy[wk] = s_hasy;
    nhills[wk] = s_nh;
    counters[3 * wk] += c_exp;
    counters[3 * wk + 1] += c_cheap;
    counters[3 * wk + 2] += c_reas;
    if (flags) flags[wk] |= (uint8_t)s_flags;
  }
}

cudaError_t launch_toysim(const ToyParams& P, int W, const double* refs, const double* refg, const double* refmom,
                          const double* q, const double* w, const double* wa, double* xs, double* ys, double* rays,
                          int* hasy, double* hills, int* nhills, long long* counters, double* cv, uint8_t* rlog,
                          double* traj, uint8_t* flags, cudaStream_t stream, uint8_t* act, long long* nl_last) {
  if (W <= 0 || P.steps <= 0) return cudaSuccess;
  if (P.nl_m > 0 && (!act || !nl_last || P.nl_m > P.L || P.nl_stride < 1 || P.mode == 0))
    return cudaErrorInvalidValue;
  const size_t dsm = sizeof(double) * 36 * (P.L + 1);  // <= 37 KB (L <= 128)
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(toysim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 36 * 8 * (TMAXL + 1));
    attr = true;
  }
  toysim_kernel<<<W, TNT, dsm, stream>>>(P, refs, refg, refmom, q, w, wa, xs, ys, rays, hasy, hills, nhills, counters,
                                       cv, rlog, traj, flags, act, nl_last);
  return cudaGetLastError();
}

}  // namespace mc
