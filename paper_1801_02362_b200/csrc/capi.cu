// extern "C" boundary of libmcb200.so (declared in include/mcb200.h).
// Argument validation maps to the reference error taxonomy (errors.py:4-35);
// CUDA launch errors map to MC_ERR_CUDA_BASE - cudaError_t.
#include <cstdlib>

#include "../../include/mcb200.h"
#include "launch.h"

namespace {
inline int cuda_status(cudaError_t e) { return e == cudaSuccess ? MC_OK : MC_ERR_CUDA_BASE - (int)e; }
inline cudaStream_t S_(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool bad_pad(int32_t n, int32_t npad) { return n < 1 || npad < n || (npad % 32) != 0; }
}  // namespace

extern "C" {

int mc_version(void) { return 1; }

int mc_center(const void* coords, int dtype, int64_t count, int32_t n, int32_t npad, const double* w_align,
              const double* w_disp, double* planes, double* wplanes, double* centroid, double* gnorm,
              double* wbar, double* mom, uint8_t* flags, void* stream) {
  if (count < 0 || (count > 0 && (!coords || !planes || !gnorm || !w_disp))) return MC_ERR_CONFIG;
  if (dtype != MC_F32 && dtype != MC_F64) return MC_ERR_CONFIG;
  if (n < 2) return MC_ERR_INVALID_STRUCTURE;  // geometry.py:39-40
  if (bad_pad(n, npad)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_center(coords, dtype, count, n, npad, w_align, w_disp, planes, wplanes, centroid,
                                       gnorm, wbar, mom, flags, S_(stream)));
}

int mc_cov_f64(const double* fplanes, const double* lwplanes, int32_t T, int32_t L, int32_t npad, double* S,
               void* stream) {
  if (T < 0 || L < 0 || npad % 32 != 0 || ((int64_t)T * L > 0 && (!fplanes || !lwplanes || !S))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_cov_f64(fplanes, lwplanes, T, L, npad, S, S_(stream)));
}

int mc_cov_pairs(const double* xplanes, const double* aplanes, const int32_t* xi, const int32_t* ai, int64_t P,
                 int32_t npad, const double* w, double* S, void* stream) {
  if (P < 0 || npad % 32 != 0 || (P > 0 && (!xplanes || !aplanes || !S))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_cov_pairs(xplanes, aplanes, xi, ai, P, npad, w, S, S_(stream)));
}

int mc_fit_dense(const double* S, int32_t T, int32_t L, const double* gx, const double* ga,
                 const uint8_t* rowmask, double* D, double* rot, double* quat, uint8_t* flags, void* stream) {
  if (T < 0 || L < 0 || ((int64_t)T * L > 0 && (!S || !gx || !ga || !D))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_fit_dense(S, T, L, gx, ga, rowmask, D, rot, quat, flags, S_(stream)));
}

int mc_fit_list_msd(const double* S, int64_t P, const int32_t* xi, const int32_t* ai, const double* gx,
                    const double* ga, double* D, void* stream) {
  if (P < 0 || (P > 0 && (!S || !gx || !ga || !D))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_fit_list_msd(S, P, xi, ai, gx, ga, D, S_(stream)));
}

int mc_fit_full(const double* S, int64_t P, const int32_t* xi, const int32_t* ai, const double* gx,
                const double* ga, double* eig, double* quat, double* rot, uint8_t* flags, void* stream) {
  if (P < 0 || (P > 0 && (!S || !gx || !ga))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_fit_full(S, P, xi, ai, gx, ga, eig, quat, rot, flags, S_(stream)));
}

int mc_rot_grad(const double* xplanes, const double* aplanes, const int32_t* xi, const int32_t* ai, int64_t P,
                int32_t n, int32_t npad, const double* w, const double* eig, double* out, void* stream) {
  if (P < 0 || bad_pad(n, npad) || (P > 0 && (!xplanes || !aplanes || !w || !eig || !out))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_rot_grad(xplanes, aplanes, xi, ai, P, n, npad, w, eig, out, S_(stream)));
}

int mc_jacobi_n(const double* mats, int64_t B, int32_t n, double tol, int32_t max_sweeps, double* vals, double* vecs,
                uint8_t* flags, void* stream) {
  if (B < 0 || n < 1 || n > 48 || max_sweeps < 0 || !(tol >= 0.0)) return MC_ERR_CONFIG;
  if (B > 0 && (!mats || !vals || !vecs)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_jacobi_n(mats, B, n, tol, max_sweeps, vals, vecs, flags, S_(stream)));
}

int mc_jacobi4(const double* mats, int64_t B, double* vals, double* vecs, uint8_t* flags, void* stream) {
  if (B < 0 || (B > 0 && (!mats || !vals || !vecs))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_jacobi4(mats, B, vals, vecs, flags, S_(stream)));
}

int mc_window_pairs(int32_t walkers, int32_t steps, int32_t K, int32_t* xi, int32_t* ai, void* stream) {
  if (walkers < 0 || steps < 0 || K < 1 || !xi || !ai) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_window_pairs(walkers, steps, K, xi, ai, S_(stream)));
}

int mc_close_scan(const double* fplanes, const double* gx, int32_t walkers, int32_t steps, int32_t npad,
                  const double* w, const double* dwin, int32_t K, double eps, uint8_t* refresh, int32_t* ridx,
                  double* dxy, int32_t* n_onthefly, void* stream) {
  if (walkers < 0 || steps < 0 || K < 1 || K > 32 || npad % 32 != 0) return MC_ERR_CONFIG;
  if (!(eps >= 0.0)) return MC_ERR_CONFIG;
  if (walkers * (int64_t)steps > 0 && (!fplanes || !gx || !w || !dwin || !refresh || !ridx || !dxy))
    return MC_ERR_CONFIG;
  return cuda_status(mc::launch_close_scan(fplanes, gx, walkers, steps, npad, w, dwin, K, eps, refresh, ridx, dxy,
                                           n_onthefly, S_(stream)));
}

int mc_xy_eig(const double* fplanes, const double* gx, int64_t T, int32_t npad, const double* w,
              const uint8_t* refresh, const int32_t* ridx, double* xyeig, double* rxy, uint8_t* flags, void* stream) {
  if (T < 0 || npad % 32 != 0 || (T > 0 && (!fplanes || !gx || !w || !refresh || !ridx || !xyeig || !rxy)))
    return MC_ERR_CONFIG;
  return cuda_status(mc::launch_xy_eig(fplanes, gx, T, npad, w, refresh, ridx, xyeig, rxy, flags, S_(stream)));
}

int mc_shard_rescale(int32_t T, int32_t cap, const int32_t* nsig, const double* alpha, const double* beta,
                     double* sig_coef, double* fvec, void* stream) {
  if (T < 0 || cap < 1) return MC_ERR_CONFIG;
  if (T > 0 && (!nsig || !alpha || !beta || !sig_coef || !fvec)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_shard_rescale(T, cap, nsig, alpha, beta, sig_coef, fvec, S_(stream)));
}

int mc_pathcv_weights(int32_t T, int32_t t0, int32_t L, double lam, double cutoff, int32_t cap, int32_t ld, const int32_t* rowlo,
                      const int32_t* rowcnt, double* D, const double* q, const double* R, const double* fwbar,
                      const double* lwbar, const uint8_t* refresh, const int32_t* ridx, const double* S,
                      const double* rxy, const double* xyeig, const double* gx, const double* ga, const double* lmom,
                      double* s, double* z, int32_t* sig_idx, double* sig_coef, int32_t* nsig, double* fvec,
                      uint8_t* flags, void* stream) {
  if (T < 0 || t0 < 0) return MC_ERR_CONFIG;
  if (T > 0 && L < 1) return MC_ERR_EMPTY_ACTIVE_SET;
  if (!(lam > 0.0) || !(cutoff > 0.0) || cap < 1) return MC_ERR_CONFIG;
  if ((rowlo == nullptr) != (rowcnt == nullptr)) return MC_ERR_CONFIG;
  if (!rowcnt && ld != L) return MC_ERR_CONFIG;
  if (T > 0 && (!D || !q || !R || !fwbar || !lwbar || !s || !z || !sig_idx || !sig_coef || !nsig || !fvec))
    return MC_ERR_CONFIG;
  if (refresh && (!ridx || !S || !rxy || !xyeig || !gx || !ga || !lmom)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_cv_weights(T, t0, L, lam, cutoff, cap, ld, rowlo, rowcnt, D, q, R, fwbar, lwbar, refresh,
                                           ridx, S, rxy, xyeig, gx, ga, lmom, s, z, sig_idx, sig_coef, nsig, fvec,
                                           flags, S_(stream)));
}

int mc_pathcv_weights_nl(int32_t T, int32_t t0, int32_t L, double lam, double cutoff, int32_t cap,
                         const int32_t* nb_idx, const int32_t* nb_row, int32_t nb_m, int32_t dmode, double* D,
                         const double* q, const double* R, const double* fwbar, const double* lwbar,
                         const uint8_t* refresh, const int32_t* ridx, const double* S, const double* rxy,
                         const double* xyeig, const double* gx, const double* ga, const double* lmom, double* s,
                         double* z, int32_t* sig_idx, double* sig_coef, int32_t* nsig, double* fvec, uint8_t* flags,
                         void* stream) {
  if (T < 0 || t0 < 0 || dmode < 0 || dmode > 2) return MC_ERR_CONFIG;
  if (T > 0 && L < 1) return MC_ERR_EMPTY_ACTIVE_SET;
  if (!(lam > 0.0) || !(cutoff > 0.0) || cap < 1) return MC_ERR_CONFIG;
  if ((nb_idx == nullptr) != (nb_row == nullptr)) return MC_ERR_CONFIG;
  if (nb_idx && (nb_m < 1 || nb_m > L || L > 16384)) return MC_ERR_CONFIG;
  if (T > 0 && (!D || !R || !fwbar || !lwbar)) return MC_ERR_CONFIG;
  if (T > 0 && dmode != 1 && (!q || !s || !z || !sig_idx || !sig_coef || !nsig || !fvec)) return MC_ERR_CONFIG;
  if (refresh && (!ridx || !S || !rxy || !xyeig || !gx || !ga || !lmom)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_cv_weights(T, t0, L, lam, cutoff, cap, L, nullptr, nullptr, D, q, R, fwbar, lwbar,
                                           refresh, ridx, S, rxy, xyeig, gx, ga, lmom, s, z, sig_idx, sig_coef, nsig,
                                           fvec, flags, S_(stream), nb_idx, nb_row, nb_m, dmode));
}

int mc_neighbour_topm(const void* D, int dtype, int32_t nrows, int32_t L, int64_t ldd, const int32_t* rows, int32_t M,
                      int32_t* idx, void* stream) {
  if (dtype != MC_F32 && dtype != MC_F64) return MC_ERR_CONFIG;
  if (nrows < 0 || L < 1 || ldd < L || M < 1 || M > L) return MC_ERR_CONFIG;  // SPEC: M > N -> configuration error
  if (nrows > 0 && (!D || !idx)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_topm(D, dtype, nrows, L, ldd, rows, M, idx, S_(stream)));
}

int mc_pathcv_grad(int32_t T, int32_t t0, int32_t n, int32_t npad, int32_t cap, const double* fplanes, const double* lplanes,
                   const double* w, const double* w_align, const int32_t* sig_idx, const double* sig_coef,
                   const int32_t* nsig, const double* fvec, const uint8_t* refresh, const int32_t* ridx,
                   const double* xyeig, void* ds, void* dz, int32_t out_f32, const float* fraw, const double* fcen,
                   const float* lraw, const double* lcen, const int32_t* perm, void* stream) {
  if (T < 0 || t0 < 0 || bad_pad(n, npad) || cap < 1) return MC_ERR_CONFIG;
  if (T > 0 && (!w || !w_align || !sig_idx || !sig_coef || !nsig || !fvec || !ds || !dz)) return MC_ERR_CONFIG;
  if (t0 > 0 && !(fplanes && lplanes && !perm)) return MC_ERR_CONFIG;  // chunked launches: planes path only
  if (T > 0 && !fplanes && !(fraw && fcen)) return MC_ERR_CONFIG;
  if (T > 0 && !lplanes && !(lraw && lcen)) return MC_ERR_CONFIG;
  if (refresh && (!ridx || !xyeig || !fplanes)) return MC_ERR_CONFIG;
  if (fplanes && lplanes && !perm)  // fp64 planes: the frame-group blocked pass (grad_block.cu)
    return cuda_status(mc::launch_cv_grad_block_planes(T, t0, n, npad, cap, fplanes, lplanes, w, w_align, sig_idx,
                                                       sig_coef, nsig, fvec, refresh, ridx, xyeig, ds, dz, out_f32,
                                                       S_(stream)));
  return cuda_status(mc::launch_cv_grad(T, n, npad, cap, fplanes, lplanes, w, w_align, sig_idx, sig_coef, nsig, fvec,
                                        refresh, ridx, xyeig, ds, dz, out_f32, fraw, fcen, lraw, lcen, perm,
                                        S_(stream)));
}

int mc_msd_tf32_2sm(const float* fhi, const float* flo, const float* lhi, const float* llo, const double* gx,
                    const double* ga, int32_t T, int32_t L, int32_t kpad, float* D, int64_t ldd, int32_t grid,
                    void* stream) {
  if (T < 0 || L < 0 || kpad % 16 != 0 || kpad < 16 || ldd < L) return MC_ERR_CONFIG;
  if ((int64_t)T * L > 0 && (!fhi || !flo || !lhi || !llo || !gx || !ga || !D)) return MC_ERR_CONFIG;
  if (3LL * T > 0x7fffffffLL || 3LL * L > 0x7fffffffLL) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_msd_tf32_2sm(fhi, flo, lhi, llo, gx, ga, T, L, kpad, D, ldd, grid, S_(stream)));
}

int mc_pathcv_grad_block(int32_t T, int32_t n, int32_t cap, const float* fraw, const double* fcen, const float* lraw,
                         const double* lcen, const double* w, const double* w_align, const int32_t* sig_idx,
                         const double* sig_coef, const int32_t* nsig, const double* fvec, const int32_t* perm,
                         const int32_t* out_map, void* ds, void* dz, int32_t out_f32, void* stream) {
  if (T < 0 || n < 2 || cap < 1) return MC_ERR_CONFIG;
  if (T > 0 && (!fraw || !fcen || !lraw || !lcen || !w || !w_align || !sig_idx || !sig_coef || !nsig || !fvec ||
                !ds || !dz))
    return MC_ERR_CONFIG;
  // fp64 tensor-core (DMMA) contraction by default; MC_GRAD_VECTOR=1 selects the
  // CUDA-core kernel (grad_block.cu) for A/B comparison
  static const bool vec = [] {
    const char* e = getenv("MC_GRAD_VECTOR");
    return e && e[0] == '1';
  }();
  if (vec) {
    if (out_map) return MC_ERR_CONFIG;  // the CUDA-core comparison kernel writes rows in place
    return cuda_status(mc::launch_cv_grad_block(T, n, cap, fraw, fcen, lraw, lcen, w, w_align, sig_idx, sig_coef,
                                                nsig, fvec, perm, ds, dz, out_f32, S_(stream)));
  }
  return cuda_status(mc::launch_cv_grad_dmma(T, n, cap, fraw, fcen, lraw, lcen, w, w_align, sig_idx, sig_coef, nsig,
                                             fvec, perm, out_map, ds, dz, out_f32, S_(stream)));
}

int mc_ldig_prep(const float* lraw, const double* lcen, int32_t L, int32_t n, int32_t npad, int32_t kpad,
                 int32_t* eB, int8_t* dig, void* stream) {
  if (L < 1 || n < 2 || npad < n || npad % 128 != 0 || kpad < 3 * L || kpad % 32 != 0) return MC_ERR_CONFIG;
  if (!lraw || !lcen || !eB || !dig) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_ldig(lraw, lcen, L, n, npad, kpad, eB, dig, S_(stream)));
}

int mc_pathcv_grad_i8(int32_t T, int32_t n, int32_t cap, const float* fraw, const double* fcen, const float* lraw,
                      const double* lcen, const double* w, const double* w_align, const int8_t* dig,
                      const int32_t* eB, int32_t npad, int32_t kpad, const int32_t* sig_idx, const double* sig_coef,
                      const int32_t* nsig, const double* fvec, const double* dV, const int32_t* perm,
                      const int32_t* out_map, void* out0, void* out1, int32_t out_f32, int32_t ncv,
                      int32_t* wide_flag, void* workspace, int64_t ws_bytes, void* stream) {
  if (T < 0 || n < 2 || cap < 1 || (ncv != 1 && ncv != 2)) return MC_ERR_CONFIG;
  if (T > 0 && (!fraw || !fcen || !lraw || !lcen || !w || !w_align || !dig || !eB || !sig_idx || !sig_coef ||
                !nsig || !fvec || !out0 || (ncv == 2 && !out1) || (ncv == 1 && !dV)))
    return MC_ERR_CONFIG;
  if (npad < n || npad % 128 != 0 || kpad % 32 != 0) return MC_ERR_CONFIG;
  if (ncv == 1 && (n % 4 != 0 || !workspace || ws_bytes < (int64_t)mc::grad_i8_workspace(T, 1)))
    return MC_ERR_CONFIG;  // the fused force runs only on the tensor-core kernel
  return cuda_status(mc::launch_cv_grad_i8(T, n, cap, fraw, fcen, lraw, lcen, w, w_align, dig, eB, npad, kpad,
                                           sig_idx, sig_coef, nsig, fvec, dV, perm, out_map, out0, out1, out_f32,
                                           ncv, wide_flag, workspace, ws_bytes < 0 ? 0 : (size_t)ws_bytes,
                                           S_(stream)));
}

int mc_row_digits(const float* raw, const double* centroid, const double* w, const int32_t* perm,
                  const int32_t* fmap, int32_t B, int32_t n, int32_t kpad, int8_t* dig, int32_t* e,
                  const int32_t* ein, int32_t planes, void* stream) {
  if (B < 0 || n < 2 || kpad < n || kpad % 32 != 0 || (planes != 0 && planes != 1)) return MC_ERR_CONFIG;
  if (B > 0 && (!raw || !centroid || !dig || !e)) return MC_ERR_CONFIG;
  if (ein && w) return MC_ERR_CONFIG;  // precomputed exponents are those of the unweighted rows
  return cuda_status(mc::launch_rdig(raw, centroid, w, perm, fmap, B, n, kpad, dig, e, S_(stream), ein, planes));
}

int mc_refine_i8(const int8_t* ldig, const int32_t* eL, const int8_t* fdig, const int32_t* eF, int32_t T, int32_t L,
                 int32_t n, int32_t kpad, const int32_t* perm, const int32_t* lo, const int32_t* cnt, const double* gx,
                 const double* ga, int32_t cap, double* Dex, double* Rex, float* Dd, int64_t ldd, uint8_t* flags,
                 void* stream) {
  if (T < 0 || L < 1 || n < 2 || n >= 32768 || kpad < n || kpad % 32 != 0) return MC_ERR_CONFIG;
  if ((lo == nullptr) != (cnt == nullptr)) return MC_ERR_CONFIG;
  if (T > 0 && (!ldig || !eL || !fdig || !eF || !gx || !ga)) return MC_ERR_CONFIG;
  if (!Dex && !Dd) return MC_ERR_CONFIG;
  if ((Dex || Rex) && cap < 1) return MC_ERR_CONFIG;
  if (Dd && ldd < L) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_refine_i8(ldig, eL, fdig, eF, T, L, n, kpad, perm, lo, cnt, gx, ga, cap, Dex, Rex, Dd,
                                          ldd, flags, S_(stream)));
}

int mc_grad_i8_wide_plan(int32_t T, int32_t cap, int32_t ncv, const int32_t* sig_idx, const int32_t* nsig,
                         const int32_t* perm, int64_t* bytes, void* stream) {
  if (T < 0 || cap < 1 || (ncv != 1 && ncv != 2)) return MC_ERR_CONFIG;
  if (T > 0 && (!sig_idx || !nsig || !bytes)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_grad_i8_plan(T, cap, ncv, sig_idx, nsig, perm, reinterpret_cast<long long*>(bytes),
                                             S_(stream)));
}

int64_t mc_grad_i8_wide_header_size(int32_t nwide, int32_t ncv) {
  if (nwide < 0 || (ncv != 1 && ncv != 2)) return -1;
  return (int64_t)mc::grad_i8_wide_header_bytes(nwide, ncv);
}

int mc_pathcv_grad_i8_wide(int32_t T, int32_t n, int32_t cap, const float* fraw, const double* fcen, const double* w,
                           const double* w_align, const int8_t* dig, const int32_t* eB, int32_t npad, int32_t kpad,
                           const int32_t* sig_idx, const double* sig_coef, const int32_t* nsig, const double* fvec,
                           const double* dV, const int32_t* perm, const int32_t* out_map, void* out0, void* out1,
                           int32_t out_f32, int32_t ncv, const int32_t* wide_ids, int32_t nwide,
                           const int64_t* wide_off, void* hws, int64_t hws_bytes, void* wimg, void* stream) {
  if (T < 0 || n < 2 || cap < 1 || nwide < 0 || (ncv != 1 && ncv != 2)) return MC_ERR_CONFIG;
  if (nwide == 0) return MC_OK;
  if (!fraw || !fcen || !w || !w_align || !dig || !eB || !sig_idx || !sig_coef || !nsig || !fvec || !out0 ||
      (ncv == 2 && !out1) || (ncv == 1 && !dV) || !wide_ids || !wide_off || !hws || !wimg)
    return MC_ERR_CONFIG;
  if (n % 4 != 0 || npad < n || npad % 128 != 0 || kpad % 32 != 0) return MC_ERR_CONFIG;
  if (hws_bytes < (int64_t)mc::grad_i8_wide_header_bytes(nwide, ncv)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_cv_grad_i8_wide(T, n, cap, fraw, fcen, w, w_align, dig, eB, npad, kpad, sig_idx,
                                                sig_coef, nsig, fvec, dV, perm, out_map, out0, out1, out_f32, ncv,
                                                wide_ids, nwide, reinterpret_cast<const long long*>(wide_off), hws,
                                                wimg, S_(stream)));
}

int64_t mc_grad_i8_workspace_size(int32_t T, int32_t ncv) {
  if (T < 0 || (ncv != 1 && ncv != 2)) return -1;
  return (int64_t)mc::grad_i8_workspace(T, ncv);
}

int mc_refine_i8_close(const int8_t* ldig, const int32_t* eL, const int8_t* fdig, const int32_t* eF, int32_t T,
                       int32_t L, int32_t n, int32_t kpad, const int32_t* perm, const int32_t* lo, const int32_t* cnt,
                       const double* gx, const double* ga, int32_t cap, const uint8_t* fitmask, double* Sex,
                       double* Dex, double* Rex, uint8_t* flags, void* stream) {
  if (T < 0 || L < 1 || n < 2 || n >= 32768 || kpad < n || kpad % 32 != 0 || cap < 1) return MC_ERR_CONFIG;
  if (T > 0 && (!ldig || !eL || !fdig || !eF || !gx || !ga || !lo || !cnt || !fitmask || !Sex || !Dex || !Rex))
    return MC_ERR_CONFIG;
  return cuda_status(mc::launch_refine_i8(ldig, eL, fdig, eF, T, L, n, kpad, perm, lo, cnt, gx, ga, cap, Dex, Rex,
                                          nullptr, 0, flags, S_(stream), Sex, fitmask));
}

int mc_candidates(const float* D, int32_t T, int32_t L, int64_t ldd, double lam, double thr, const double* fnorm,
                  double fcoef, const int32_t* rlo, const int32_t* rhi, const float* dref, int32_t cap, int32_t* lo,
                  int32_t* cnt, float* dmin, uint8_t* flags, void* stream) {
  if (T < 0 || L < 1 || ldd < L || cap < 1 || !(lam > 0.0) || !(thr >= 0.0) || !(fcoef >= 0.0))
    return MC_ERR_CONFIG;
  if (T > 0 && (!D || !lo || !cnt)) return MC_ERR_CONFIG;
  if ((rlo == nullptr) != (rhi == nullptr)) return MC_ERR_CONFIG;
  return cuda_status(
      mc::launch_candidates(D, T, L, ldd, lam, thr, fnorm, fcoef, rlo, rhi, dref, cap, lo, cnt, dmin, flags,
                                              S_(stream)));
}

int mc_candidates_life(const float* D, int32_t T, int32_t L, int64_t ldd, double lam, double thr,
                       const double* fnorm, double fcoef, const double* dlife, int32_t cap, int32_t* lo, int32_t* cnt,
                       float* dmin, uint8_t* flags, void* stream) {
  if (T < 0 || L < 1 || ldd < L || cap < 1 || !(lam > 0.0) || !(thr >= 0.0) || !(fcoef >= 0.0)) return MC_ERR_CONFIG;
  if (T > 0 && (!D || !lo || !cnt || !dlife)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_candidates(D, T, L, ldd, lam, thr, fnorm, fcoef, nullptr, nullptr, nullptr, cap, lo, cnt,
                                           dmin, flags, S_(stream), dlife));
}

int mc_prune_plan(const float* Dc, int32_t T, int32_t C, int64_t lddc, const double* fnorm, const double* cnorm,
                  const double* frnorm, const double* crnorm, double c_unit, const float* mind, const float* maxd, int32_t cstride, int32_t ntl, double thr,
                  int32_t knear, int32_t wide, const double* dub_in, double* dub_out, int32_t* hull_lo,
                  int32_t* hull_hi, int32_t* key, void* stream) {
  if (T < 0 || C < 1 || C > 1024 || lddc < C || ntl < 1 || knear < 1 || knear > 8 || !(c_unit >= 0.0) ||
      !(thr >= 0.0) || (maxd && cstride < 1) || ((frnorm == nullptr) != (crnorm == nullptr)))
    return MC_ERR_CONFIG;
  // bound-only pass: dub_out set, no hull outputs
  const bool hulls = hull_lo || hull_hi || key;
  if (T > 0 && (!Dc || !fnorm || !cnorm)) return MC_ERR_CONFIG;
  if (T > 0 && hulls && (!mind || !hull_lo || !hull_hi || !key)) return MC_ERR_CONFIG;
  if (T > 0 && !hulls && !dub_out) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_prune_plan(Dc, T, C, lddc, fnorm, cnorm, frnorm, crnorm, c_unit, mind, maxd, cstride,
                                           ntl, thr, knear, wide, dub_in, dub_out, hull_lo, hull_hi, key,
                                           S_(stream)));
}

int mc_band_tiles(const int32_t* perm, int32_t T, const int32_t* hull_lo, const int32_t* hull_hi, int32_t BM,
                  int32_t BL, int32_t L, int32_t* tlist, int32_t* nlist, int32_t* row_lo, int32_t* row_hi,
                  void* stream) {
  if (T < 0 || BM < 1 || BL < 1 || L < 1) return MC_ERR_CONFIG;
  if (T > 0 && (!perm || !hull_lo || !hull_hi || !tlist || !nlist || !row_lo || !row_hi)) return MC_ERR_CONFIG;
  return cuda_status(
      mc::launch_band_tiles(perm, T, hull_lo, hull_hi, BM, BL, L, tlist, nlist, row_lo, row_hi, S_(stream)));
}

int mc_gather_rows(const void* src, int32_t esz, int64_t rowlen, const int32_t* idx, int32_t rows, void* dst,
                   void* stream) {
  if ((esz != 4 && esz != 8) || rowlen < 0 || rows < 0) return MC_ERR_CONFIG;
  if (rows > 0 && rowlen > 0 && (!src || !idx || !dst)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_gather_rows(src, esz, rowlen, idx, rows, dst, S_(stream)));
}

int mc_sort_by_key(const int32_t* key, int32_t T, int32_t nbins, int32_t* bins, int32_t* perm, void* stream) {
  if (T < 0 || nbins < 1 || (T > 0 && (!key || !bins || !perm))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_sort_by_key(key, T, nbins, bins, perm, S_(stream)));
}

int mc_cov_dmma(const float* frames, const double* fcentroid, const double* fwbar, const float* landmarks,
                const double* lcentroid, const double* lwbar, const double* w, double wuni, int32_t T, int32_t L,
                int32_t n, double* S, void* stream) {
  if (T < 0 || L < 1 || n < 2 || !(wuni > 0.0)) return MC_ERR_CONFIG;
  if (T > 0 && (!frames || !fcentroid || !fwbar || !landmarks || !lcentroid || !lwbar || !w || !S))
    return MC_ERR_CONFIG;
  return cuda_status(mc::launch_refine_dmma(frames, fcentroid, landmarks, lcentroid, lwbar, w, nullptr, nullptr, fwbar,
                                            wuni, nullptr, T, L, n, nullptr, nullptr, nullptr, 0, nullptr, nullptr,
                                            nullptr, 0, nullptr, S_(stream), S));
}

int mc_close_grad_fix(int32_t T, int32_t t0, int32_t n, const uint8_t* refresh, const int32_t* ridx,
                      const double* xyeig, const double* fvec, const double* w, const float* frames,
                      const double* fcentroid, void* ds, void* dz, int32_t out_f32, void* stream) {
  if (T < 0 || t0 < 0 || n < 1) return MC_ERR_CONFIG;
  if (T > 0 && (!refresh || !ridx || !xyeig || !fvec || !w || !frames || !fcentroid || !ds || !dz))
    return MC_ERR_CONFIG;
  return cuda_status(mc::launch_close_grad_fix(T, t0, n, refresh, ridx, xyeig, fvec, w, frames, fcentroid, ds, dz,
                                               out_f32, S_(stream)));
}

int mc_refine(const float* frames, const double* fcentroid, const float* landmarks, const double* lcentroid,
              const double* lwbar, const double* w, const double* gx, const double* ga, int32_t T, int32_t L, int32_t n,
              const int32_t* perm, const int32_t* lo, const int32_t* cnt, int32_t cap, double* Dex, double* Rex,
              float* Dd, int64_t ldd, const int32_t* fmap, const double* fwbar, double wuni, uint8_t* flags,
              void* stream) {
  if (T < 0 || L < 1 || n < 2) return MC_ERR_CONFIG;
  if ((lo == nullptr) != (cnt == nullptr)) return MC_ERR_CONFIG;
  if (T > 0 && (!frames || !fcentroid || !landmarks || !lcentroid || !w || !gx || !ga)) return MC_ERR_CONFIG;
  if (!Dex && !Dd) return MC_ERR_CONFIG;
  if ((Dex || Rex) && cap < 1) return MC_ERR_CONFIG;
  if (Dd && ldd < L) return MC_ERR_CONFIG;
  // fp64 tensor-core (DMMA) tiles by default; MC_REFINE_VECTOR=1 selects the CUDA-core kernel
  static const bool vec = [] {
    const char* e = getenv("MC_REFINE_VECTOR");
    return e && e[0] == '1';
  }();
  if (vec) {
    if (fmap) return MC_ERR_CONFIG;  // the CUDA-core comparison kernel reads frames in place
    return cuda_status(mc::launch_refine(frames, fcentroid, landmarks, lcentroid, w, gx, ga, T, L, n, perm, lo, cnt,
                                         cap, Dex, Rex, Dd, ldd, flags, S_(stream)));
  }
  return cuda_status(mc::launch_refine_dmma(frames, fcentroid, landmarks, lcentroid, lwbar, w, gx, fmap, fwbar, wuni,
                                            ga, T, L, n, perm, lo, cnt, cap, Dex, Rex, Dd, ldd, flags, S_(stream)));
}

int mc_pair_grad(int64_t P, int32_t n, int32_t npad, const double* xplanes, const double* aplanes, const int32_t* xi,
                 const int32_t* ai, const double* rot, const double* w, const double* w_align, const double* xwbar,
                 const double* awbar, const int32_t* approx, const int32_t* yi, const double* S, const double* amom,
                 const double* xyeig, const double* rxy, const double* gx, const double* ga, double* value,
                 double* grad, void* stream) {
  if (P < 0 || bad_pad(n, npad)) return MC_ERR_CONFIG;
  if (P > 0 && (!xplanes || !aplanes || !xi || !ai || !rot || !w || !w_align || !xwbar || !awbar || !grad))
    return MC_ERR_CONFIG;
  if (approx && (!yi || !S || !amom || !xyeig || !rxy || !gx || !ga || !value)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_pair_grad(P, n, npad, xplanes, aplanes, xi, ai, rot, w, w_align, xwbar, awbar, approx,
                                          yi, S, amom, xyeig, rxy, gx, ga, value, grad, S_(stream)));
}

int mc_property_map(int32_t L, int32_t n, const double* D, const double* grads, const double* q, double lam,
                    double* out, double* ds, double* dz, void* stream) {
  if (L < 1) return MC_ERR_EMPTY_ACTIVE_SET;
  if (!(lam > 0.0) || !D || !q || !out || (grads && (n < 1 || !ds || !dz))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_property_map(L, n, D, grads, q, lam, out, ds, dz, S_(stream)));
}

int mc_center_split(const void* coords, int dtype, int64_t count, int32_t n, int32_t kpad, const double* w_align,
                    const double* w_disp, int32_t weighted, float* hi, float* lo, double* centroid, double* gnorm,
                    double* wbar, double* mom, uint8_t* flags, void* stream) {
  if (dtype != MC_F32 && dtype != MC_F64) return MC_ERR_CONFIG;
  if (n < 2) return MC_ERR_INVALID_STRUCTURE;
  if (count < 0 || kpad < n || kpad % 16 != 0) return MC_ERR_CONFIG;
  if (count > 0 && (!coords || !w_align || !w_disp || !hi || !lo || !gnorm)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_center_split(coords, dtype, count, n, kpad, w_align, w_disp, weighted, hi, lo, centroid,
                                             gnorm, wbar, mom, flags, S_(stream)));
}

int mc_msd_tf32(const float* fhi, const float* flo, const float* lhi, const float* llo, const double* gx,
                const double* ga, int32_t T, int32_t L, int32_t kpad, float* D, int64_t ldd, int32_t grid,
                void* stream) {
  if (T < 0 || L < 0 || kpad % 16 != 0 || kpad < 16 || ldd < L) return MC_ERR_CONFIG;
  if ((int64_t)T * L > 0 && (!fhi || !flo || !lhi || !llo || !gx || !ga || !D)) return MC_ERR_CONFIG;
  if (3LL * T > 0x7fffffffLL || 3LL * L > 0x7fffffffLL) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_msd_tf32(fhi, flo, lhi, llo, gx, ga, T, L, kpad, D, ldd, grid, S_(stream)));
}

int mc_center_split16(const void* coords, int dtype, int64_t count, int32_t n, int32_t kpad, const double* w_align,
                      const double* w_disp, int32_t weighted, int32_t terms, void* hl, double* scale_inv,
                      double* opnorm, double* rnorm, double* centroid, double* gnorm, double* wbar, double* mom,
                      uint8_t* flags, void* stream) {
  if (dtype != MC_F32 && dtype != MC_F64) return MC_ERR_CONFIG;
  if (n < 2) return MC_ERR_INVALID_STRUCTURE;
  if (terms != 1 && terms != 3) return MC_ERR_CONFIG;
  if (count < 0 || kpad < n || kpad % (terms == 1 ? 64 : 32) != 0) return MC_ERR_CONFIG;
  if (count > 0 && (!coords || !w_align || !w_disp || !hl || !scale_inv || !gnorm)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_center_split16(coords, dtype, count, n, kpad, w_align, w_disp, weighted, terms, hl,
                                               scale_inv, opnorm, rnorm, centroid, gnorm, wbar, mom, flags,
                                               S_(stream)));
}

int mc_center_split16_uniform(const float* coords, int64_t count, int32_t n, int32_t kpad, double wuni, void* hl,
                              double* scale_inv, double* opnorm, double* rnorm, double* centroid, double* gnorm,
                              double* wbar, uint8_t* flags, int32_t* dexp, void* stream) {
  if (n < 2) return MC_ERR_INVALID_STRUCTURE;
  if (count < 0 || kpad < n || kpad % 64 != 0 || n % 4 != 0 || !(wuni > 0.0)) return MC_ERR_CONFIG;
  if (count > 0 && (!coords || !hl || !scale_inv || !gnorm || (reinterpret_cast<uintptr_t>(coords) & 15)))
    return MC_ERR_CONFIG;
  return cuda_status(mc::launch_center_split16_uniform(coords, count, n, kpad, wuni, hl, scale_inv, opnorm, rnorm,
                                                       centroid, gnorm, wbar, flags, dexp, S_(stream)));
}

static int msd_f16_args(const void* fhl, const void* lhl, const double* fsc, const double* lsc, const double* gx,
                        const double* ga, int32_t T, int32_t L, int32_t kpad, int32_t terms, const float* D,
                        int64_t ldd) {
  if (terms != 1 && terms != 3) return MC_ERR_CONFIG;
  if (T < 0 || L < 0 || kpad % (terms == 1 ? 64 : 32) != 0 || kpad < 32 || ldd < L) return MC_ERR_CONFIG;
  if ((int64_t)T * L > 0 && (!fhl || !lhl || !fsc || !lsc || !gx || !ga || !D)) return MC_ERR_CONFIG;
  if (3LL * T > 0x7fffffffLL || 3LL * L > 0x7fffffffLL) return MC_ERR_CONFIG;
  return MC_OK;
}

int mc_msd_f16(const void* fhl, const void* lhl, const double* fscale, const double* lscale, const double* gx,
               const double* ga, int32_t T, int32_t L, int32_t kpad, int32_t terms, const int32_t* tlist,
               const int32_t* nlist, float* D, int64_t ldd, int32_t grid, void* stream) {
  const int st = msd_f16_args(fhl, lhl, fscale, lscale, gx, ga, T, L, kpad, terms, D, ldd);
  if (st != MC_OK) return st;
  if ((tlist == nullptr) != (nlist == nullptr)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_msd_f16(fhl, lhl, fscale, lscale, gx, ga, T, L, kpad, terms, D, ldd, grid, S_(stream),
                                        tlist, nlist));
}

int mc_msd_f16_2sm(const void* fhl, const void* lhl, const double* fscale, const double* lscale, const double* gx,
                   const double* ga, int32_t T, int32_t L, int32_t kpad, float* D, int64_t ldd, int32_t grid,
                   void* stream) {
  const int st = msd_f16_args(fhl, lhl, fscale, lscale, gx, ga, T, L, kpad, 3, D, ldd);
  if (st != MC_OK) return st;
  return cuda_status(mc::launch_msd_f16_2sm(fhl, lhl, fscale, lscale, gx, ga, T, L, kpad, D, ldd, grid, S_(stream)));
}

static bool bad_grid(int32_t d, const double* lo, const double* hi, const int32_t* bins) {
  if (d < 1 || d > 2 || !lo || !hi || !bins) return true;
  for (int i = 0; i < d; ++i)
    if (!(hi[i] > lo[i]) || bins[i] < 1) return true;
  return false;
}

int mc_mtd_bias_direct(const double* cv, int32_t T, int32_t d, const double* centers, const double* sigmas,
                       const double* heights, int32_t H, double* V, double* dV, void* stream) {
  if (T < 0 || d < 1 || d > 3 || H < 0) return MC_ERR_CONFIG;
  if (T > 0 && (!cv || !V || !dV || (H > 0 && (!centers || !sigmas || !heights)))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_mtd_bias(cv, T, d, centers, sigmas, heights, H, V, dV, S_(stream)));
}

int mc_mtd_grid_deposit(double* val, double* dgrid, double* dxy, int32_t d, const double* lo, const double* hi,
                        const int32_t* bins, const double* center, const double* sigma, double height, double cutoff,
                        uint8_t* flag, void* stream) {
  if (bad_grid(d, lo, hi, bins) || !val || !dgrid || (d == 2 && !dxy) || !center || !sigma) return MC_ERR_CONFIG;
  if (!(height >= 0.0) || !(cutoff > 0.0)) return MC_ERR_CONFIG;
  return cuda_status(
      mc::launch_mtd_deposit(val, dgrid, dxy, d, lo, hi, bins, center, sigma, height, cutoff, flag, S_(stream)));
}

int mc_mtd_grid_eval(const double* val, const double* dgrid, const double* dxy, int32_t d, const double* lo,
                     const double* hi, const int32_t* bins, const double* cv, int32_t T, double* V, double* dV,
                     uint8_t* flags, void* stream) {
  if (bad_grid(d, lo, hi, bins) || T < 0) return MC_ERR_CONFIG;
  if (T > 0 && (!val || !dgrid || (d == 2 && !dxy) || !cv || !V || !dV)) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_mtd_eval(val, dgrid, dxy, d, lo, hi, bins, cv, T, V, dV, flags, S_(stream)));
}

int mc_mtd_force(const double* dV, int32_t T, int32_t d, const void* g0, const void* g1, const void* g2, int dtype,
                 int32_t n, void* F, void* stream) {
  if (dtype != MC_F32 && dtype != MC_F64) return MC_ERR_CONFIG;
  if (T < 0 || n < 1 || d < 1 || d > 3) return MC_ERR_CONFIG;
  if (T > 0 && (!dV || !g0 || !F || (d > 1 && !g1) || (d > 2 && !g2))) return MC_ERR_CONFIG;
  return cuda_status(mc::launch_mtd_force(dV, T, d, g0, g1, g2, dtype, n, F, S_(stream)));
}

int mc_toysim_run(int32_t W, int32_t n, int32_t L, int32_t steps, int64_t step0, int32_t mode, int32_t tau_g,
                  int32_t max_hills, int32_t traj_stride, double bond_k, double bond_r0, double angle_k,
                  double theta0, double mob, double noise, double lam, double eps, double hill_h, double hill_sigma,
                  uint64_t seed, const double* refs, const double* refg, const double* refmom, const double* q,
                  const double* w, const double* wa, double* x, double* y, double* rays, int32_t* hasy,
                  double* hills, int32_t* nhills, int64_t* counters, double* cv, uint8_t* rlog, double* traj,
                  uint8_t* flags, int32_t nl_m, int32_t nl_stride, uint8_t* act, int64_t* nl_last, void* stream) {
  if (W < 0 || n < 3 || n > 64 || steps < 0 || step0 < 0 || mode < 0 || mode > 2 || tau_g < 0 || max_hills < 0 ||
      traj_stride < 0 || !(mob > 0.0) || !(noise >= 0.0) || !(bond_r0 > 0.0))
    return MC_ERR_CONFIG;
  if (nl_m < 0 || (nl_m > 0 && (mode == 0 || nl_m > L || nl_stride < 1 || (W > 0 && (!act || !nl_last)))))
    return MC_ERR_CONFIG;  // neighbour list: 1 <= M <= N, stride >= 1
  if (mode != 0 && (L < 1 || L > 128 || !(lam > 0.0) || !(eps >= 0.0) || !(hill_sigma > 0.0) || !(hill_h >= 0.0)))
    return MC_ERR_CONFIG;
  if (traj_stride > 0 && step0 % traj_stride != 0) return MC_ERR_CONFIG;
  if (W > 0 && steps > 0) {
    if (!x || !y || !w || !wa || !hasy || !nhills || !counters || (traj_stride > 0 && !traj)) return MC_ERR_CONFIG;
    if (mode != 0 && (!refs || !refg || !refmom || !q || !cv || !rlog || (max_hills > 0 && !hills)))
      return MC_ERR_CONFIG;
    if (mode == 2 && !rays) return MC_ERR_CONFIG;
  }
  mc::ToyParams P{n, L, steps, mode, tau_g, max_hills, traj_stride, (long long)step0, bond_k, bond_r0, angle_k,
                  theta0, mob, noise, lam, eps, hill_h, hill_sigma, (unsigned long long)seed, nl_m, nl_stride};
  return cuda_status(mc::launch_toysim(P, W, refs, refg, refmom, q, w, wa, x, y, rays, hasy, hills, nhills,
                                       reinterpret_cast<long long*>(counters), cv, rlog, traj, flags, S_(stream), act,
                                       reinterpret_cast<long long*>(nl_last)));
}

}  // extern "C"
