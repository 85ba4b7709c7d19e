// Internal host launchers (one per kernel family); capi.cu wraps them in the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace mc {
cudaError_t launch_center(const void* coords, int dtype, int64_t count, int n, int npad, const double* w_align,
                          const double* w_disp, double* planes, double* wplanes, double* centroid, double* gnorm,
                          double* wbar, double* mom, uint8_t* flags, cudaStream_t stream);
cudaError_t launch_cov_f64(const double* fpl, const double* lpl, int T, int L, int npad, double* S,
                           cudaStream_t stream);
cudaError_t launch_cov_pairs(const double* xpl, const double* apl, const int* xi, const int* ai, int64_t P,
                             int npad, const double* w, double* S, cudaStream_t stream);
cudaError_t launch_fit_dense(const double* S, int T, int L, const double* gx, const double* ga,
                             const uint8_t* rowmask, double* D, double* rot, double* quat, uint8_t* flags,
                             cudaStream_t stream);
cudaError_t launch_fit_list_msd(const double* S, int64_t P, const int* xi, const int* ai, const double* gx,
                                const double* ga, double* D, cudaStream_t stream);
cudaError_t launch_fit_full(const double* S, int64_t P, const int* xi, const int* ai, const double* gx,
                            const double* ga, double* eig, double* quat, double* rot, uint8_t* flags,
                            cudaStream_t stream);
cudaError_t launch_rot_grad(const double* xpl, const double* apl, const int* xi, const int* ai, int64_t P, int n,
                            int npad, const double* w, const double* eig, double* out, cudaStream_t stream);
cudaError_t launch_jacobi_n(const double* mats, int64_t B, int n, double tol, int max_sweeps, double* vals,
                            double* vecs, uint8_t* flags, cudaStream_t stream);
cudaError_t launch_jacobi4(const double* mats, int64_t B, double* vals, double* vecs, uint8_t* flags,
                           cudaStream_t stream);
cudaError_t launch_window_pairs(int walkers, int steps, int K, int* xi, int* ai, cudaStream_t stream);
cudaError_t launch_close_scan(const double* fpl, const double* gx, int walkers, int steps, int npad,
                              const double* w, const double* dwin, int K, double eps, uint8_t* refresh, int* ridx,
                              double* dxy, int* n_onthefly, cudaStream_t stream);
cudaError_t launch_xy_eig(const double* fpl, const double* gx, int64_t T, int npad, const double* w,
                          const uint8_t* refresh, const int* ridx, double* xyeig, double* rxy, uint8_t* flags,
                          cudaStream_t stream);
cudaError_t launch_shard_rescale(int T, int cap, const int* nsig, const double* alpha, const double* beta,
                                 double* sig_coef, double* fvec, cudaStream_t stream);
cudaError_t launch_cv_weights(int T, int t0, int L, double lam, double cutoff, int cap, int ld, const int* rowlo,
                              const int* rowcnt, double* D, const double* q,
                              const double* R, const double* fwbar, const double* lwbar, const uint8_t* refresh,
                              const int* ridx, const double* S, const double* rxy, const double* xyeig,
                              const double* gx, const double* ga, const double* lmom, double* s, double* z,
                              int* sig_idx, double* sig_coef, int* nsig, double* fvec, uint8_t* flags,
                              cudaStream_t stream, const int* nb_idx = nullptr, const int* nb_row = nullptr,
                              int nb_m = 0, int dmode = 0);
cudaError_t launch_mtd_bias(const double* cv, int T, int d, const double* centers, const double* sigmas,
                            const double* heights, int H, double* V, double* dV, cudaStream_t stream);
cudaError_t launch_mtd_deposit(double* val, double* dgrid, double* dxy, int d, const double* lo, const double* hi,
                               const int* bins, const double* center, const double* sigma, double height,
                               double cutoff, uint8_t* flag, cudaStream_t stream);
cudaError_t launch_mtd_eval(const double* val, const double* dgrid, const double* dxy, int d, const double* lo,
                            const double* hi, const int* bins, const double* cv, int T, double* V, double* dV,
                            uint8_t* flags, cudaStream_t stream);
cudaError_t launch_mtd_force(const double* dV, int T, int d, const void* g0, const void* g1, const void* g2,
                             int dtype, int n, void* F, cudaStream_t stream);
cudaError_t launch_topm(const void* D, int dtype, int nrows, int L, int64_t ldd, const int* rows, int M, int* idx,
                        cudaStream_t stream);
cudaError_t launch_close_grad_fix(int T, int t0, int n, const uint8_t* refresh, const int* ridx, const double* xyeig,
                                  const double* fvec, const double* w, const float* fraw, const double* fcen, void* ds,
                                  void* dz, int out_f32, cudaStream_t stream);
cudaError_t launch_cv_grad(int T, int n, int npad, int cap, const double* fpl, const double* lpl, const double* w,
                           const double* wa, const int* sig_idx, const double* sig_coef, const int* nsig,
                           const double* fvec, const uint8_t* refresh, const int* ridx, const double* xyeig,
                           void* ds, void* dz, int out_f32, const float* fraw, const double* fcen,
                           const float* lraw, const double* lcen, const int* perm, cudaStream_t stream);
cudaError_t launch_msd_tf32_2sm(const float* fh, const float* fl, const float* lh, const float* ll, const double* gx,
                                const double* ga, int T, int L, int kpad, float* D, int64_t ldd, int grid,
                                cudaStream_t stream);
cudaError_t launch_cv_grad_dmma(int T, int n, int cap, const float* fraw, const double* fcen, const float* lraw,
                                const double* lcen, const double* w, const double* wa, const int* sig_idx,
                                const double* sig_coef, const int* nsig, const double* fvec, const int* perm,
                                const int* out_map, void* ds, void* dz, int out_f32, cudaStream_t stream,
                                int min_width = -1, int i8_dg = 0);
cudaError_t launch_ldig(const float* lraw, const double* lcen, int L, int n, int npad, int kpad, int* eB,
                        int8_t* dig, cudaStream_t stream);
cudaError_t launch_cv_grad_i8(int T, int n, int cap, const float* fraw, const double* fcen, const float* lraw,
                              const double* lcen, const double* w, const double* wa, const int8_t* dig, const int* eB,
                              int npad, int kpad, const int* sig_idx, const double* sig_coef, const int* nsig,
                              const double* fvec, const double* dV, const int* perm, const int* out_map, void* out0,
                              void* out1, int out_f32, int ncv, int* wide_flag, void* ws, size_t ws_bytes,
                              cudaStream_t stream);
size_t grad_i8_workspace(int T, int ncv);
cudaError_t launch_center_split16_uniform(const float* coords, int64_t B, int n, int kpad, double wuni, void* hl,
                                          double* scale_inv, double* opnorm, double* rnorm, double* centroid,
                                          double* gnorm, double* wbar, uint8_t* flags, int* dexp,
                                          cudaStream_t stream);
cudaError_t launch_grad_i8_plan(int T, int cap, int ncv, const int* sig_idx, const int* nsig, const int* perm,
                                long long* bytes, cudaStream_t stream);
size_t grad_i8_wide_header_bytes(int nwide, int ncv);
cudaError_t launch_cv_grad_i8_wide(int T, int n, int cap, const float* fraw, const double* fcen, const double* w,
                                   const double* wa, const int8_t* dig, const int* eB, int npad, int kpad,
                                   const int* sig_idx, const double* sig_coef, const int* nsig, const double* fvec,
                                   const double* dV, const int* perm, const int* out_map, void* out0, void* out1,
                                   int out_f32, int ncv, const int* wide_ids, int nwide, const long long* wide_off,
                                   void* hws, void* wimg, cudaStream_t stream);
cudaError_t launch_rdig(const float* raw, const double* cen, const double* w, const int* perm, const int* fmap, int B,
                        int n, int kpad, int8_t* dig, int* e, cudaStream_t stream, const int* ein = nullptr,
                        int planes = 0);
cudaError_t launch_refine_i8(const int8_t* ldig, const int* eL, const int8_t* fdig, const int* eF, int T, int L, int n,
                             int kpad, const int* perm, const int* lo, const int* cnt, const double* gx,
                             const double* ga, int cap, double* Dex, double* Rex, float* Dd, int64_t ldd,
                             uint8_t* flags, cudaStream_t stream, double* Sex = nullptr,
                             const uint8_t* fitmask = nullptr);
cudaError_t launch_cv_grad_block(int T, int n, int cap, const float* fraw, const double* fcen, const float* lraw,
                                 const double* lcen, const double* w, const double* wa, const int* sig_idx,
                                 const double* sig_coef, const int* nsig, const double* fvec, const int* perm,
                                 void* ds, void* dz, int out_f32, cudaStream_t stream);
cudaError_t launch_cv_grad_block_planes(int T, int t0, int n, int npad, int cap, const double* fpl, const double* lpl,
                                        const double* w, const double* wa, const int* sig_idx,
                                        const double* sig_coef, const int* nsig, const double* fvec,
                                        const uint8_t* refresh, const int* ridx, const double* xyeig, void* ds,
                                        void* dz, int out_f32, cudaStream_t stream);
cudaError_t launch_candidates(const float* D, int T, int L, int64_t ldd, double lam, double thr, const double* fnorm,
                              double fcoef, const int* rlo, const int* rhi, const float* dref, int cap, int* lo,
                              int* cnt, float* dmin, uint8_t* flags, cudaStream_t stream,
                              const double* dlife = nullptr);
cudaError_t launch_sort_by_key(const int* key, int T, int nbins, int* bins, int* perm, cudaStream_t stream);
cudaError_t launch_refine_dmma(const float* fr, const double* fc, const float* lr, const double* lc,
                               const double* lwbar, const double* w, const double* gx, const int* fmap,
                               const double* fwbar, double wuni, const double* ga, int T, int L, int n,
                               const int* perm, const int* lo, const int* cnt, int cap, double* Dex, double* Rex,
                               float* Dd, int64_t ldd, uint8_t* flags, cudaStream_t stream, double* Sout = nullptr);
cudaError_t launch_refine(const float* fr, const double* fc, const float* lr, const double* lc, const double* w,
                          const double* gx, const double* ga, int T, int L, int n, const int* perm, const int* lo,
                          const int* cnt, int cap, double* Dex, double* Rex, float* Dd, int64_t ldd, uint8_t* flags,
                          cudaStream_t stream);
cudaError_t launch_pair_grad(int64_t P, int n, int npad, const double* xpl, const double* apl, const int* xi,
                             const int* ai, const double* rot, const double* w, const double* wa, const double* xwbar,
                             const double* awbar, const int* approx, const int* yi, const double* S,
                             const double* amom, const double* xyeig, const double* rxy, const double* gx,
                             const double* ga, double* value, double* grad, cudaStream_t stream);
cudaError_t launch_property_map(int L, int n, const double* D, const double* grads, const double* q, double lam,
                                double* out, double* ds, double* dz, cudaStream_t stream);
cudaError_t launch_center_split(const void* coords, int dtype, int64_t B, int n, int kpad, const double* w_align,
                                const double* w_disp, int weighted, float* hi, float* lo, double* centroid,
                                double* gnorm, double* wbar, double* mom, uint8_t* flags, cudaStream_t stream);
cudaError_t launch_msd_tf32(const float* fh, const float* fl, const float* lh, const float* ll, const double* gx,
                            const double* ga, int T, int L, int kpad, float* D, int64_t ldd, int grid,
                            cudaStream_t stream);
cudaError_t launch_center_split16(const void* coords, int dtype, int64_t B, int n, int kpad, const double* w_align,
                                  const double* w_disp, int weighted, int terms, void* hl, double* scale_inv,
                                  double* opnorm, double* rnorm, double* centroid, double* gnorm, double* wbar,
                                  double* mom, uint8_t* flags, cudaStream_t stream);
cudaError_t launch_msd_f16(const void* fhl, const void* lhl, const double* fsc, const double* lsc, const double* gx,
                           const double* ga, int T, int L, int kpad, int terms, float* D, int64_t ldd, int grid,
                           cudaStream_t stream, const int* tlist = nullptr, const int* nlist = nullptr);
cudaError_t launch_prune_plan(const float* Dc, int T, int C, int64_t lddc, const double* fnorm, const double* cnorm,
                              const double* frnorm, const double* crnorm, double c_unit, const float* mind, const float* maxd, int cstride, int ntl, double thr,
                              int knear, int wide, const double* dub_in, double* dub_out, int* hull_lo, int* hull_hi,
                              int* key, cudaStream_t stream);
cudaError_t launch_band_tiles(const int* perm, int T, const int* hull_lo, const int* hull_hi, int BM, int BL, int L,
                              int* tlist, int* nlist, int* row_lo, int* row_hi, cudaStream_t stream);
cudaError_t launch_gather_rows(const void* src, int esz, int64_t rowlen, const int* idx, int rows, void* dst,
                               cudaStream_t stream);
cudaError_t launch_msd_f16_2sm(const void* fhl, const void* lhl, const double* fsc, const double* lsc,
                               const double* gx, const double* ga, int T, int L, int kpad, float* D, int64_t ldd,
                               int grid, cudaStream_t stream);
struct ToyParams {  // csrc/toysim.cu
  int n, L, steps, mode, tau_g, max_hills, traj_stride;
  long long step0;
  double bond_k, bond_r0, angle_k, theta0, mob, noise, lam, eps, hill_h, hill_sigma;
  unsigned long long seed;
  int nl_m, nl_stride;  // neighbour list (SPEC neighbourlist): size M (0: none) and stride
};
cudaError_t launch_toysim(const ToyParams& P, int W, const double* refs, const double* refg, const double* refmom,
                          const double* q, const double* w, const double* wa, double* xs, double* ys, double* rays,
                          int* hasy, double* hills, int* nhills, long long* counters, double* cv, uint8_t* rlog,
                          double* traj, uint8_t* flags, cudaStream_t stream, uint8_t* act = nullptr,
                          long long* nl_last = nullptr);
}  // namespace mc
