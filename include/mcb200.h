/*
 * mcb200.h — C ABI of libmcb200.so, the B200 (sm_100a) implementation of the
 * aligned-MSD / path-CV / floating-close-structure hot path of
 * arXiv 1801.02362 (reference: /root/reference/pkg/src/metadyn_close).
 *
 * The reference is a pure-Python package with no FFI; its boundary is the
 * Python call surface of geometry.py plus the SPEC.md msd-engine / colvar
 * operations.  Each entry point below is the device primitive that a
 * maintainer would bind (ctypes / cffi) underneath the
 * reference call named in its comment.
 *
 * Conventions
 *  - All array pointers are DEVICE pointers owned by the caller; the library
 *    allocates nothing, frees nothing and keeps no global state.  Calls are
 *    stream-ordered on `stream` (a cudaStream_t passed as void*; NULL = the
 *    legacy default stream) and re-entrant across streams and devices.
 *  - Centred structures live as zero-padded fp64 planes [count, 3, npad]
 *    (npad a multiple of 32, npad >= n); padding atoms carry zero weight.
 *  - Covariances S are [.., 9] fp64 with S[b*3+g] = sum_j w_j x_{j,b} a_{j,g}
 *    (x fitted, a reference), so that the reference's Kearsley matrix is
 *    K = (Gx + Ga) I - 2 N_Horn(S) and eigvals[0] = the weighted MSD.
 *  - Eigen records are [.., 20] fp64: 4 ascending eigenvalues of K, then the
 *    4x4 eigenvector matrix row-major (columns = eigenvectors, each with its
 *    largest-|component| positive, geometry.py:149-152).
 *  - Return value: MC_OK or a negative status.  Per-item faults are reported
 *    through optional uint8 flag arrays (MC_FLAG_*); the Python shim raises
 *    the matching metadyn_close error class (errors.py:4-35).
 */
#ifndef MCB200_H
#define MCB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (errors.py:4-35) */
#define MC_OK 0
#define MC_ERR_INVALID_STRUCTURE (-1) /* InvalidStructureError  errors.py:8  */
#define MC_ERR_DEGENERATE_FIT (-2)    /* DegenerateFitError     errors.py:12 */
#define MC_ERR_CONFIG (-3)            /* ConfigError            errors.py:16 */
#define MC_ERR_OUT_OF_GRID (-4)       /* OutOfGridError         errors.py:20 */
#define MC_ERR_EMPTY_ACTIVE_SET (-5)  /* EmptyActiveSetError    errors.py:24 */
#define MC_ERR_CUDA_BASE (-100)       /* -100 - cudaError_t                  */

/* per-item flags */
#define MC_FLAG_DEGENERATE 1u   /* eigvals[1]-eigvals[0] < 1e-9 (geometry.py:251-256) */
#define MC_FLAG_NO_CONVERGE 2u  /* Jacobi exceeded 60 sweeps (geometry.py:144-145)    */
#define MC_FLAG_NON_FINITE 4u   /* non-finite coordinates or results (geometry.py:41) */
#define MC_FLAG_ADJ_FALLBACK 8u /* informational: Jacobi used instead of adjugate      */
#define MC_FLAG_SIG_OVERFLOW 16u /* significant-landmark list exceeded its capacity     */
#define MC_FLAG_OUT_OF_GRID 32u /* CV value / hill centre outside the bias grid (SPEC metadynamics) */

/* dtypes */
#define MC_F32 0
#define MC_F64 1

int mc_version(void);

/* K1 — Structure.center / centroid batched (geometry.py:67-84).
 * coords [count, n, 3] (dtype), weights [n] normalised (geometry.py:49-61).
 * Writes centred planes, optional w-weighted planes, centroid [count,3],
 * G = sum w|x_c|^2 [count], wbar = sum w x_c [count,3], mom = sum w x_c x_c^T
 * (xx,xy,xz,yy,yz,zz) [count,6]; flags [count] (MC_FLAG_NON_FINITE). */
int mc_center(const void* coords, int dtype, int64_t count, int32_t n, int32_t npad, const double* w_align,
              const double* w_disp, double* planes, double* wplanes, double* centroid, double* gnorm,
              double* wbar, double* mom, uint8_t* flags, void* stream);

/* All-pairs covariance (the linear part of _kearsley_matrix, geometry.py:180-196),
 * fp64 CUDA-core tiles: S [T, L, 9] from frame planes and w-weighted landmark planes. */
int mc_cov_f64(const double* fplanes, const double* lwplanes, int32_t T, int32_t L, int32_t npad, double* S,
               void* stream);

/* Listed-pair covariance: S[p] for (xplanes[xi[p]], aplanes[ai[p]]) with weights w
 * (xi/ai NULL = identity; ai[p] < 0 gives S = 0).  One warp per pair. */
int mc_cov_pairs(const double* xplanes, const double* aplanes, const int32_t* xi, const int32_t* ai, int64_t P,
                 int32_t npad, const double* w, double* S, void* stream);

/* K3 — kearsley_fit without derivatives, dense frame x landmark (geometry.py:227-249):
 * D [T,L] = eigvals[0]; optional rot [T,L,9], quat [T,L,4], flags [T,L].
 * Rows with rowmask[t] == 0 are skipped (rowmask may be NULL). */
int mc_fit_dense(const double* S, int32_t T, int32_t L, const double* gx, const double* ga,
                 const uint8_t* rowmask, double* D, double* rot, double* quat, uint8_t* flags, void* stream);

/* Listed pairs, MSD only: D[p] = eigvals[0] of (S[p], gx[xi[p]], ga[ai[p]]). */
int mc_fit_list_msd(const double* S, int64_t P, const int32_t* xi, const int32_t* ai, const double* gx,
                    const double* ga, double* D, void* stream);

/* Full spectrum with the reference Jacobi (jacobi_eigh on K, geometry.py:106-153,
 * 246-249): eig [P,20], quat [P,4], rot [P,9], flags [P]. */
int mc_fit_full(const double* S, int64_t P, const int32_t* xi, const int32_t* ai, const double* gx,
                const double* ga, double* eig, double* quat, double* rot, uint8_t* flags, void* stream);

/* RotationFit.rot_grad (geometry.py:251-262 with _kearsley_matrix_grad :199-224 and
 * _rot_quat_jacobian :167-177): out [P, n, 3, 3, 3] = dR_{bg}/dx_{k,alpha}. */
int mc_rot_grad(const double* xplanes, const double* aplanes, const int32_t* xi, const int32_t* ai, int64_t P,
                int32_t n, int32_t npad, const double* w, const double* eig, double* out, void* stream);

/* jacobi_eigh (geometry.py:106-153) for general symmetric n x n matrices (1 <= n <= 48),
 * mats [B, n, n] row-major, any tolerance / sweep limit: vals [B, n] ascending, vecs
 * [B, n, n] (columns = eigenvectors, largest-|component| positive), flags [B]
 * (MC_FLAG_NO_CONVERGE when max_sweeps were not enough: geometry.py:144-145). */
int mc_jacobi_n(const double* mats, int64_t B, int32_t n, double tol, int32_t max_sweeps, double* vals, double* vecs,
                uint8_t* flags, void* stream);
/* jacobi_eigh (geometry.py:106-153) on B symmetric 4x4 matrices [B,16]:
 * vals [B,4] ascending, vecs [B,16] row-major. */
int mc_jacobi4(const double* mats, int64_t B, double* vals, double* vecs, uint8_t* flags, void* stream);

/* K5 — close-structure driver (Alg. 2).
 * mc_window_pairs: index lists for D(x_s, x_{s-k}), k=1..K, per walker.
 * mc_close_scan: sequential refresh decisions, one CTA per walker, from the window
 *   dwin [walkers*steps, K]; on-the-fly fits beyond the window.  Outputs refresh [.]
 *   (uint8), ridx [.] (global index of the close structure y), dxy [.] = D(x, y)
 *   (0 on the first frame), n_onthefly [walkers] (nullable).
 * mc_xy_eig: x<->y spectrum (eig record) and R_xy for every non-refresh frame. */
int mc_window_pairs(int32_t walkers, int32_t steps, int32_t K, int32_t* xi, int32_t* ai, void* stream);
int mc_close_scan(const double* fplanes, const double* gx, int32_t walkers, int32_t steps, int32_t npad,
                  const double* w, const double* dwin, int32_t K, double eps, uint8_t* refresh, int32_t* ridx,
                  double* dxy, int32_t* n_onthefly, void* stream);
int mc_xy_eig(const double* fplanes, const double* gx, int64_t T, int32_t npad, const double* w,
              const uint8_t* refresh, const int32_t* ridx, double* xyeig, double* rxy, uint8_t* flags, void* stream);

/* K4 — property-map s (Eq. 2), path-CV z, and their gradients
 * through Eq. 4 (exact rows) or Eq. 5/6 (non-refresh rows).
 * Both process frames t0 .. t0+T-1 of the (global) frame arrays; the
 * significant-list buffers (sig_idx, sig_coef, nsig, fvec, flags) are local to
 * the launch (row t - t0), so long trajectories are processed in chunks.
 * mc_pathcv_weights: per frame — min/LSE, s, z, significant-landmark list
 *   (sig_idx [T,cap], sig_coef [T,cap,18]), nsig [T], fvec [T,16]; writes the
 *   Eq. 5 distances of non-refresh rows into D.  refresh == NULL: all rows exact.
 *   Rows are dense (ld = L, rowlo = rowcnt = NULL) or sparse windows: row t of
 *   D/R (stride ld) holds landmarks rowlo[t] .. rowlo[t]+rowcnt[t]-1 (the
 *   refined candidates of the tensor-core path; landmarks outside a window
 *   have lam (D - D_min) > cutoff and weight < e^-cutoff).  With refresh and
 *   windows (the pruned close replay) a non-refresh row t has the window of its
 *   close structure ridx[t]: S row t and R row ridx[t] share the slot layout.
 * mc_pathcv_grad: one pass over atoms writing ds, dz [T, n, 3] (fp64, or fp32 if
 *   out_f32).  Coordinates from centred fp64 planes, or (fplanes/lplanes NULL)
 *   from raw fp32 AoS input + fp64 centroids.  perm (nullable): frame visiting order
 *   (the candidate sort, so neighbouring CTAs share landmarks in L2). */
int mc_pathcv_weights(int32_t T, int32_t t0, int32_t L, double lam, double cutoff, int32_t cap, int32_t ld, const int32_t* rowlo,
                      const int32_t* rowcnt, double* D, const double* q, const double* R, const double* fwbar,
                      const double* lwbar, const uint8_t* refresh, const int32_t* ridx, const double* S,
                      const double* rxy, const double* xyeig, const double* gx, const double* ga, const double* lmom,
                      double* s, double* z, int32_t* sig_idx, double* sig_coef, int32_t* nsig, double* fvec,
                      uint8_t* flags, void* stream);
/* Landmark-sharded evaluation (north_star "landmarks sharded ...
 * all-reduce of the per-frame exp-weighted partial sums"): after the host merged every
 * shard's (s_g, z_g) into s, z, it rescales this shard's K4 coefficients to the global
 * softmax, cs' = alpha (cs + beta cz), cz' = alpha cz with alpha[t] = Z_g / Z and
 * beta[t] = -lam (s_g - s) -- sig_coef [T, cap, 18] (first nsig[t] entries) and fvec
 * [T, 16] in place -- so mc_pathcv_grad_block then writes this shard's share of the
 * global gradients (replaces the SPEC property_map gradient, for the
 * shard's landmarks). */
int mc_shard_rescale(int32_t T, int32_t cap, const int32_t* nsig, const double* alpha, const double* beta,
                     double* sig_coef, double* fvec, void* stream);
/* Neighbour-list variant of mc_pathcv_weights on dense rows (SPEC neighbourlist +
 * colvar active set): row t sums over the nb_m landmarks
 * nb_idx[nb_row[t] * nb_m ..] only.  dmode 1 writes the row distances (Eq. 5 on
 * non-refresh rows) into D and returns; dmode 2 takes D as already filled. */
int mc_pathcv_weights_nl(int32_t T, int32_t t0, int32_t L, double lam, double cutoff, int32_t cap,
                         const int32_t* nb_idx, const int32_t* nb_row, int32_t nb_m, int32_t dmode, double* D,
                         const double* q, const double* R, const double* fwbar, const double* lwbar,
                         const uint8_t* refresh, const int32_t* ridx, const double* S, const double* rxy,
                         const double* xyeig, const double* gx, const double* ga, const double* lmom, double* s,
                         double* z, int32_t* sig_idx, double* sig_coef, int32_t* nsig, double* fvec, uint8_t* flags,
                         void* stream);
/* mc_neighbour_topm (SPEC neighbourlist.maybe_update): for each of nrows rows
 * (rows[k], nullable = 0..nrows-1) of D [*, ldd] (fp32/fp64), the indices of the M
 * smallest distances, ties by lower index, ascending, into idx [nrows, M].
 * M > L -> MC_ERR_CONFIG. */
int mc_neighbour_topm(const void* D, int dtype, int32_t nrows, int32_t L, int64_t ldd, const int32_t* rows, int32_t M,
                      int32_t* idx, void* stream);
int mc_pathcv_grad(int32_t T, int32_t t0, int32_t n, int32_t npad, int32_t cap, const double* fplanes, const double* lplanes,
                   const double* w, const double* w_align, const int32_t* sig_idx, const double* sig_coef,
                   const int32_t* nsig, const double* fvec, const uint8_t* refresh, const int32_t* ridx,
                   const double* xyeig, void* ds, void* dz, int32_t out_f32, const float* fraw, const double* fcen,
                   const float* lraw, const double* lcen, const int32_t* perm, void* stream);

/* ---- fp32-coordinate path (configs 2-4): tensor-core estimate + exact refinement ----
 * mc_center_split (K1s, geometry.py:67-76 + operand prep): centre in fp64, optionally
 *   fold w into the operand (weighted), split into TF32 hi/lo planes [3, count, kpad]
 *   (kpad % 16 == 0); G, centroid, wbar, mom as mc_center.
 * mc_msd_tf32 (K2+K3, _kearsley_matrix + eigvals[0] of geometry.py:180-249): all-pairs
 *   3x3 covariance on tcgen05 (3xTF32, TMEM accumulators, TMA pipeline) with the
 *   fp64 Newton lambda_max in the epilogue -> MSD estimate D [T, ldd] fp32.  grid 0 = #SMs.
 * mc_candidates: per frame D_min and the landmark window {lam (D - D_min) <= thr_t},
 *   thr_t = thr + fcoef * fnorm[t] (fnorm nullable: thr_t = thr) -- the per-frame
 *   estimate-error allowance of the one-term screen.  dref [T] (nullable): landmark-
 *   sharded evaluation -- D_min = min(row minimum, dref[t]) with dref the minimum over
 *   every shard's estimate; a shard holding no window landmark returns cnt = 0.
 * mc_sort_by_key: counting sort of frames by window start (workspace bins [nbins]).
 * mc_refine: exact fp64 covariance + fit of the in-window pairs (or, with lo = cnt =
 *   NULL, of all pairs: the dense exact MSD matrix into Dd).  lwbar [L, 3] (nullable)
 *   = sum_j w_j (a_lj - c_l) (mc_center_split's wbar of the landmarks): frames then
 *   enter the fp64 contraction uncentred, S = S_half - c_x lwbar^T.  fmap [T] (nullable):
 *   frame t's row in `frames` (the per-frame scalars stay indexed by t).  wuni > 0 (all
 *   displacement weights equal to wuni) with fwbar [T, 3] (frames' wbar) and lwbar: both
 *   operands enter raw, S = wuni S_raw - fwbar c_l^T - c_x lwbar^T - n wuni c_x c_l^T. */
int mc_center_split(const void* coords, int dtype, int64_t count, int32_t n, int32_t kpad, const double* w_align,
                    const double* w_disp, int32_t weighted, float* hi, float* lo, double* centroid, double* gnorm,
                    double* wbar, double* mom, uint8_t* flags, void* stream);
int mc_msd_tf32(const float* fhi, const float* flo, const float* lhi, const float* llo, const double* gx,
                const double* ga, int32_t T, int32_t L, int32_t kpad, float* D, int64_t ldd, int32_t grid,
                void* stream);
/* Gradient pass of the fp32 path blocked over groups of 8 frames in candidate-sort
 * order (perm): each landmark coordinate feeds 8 frames; exact-refresh rows only.
 * out_map [T] (nullable): frame t's row in fraw and in ds/dz (the other per-frame
 * inputs stay indexed by t) -- the pruned screen's sorted order back to the caller's. */
int mc_pathcv_grad_block(int32_t T, int32_t n, int32_t cap, const float* fraw, const double* fcen, const float* lraw,
                         const double* lcen, const double* w, const double* w_align, const int32_t* sig_idx,
                         const double* sig_coef, const int32_t* nsig, const double* fvec, const int32_t* perm,
                         const int32_t* out_map, void* ds, void* dz, int32_t out_f32, void* stream);
/* Landmark operand of the int8 tensor-core gradient (replaces the per-step landmark
 * reads of _kearsley_matrix's contraction, geometry.py:180-196, by exact int8 digits):
 * the centred landmark coordinates ac = lraw - lcen (fp64) split into 4 signed int8
 * digits with a power-of-two scale 2^eB[k] per atom over every (landmark, axis):
 *   ac[l,k,g] ~= 2^(eB[k] - 31) sum_q D_q[k][3l+g] 2^(24 - 8q)   (|error| <= 2^(eB-32)),
 * stored per 32-byte k-step with the 4 digits interleaved: D_q[k][kk] =
 * dig[k][kk / 32][q][kk % 32], dig int8 [npad, kpad / 32, 4, 32] (npad % 128 == 0,
 * kpad % 32 == 0, kpad >= 3L), eB int32 [npad].
 * Once per landmark set. */
int mc_ldig_prep(const float* lraw, const double* lcen, int32_t L, int32_t n, int32_t npad, int32_t kpad,
                 int32_t* eB, int8_t* dig, void* stream);
/* mc_pathcv_grad_block on the 5th-gen tensor cores (tcgen05.mma.kind::i8, int32 TMEM
 * accumulators): the coefficient side is split per frame group into 4 int8 digits per
 * row in shared memory, 10 digit products (levels p + q <= 3) are accumulated exactly,
 * and the epilogue recombines them in fp64 (relative error ~2^-31 of the contraction's
 * magnitude, SPEC.md:228-236 gradient tolerance 1e-5).  ncv = 2: ds (out0), dz (out1)
 * -- the SPEC property_map gradients; groups of 8 frames whose significant union is
 * wider than 117 landmarks (or n % 4 != 0) go to the DMMA kernel in the same call.
 * ncv = 1: the metadynamics bias force F = -(dV/ds ds + dV/dz dz) (SPEC bias_and_force,
 * Eq. 1) written to out0 [T, n, 3] from dV [T, 2] (groups of 16 frames); groups wider
 * than 123 landmarks are NOT written and set *wide_flag = 1 (the caller then takes the
 * two-output path).  Other arguments as mc_pathcv_grad_block. */
int mc_pathcv_grad_i8(int32_t T, int32_t n, int32_t cap, const float* fraw, const double* fcen, const float* lraw,
                      const double* lcen, const double* w, const double* w_align, const int8_t* dig,
                      const int32_t* eB, int32_t npad, int32_t kpad, const int32_t* sig_idx, const double* sig_coef,
                      const int32_t* nsig, const double* fvec, const double* dV, const int32_t* perm,
                      const int32_t* out_map, void* out0, void* out1, int32_t out_f32, int32_t ncv,
                      int32_t* wide_flag, void* workspace, int64_t ws_bytes, void* stream);
/* Row digits for the int8 exact refits (the operands of _kearsley_matrix's covariance,
 * geometry.py:180-196, as exact int8 slices): structure k of B is raw row fmap[perm[k]]
 * (nullable maps), centred with centroid[perm[k]] and optionally weighted by w; its
 * three axis rows 3k + b over the atoms get a power-of-two scale 2^e[3k + b] and 4
 * signed int8 digits, stored per 32-atom k-step interleaved: dig [3B, kpad/32, 4, 32]
 * (kpad % 32 == 0, kpad >= n).  Landmarks: weighted, once per set; frames: per call,
 * in the refit's window-sorted order.  ein [*, 3] (nullable, unweighted rows only): the
 * exponents of structure perm[k] precomputed by mc_center_split16_uniform (one pass).
 * planes = 1: the digit-plane layout dig [kpad/32][4][3B][32] (plane (k-step, digit) holds
 * every row's 32 bytes) -- the FRAME operand of mc_refine_i8, whose B tile is one 3-D TMA
 * box of 4 planes x 64 rows so one MMA covers several digit products; landmarks (A) keep
 * planes = 0. */
int mc_row_digits(const float* raw, const double* centroid, const double* w, const int32_t* perm,
                  const int32_t* fmap, int32_t B, int32_t n, int32_t kpad, int8_t* dig, int32_t* e,
                  const int32_t* ein, int32_t planes, void* stream);
/* mc_refine on the int8 tensor cores (tcgen05.mma.kind::i8, 10 digit products, int32
 * TMEM accumulation, S exact to ~2^-31 of its scale): same outputs as mc_refine from the
 * row digits of the landmarks (ldig, eL: mc_row_digits weighted, planes = 0) and of the
 * frames (planes = 1) in
 * perm order (fdig, eF); gx / ga = the structures' weighted G norms; n < 32768. */
int mc_refine_i8(const int8_t* ldig, const int32_t* eL, const int8_t* fdig, const int32_t* eF, int32_t T, int32_t L,
                 int32_t n, int32_t kpad, const int32_t* perm, const int32_t* lo, const int32_t* cnt, const double* gx,
                 const double* ga, int32_t cap, double* Dex, double* Rex, float* Dd, int64_t ldd, uint8_t* flags,
                 void* stream);
/* Wide frame groups of mc_pathcv_grad_i8 (significant union wider than 117 landmarks, e.g.
 * the close-structure replay of config 3 with ~430 significant landmarks per frame):
 * mc_grad_i8_wide_plan writes per frame group (8 frames for ncv = 2, 16 for ncv = 1, in
 * perm order) the bytes of its A-digit image if it is wide, else 0 (bytes [groups]);
 * the caller lists the wide groups (wide_ids [nwide]), places their images (wide_off
 * [nwide] byte offsets into wimg, 16-byte aligned; sum of bytes) and calls
 * mc_pathcv_grad_i8 with a non-NULL wide_flag (the narrow groups; wide ones are left
 * out) and mc_pathcv_grad_i8_wide (the listed groups: the A digits streamed with the B
 * boxes instead of resident; hws = mc_grad_i8_wide_header_size bytes).  Same outputs
 * and exactness as mc_pathcv_grad_i8. */
int mc_grad_i8_wide_plan(int32_t T, int32_t cap, int32_t ncv, const int32_t* sig_idx, const int32_t* nsig,
                         const int32_t* perm, int64_t* bytes, void* stream);
int64_t mc_grad_i8_wide_header_size(int32_t nwide, int32_t ncv);
int mc_pathcv_grad_i8_wide(int32_t T, int32_t n, int32_t cap, const float* fraw, const double* fcen, const double* w,
                           const double* w_align, const int8_t* dig, const int32_t* eB, int32_t npad, int32_t kpad,
                           const int32_t* sig_idx, const double* sig_coef, const int32_t* nsig, const double* fvec,
                           const double* dV, const int32_t* perm, const int32_t* out_map, void* out0, void* out1,
                           int32_t out_f32, int32_t ncv, const int32_t* wide_ids, int32_t nwide,
                           const int64_t* wide_off, void* hws, int64_t hws_bytes, void* wimg, void* stream);
/* mc_refine_i8 for the pruned close-structure replay (PathCV.close_replay, fp32 frames;
 * replaces the dense covariances of _kearsley_matrix, geometry.py:180-196, for the Eq. 5
 * rows of SPEC.md:124-132): the exact covariances S of every window pair to Sex
 * [T, cap, 9] and, on the rows with fitmask[t] != 0 (the refresh rows, Alg. 2 step 5),
 * the fits (Dex [T, cap], Rex [T, cap, 9]); windows lo / cnt are required. */
int mc_refine_i8_close(const int8_t* ldig, const int32_t* eL, const int8_t* fdig, const int32_t* eF, int32_t T,
                       int32_t L, int32_t n, int32_t kpad, const int32_t* perm, const int32_t* lo, const int32_t* cnt,
                       const double* gx, const double* ga, int32_t cap, const uint8_t* fitmask, double* Sex,
                       double* Dex, double* Rex, uint8_t* flags, void* stream);
/* Bytes of caller workspace mc_pathcv_grad_i8 needs for T frames (per frame group: a
 * header and the A-digit image, <= 73 KB); -1 on bad arguments. */
int64_t mc_grad_i8_workspace_size(int32_t T, int32_t ncv);
/* mc_msd_tf32 on CTA pairs (tcgen05.mma.cta_group::2, M = 256 frames per pair):
 * same inputs/outputs; each SM stages half of the landmark operand. */
int mc_msd_tf32_2sm(const float* fhi, const float* flo, const float* lhi, const float* llo, const double* gx,
                    const double* ga, int32_t T, int32_t L, int32_t kpad, float* D, int64_t ldd, int32_t grid,
                    void* stream);
/* Same contraction with an FP16 operand format (kind::f16 tcgen05.mma, K = 16):
 * mc_center_split16 scales each structure by a power of two 2^e (max |value| < 2^14)
 *   and writes IEEE halves: terms = 3 -> hi + lo (22 significant bits, like the TF32
 *   pair) interleaved, hl [3, count, 2 kpad] (kpad % 32 == 0), per 32-atom block
 *   [hi x32 | lo x32] = one 128 B line; terms = 1 -> hi only, hl [3, count, kpad]
 *   (kpad % 64 == 0).  scale_inv[count] = 2^-e; opnorm[count] (nullable) = the fp64
 *   2-norm of the (weighted, centred) operand and rnorm[count] (nullable, terms = 1)
 *   the 2-norm of its half-precision rounding residual, for the one-term error bound.
 * mc_msd_f16 / mc_msd_f16_2sm: as mc_msd_tf32 / _2sm on hl operands, S rescaled by
 *   fscale[t] * lscale[l] (exact) before the epilogue.  terms = 3: hi*hi + hi*lo +
 *   lo*hi (split precision); terms = 1: hi*hi, a screening estimate with
 *   |D_est - D| <= 4 ||dS||_F, ||dS||_F <= rn_t op_l + op_t rn_l + rn_t rn_l
 *   + n 2^-27 (op_t + rn_t)(op_l + rn_l) (op = opnorm, rn = rnorm; rn <= 2^-11 op)
 *   (+ fp32 epilogue slack);
 *   _2sm supports terms = 3 only. */
int mc_center_split16(const void* coords, int dtype, int64_t count, int32_t n, int32_t kpad, const double* w_align,
                      const double* w_disp, int32_t weighted, int32_t terms, void* hl, double* scale_inv,
                      double* opnorm, double* rnorm, double* centroid, double* gnorm, double* wbar, double* mom,
                      uint8_t* flags, void* stream);
/* mc_center_split16 for the one-term frame operand with uniform weights (w = w' = wuni on
 * the n atoms, fp32 AoS input, n % 4 == 0, 16-byte aligned): the same outputs (halves,
 * scale, opnorm, rigorous rnorm bound, centroid, G = wuni sum |x - c|^2, wbar = 0,
 * flags) from one fp64 moment pass (shifted by the first atom) and one fp32 split pass
 * (geometry.py:67-76 centring).  mom is not produced.  dexp [count, 3] (nullable): the
 * per-axis int8 row-digit exponents of the unweighted centred rows, from the per-axis
 * coordinate extrema of the first pass (mc_row_digits' ein: one pass instead of two). */
int mc_center_split16_uniform(const float* coords, int64_t count, int32_t n, int32_t kpad, double wuni, void* hl,
                              double* scale_inv, double* opnorm, double* rnorm, double* centroid, double* gnorm,
                              double* wbar, uint8_t* flags, int32_t* dexp, void* stream);
int mc_msd_f16(const void* fhl, const void* lhl, const double* fscale, const double* lscale, const double* gx,
               const double* ga, int32_t T, int32_t L, int32_t kpad, int32_t terms, const int32_t* tlist,
               const int32_t* nlist, float* D, int64_t ldd, int32_t grid, void* stream);
int mc_msd_f16_2sm(const void* fhl, const void* lhl, const double* fscale, const double* lscale, const double* gx,
                   const double* ga, int32_t T, int32_t L, int32_t kpad, float* D, int64_t ldd, int32_t grid,
                   void* stream);
int mc_candidates(const float* D, int32_t T, int32_t L, int64_t ldd, double lam, double thr, const double* fnorm,
                  double fcoef, const int32_t* rlo, const int32_t* rhi, const float* dref, int32_t cap, int32_t* lo,
                  int32_t* cnt, float* dmin, uint8_t* flags, void* stream);
/* mc_candidates with the close-structure lifetime window (DESIGN.md
 * section 5): row t is a refresh frame y and dlife[t] >= 0 the largest D(x, y) of the
 * frames x that keep y as their close structure; the window holds every landmark any of
 * them can need, thr_t = thr + fcoef fnorm[t] + lam (2 d + 2 sqrt(d) (X + dmu)),
 * dmu = sqrt(D_min + fnorm[t]), X^2 = (sqrt(d) + dmu)^2 + thr / lam. */
int mc_candidates_life(const float* D, int32_t T, int32_t L, int64_t ldd, double lam, double thr,
                       const double* fnorm, double fcoef, const double* dlife, int32_t cap, int32_t* lo, int32_t* cnt,
                       float* dmin, uint8_t* flags, void* stream);
/* Metric pruning of the screen (csrc/prune.cu):
 * mc_prune_plan: from the one-term estimate Dc [T, C] against a coarse landmark subset
 *   (coarse landmark c = landmark c * cstride), its error bound c_unit * fnorm[t] * cnorm[c]
 *   (or, with the rounding-residual norms frnorm / crnorm of mc_center_split16, the
 *   per-pair bound 5 (r_t o_c + o_t r_c + r_t r_c) + c_unit (o_t + r_t)(o_c + r_c)
 *   + 1e-6 o_t o_c, c_unit = 5 n 2^-27),
 *   and mind / maxd [C, ntl] = min / max over each 48-landmark tile of the exact RMSD
 *   coarse->landmark, the hull [hull_lo, hull_hi) of landmark tiles that can hold a
 *   landmark within cutoff of D_min (thr = cutoff / lam, D units; knear <= 8 nearest
 *   coarse landmarks; C <= 1024) and a sort key (0: hull >= `wide` tiles, else
 *   1 + hull_lo).  Both triangle bounds d(t,l) >= d(c,l) - d(t,c) (knear nearest c) and
 *   d(t,l) >= d(t,c) - d(c,l) (c within one tile of the landmark tile; maxd nullable =
 *   first bound only) are applied; requires equal alignment / displacement weights.
 *   Landmark-sharded evaluation: a first call with dub_out [T] and NULL hull outputs
 *   writes this shard's D_min upper bound; the caller all-reduces the minimum over the
 *   shards and passes it as dub_in [T] to the second call, where a frame with no
 *   admissible tile in this shard gets the empty hull [ntl, 0) (key ntl).
 * mc_band_tiles: for the key-sorted order perm, the union hull of each 128-frame band,
 *   the (band, landmark tile) list tlist [*, 2] with its length *nlist (device), and each
 *   sorted row's landmark range [row_lo, row_hi) for mc_candidates(rlo, rhi).
 * mc_gather_rows: dst[r] = src[idx[r]] for rows of rowlen elements of esz bytes. */
int mc_prune_plan(const float* Dc, int32_t T, int32_t C, int64_t lddc, const double* fnorm, const double* cnorm,
                  const double* frnorm, const double* crnorm, double c_unit, const float* mind, const float* maxd, int32_t cstride, int32_t ntl, double thr,
                  int32_t knear, int32_t wide, const double* dub_in, double* dub_out, int32_t* hull_lo,
                  int32_t* hull_hi, int32_t* key, void* stream);
int mc_band_tiles(const int32_t* perm, int32_t T, const int32_t* hull_lo, const int32_t* hull_hi, int32_t BM,
                  int32_t BL, int32_t L, int32_t* tlist, int32_t* nlist, int32_t* row_lo, int32_t* row_hi,
                  void* stream);
int mc_gather_rows(const void* src, int32_t esz, int64_t rowlen, const int32_t* idx, int32_t rows, void* dst,
                   void* stream);
int mc_sort_by_key(const int32_t* key, int32_t T, int32_t nbins, int32_t* bins, int32_t* perm, void* stream);
int mc_refine(const float* frames, const double* fcentroid, const float* landmarks, const double* lcentroid,
              const double* lwbar, const double* w, const double* gx, const double* ga, int32_t T, int32_t L, int32_t n,
              const int32_t* perm, const int32_t* lo, const int32_t* cnt, int32_t cap, double* Dex, double* Rex,
              float* Dd, int64_t ldd, const int32_t* fmap, const double* fwbar, double wuni,
              uint8_t* flags, void* stream);
/* Close-structure path on the fp64 tensor cores (fp32 coordinates, uniform weights):
 * mc_cov_dmma: dense S [T, L, 9] = sum_j w (x_tj - c_t)(a_lj - c_l)^T (the mc_cov_f64
 *   contract on raw fp32 frames / landmarks with their fp64 centroids and w-sums
 *   wbar = sum_j w (x_j - c); wuni = the common weight), exact fp64 products and sums.
 * mc_close_grad_fix: adds the Eq. 6 dR_xy term (the dk_contract closed form used by
 *   mc_pathcv_grad) to ds / dz rows t0 .. t0+T-1 of the non-refresh frames, after the
 *   contraction part came from mc_pathcv_grad_block; fvec = the chunk's K4 per-frame
 *   vectors, ridx / refresh / xyeig global by frame, frames raw fp32 [*, n, 3]. */
int mc_cov_dmma(const float* frames, const double* fcentroid, const double* fwbar, const float* landmarks,
                const double* lcentroid, const double* lwbar, const double* w, double wuni, int32_t T, int32_t L,
                int32_t n, double* S, void* stream);
int mc_close_grad_fix(int32_t T, int32_t t0, int32_t n, const uint8_t* refresh, const int32_t* ridx,
                      const double* xyeig, const double* fvec, const double* w, const float* frames,
                      const double* fcentroid, void* ds, void* dz, int32_t out_f32, void* stream);

/* Per-pair DistanceResult gradients of the reference-facing API:
 * exact_distance (Eq. 3/4) and approx_distance (Eq. 5/6,
 * SPEC.md:124-132).  Pair p = (frame xi[p], reference ai[p]) with rotation rot[p]
 * (exact: R_{a x}; approximate: the saved R_{a y}).  approx[p] != 0 selects Eq. 5/6
 * with close structure yi[p] (a frame index), S[p] = cov(x, a), amom = reference
 * second moments, xyeig/rxy = x<->y fit; value[p] receives Eq. 5 on those pairs.
 * grad [P, n, 3] w.r.t. the raw (uncentred) frame coordinates. */
int mc_pair_grad(int64_t P, int32_t n, int32_t npad, const double* xplanes, const double* aplanes, const int32_t* xi,
                 const int32_t* ai, const double* rot, const double* w, const double* w_align, const double* xwbar,
                 const double* awbar, const int32_t* approx, const int32_t* yi, const double* S, const double* amom,
                 const double* xyeig, const double* rxy, const double* gx, const double* ga, double* value,
                 double* grad, void* stream);

/* property_map over supplied distances D [L] (+ grads [L,n,3]):
 * out[0] = s, out[1] = z; ds, dz [n,3] when grads != NULL. */
int mc_property_map(int32_t L, int32_t n, const double* D, const double* grads, const double* q, double lam,
                    double* out, double* ds, double* dz, void* stream);

/* ---- metadynamics bias and force (SPEC [MODULE] metadynamics, PAPER Eq. 1) ----
 * mc_mtd_bias_direct: V[t] = sum_h heights[h] prod_i exp(-(cv[t,i] - centers[h,i])^2 / (2 sigmas[h,i]^2))
 *   and dV[t, i] = dV/dS_i (analytic); d <= 3 CVs, device arrays.
 * mc_mtd_grid_deposit / mc_mtd_grid_eval: uniform grid per CV (d = 1 or 2; lo, hi, bins are HOST
 *   arrays of d values; nodes lo + k h, k = 0..bins, row-major [bins0+1][bins1+1]); val, dgrid
 *   [d][nodes] and (d = 2) the cross derivative dxy store the cubic Hermite data.  deposit adds
 *   one hill (device center/sigma [d]) to every node within `cutoff` sigmas (SPEC: 6);
 *   *flag = MC_FLAG_OUT_OF_GRID for a centre off the grid (the grid is then left unchanged).
 *   eval interpolates V, dV per frame;
 *   flags[t] = MC_FLAG_OUT_OF_GRID (V = dV = 0) for a CV off the grid.
 * mc_mtd_force: F[t,k,c] = -sum_i dV[t,i] G_i[t,k,c] (physical sign, SPEC design decision),
 *   G_i = g0, g1, g2 the CV gradients [T, n, 3] (dtype f32/f64, F likewise). */
int mc_mtd_bias_direct(const double* cv, int32_t T, int32_t d, const double* centers, const double* sigmas,
                       const double* heights, int32_t H, double* V, double* dV, void* stream);
int mc_mtd_grid_deposit(double* val, double* dgrid, double* dxy, int32_t d, const double* lo, const double* hi,
                        const int32_t* bins, const double* center, const double* sigma, double height, double cutoff,
                        uint8_t* flag, void* stream);
int mc_mtd_grid_eval(const double* val, const double* dgrid, const double* dxy, int32_t d, const double* lo,
                     const double* hi, const int32_t* bins, const double* cv, int32_t T, double* V, double* dV,
                     uint8_t* flags, void* stream);
int mc_mtd_force(const double* dV, int32_t T, int32_t d, const void* g0, const void* g1, const void* g2, int dtype,
                 int32_t n, void* F, void* stream);

/* ---- toy MD driver (SPEC [MODULE] toysim run) ----
 * mc_toysim_run: W independent walkers (one CTA each) advance `steps` overdamped Langevin
 *   steps (Euler-Maruyama, x += mob F + noise xi, xi ~ N(0,1) from Philox4x32-10 keyed by
 *   `seed`, counter (bead, step, walker)) of an n-bead chain (harmonic bonds bond_k, bond_r0;
 *   harmonic angles angle_k, theta0; n <= 64) in ONE launch.  mode 0: free dynamics (the
 *   reference-set pre-run); 1: original method (Alg. 1, exact fits to all L <= 128
 *   references every step); 2: close structure (Alg. 2, threshold eps, strict '>').
 *   Per step: path CV s, z (lambda = lam) of the centred frame, metadynamics hills on s
 *   (height hill_h, width hill_sigma, deposited at the step's s when step % tau_g == 0,
 *   after the step's force; capacity max_hills), bias force -dV/ds ds/dx.
 *   refs [L, n, 3] centred, refg [L] = sum w |a|^2, refmom [L, 6] = sum w a a^T (xx, xy,
 *   xz, yy, yz, zz), q [L], w / wa [n] displacement / alignment weights.  State in/out:
 *   x, y [W, n, 3], rays [W, L, 9] (saved R_{a_i y}), hasy [W], hills [W, max_hills],
 *   nhills [W], counters [W, 3] (+= expensive, cheap, reassign; SPEC msd-engine rules).
 *   Out: cv [W, steps, 4] = (s, z, V_bias, D(x, y)), rlog [W, steps] (1 = reassigned),
 *   traj [W, ceil(steps / traj_stride), n, 3] positions at the start of steps
 *   step0 + k traj_stride (traj_stride 0: none; step0 % traj_stride == 0), flags [W]
 *   (|= NoConverge / NonFinite / SigOverflow = hill capacity exceeded).  Continuing a run:
 *   call again with step0 += steps and the same state arrays.  Neighbour list (SPEC
 *   neighbourlist; nl_m = M > 0, modes 1 and 2): state act [W, L] (uint8
 *   members) and nl_last [W] (last update step, -1 = none); updated on the first step and
 *   whenever step - nl_last >= nl_stride from that step's distances to all N (exact, or the
 *   Eq. 5 approximations in close mode) as the M smallest (ties by lower index); between
 *   updates only the members are evaluated (M expensive / cheap) and s, z and the bias
 *   force sum over them. */
int mc_toysim_run(int32_t W, int32_t n, int32_t L, int32_t steps, int64_t step0, int32_t mode, int32_t tau_g,
                  int32_t max_hills, int32_t traj_stride, double bond_k, double bond_r0, double angle_k,
                  double theta0, double mob, double noise, double lam, double eps, double hill_h, double hill_sigma,
                  uint64_t seed, const double* refs, const double* refg, const double* refmom, const double* q,
                  const double* w, const double* wa, double* x, double* y, double* rays, int32_t* hasy,
                  double* hills, int32_t* nhills, int64_t* counters, double* cv, uint8_t* rlog, double* traj,
                  uint8_t* flags, int32_t nl_m, int32_t nl_stride, uint8_t* act,
                  int64_t* nl_last, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MCB200_H */
