/*
 * C restatement of the reference CPU path — TEST INFRASTRUCTURE / CPU BASELINE
 * ONLY (never linked into the product library).
 *
 * Follows /root/reference/pkg/src/metadyn_close/geometry.py function by
 * function and restates the SPEC-only layers (SPEC.md msd-engine + colvar):
 *   oc_center            geometry.py:67-76
 *   kearsley_matrix      geometry.py:180-196   (m = x - a, p = x + a form)
 *   jacobi_eigh4         geometry.py:106-153   (cyclic Jacobi, same tolerance,
 *                                               stable ascending sort, sign rule)
 *   quat_to_rot          geometry.py:156-164
 *   oc_fit               geometry.py:227-249   (no derivatives)
 *   oc_msd_matrix        all-pairs eigvals[0]
 *   oc_path_cv_exact     Alg. 1 + Eq. 2/4, gradient
 *                        2 w d - w' sum 2 w d (Eq. 4's dR term is zero at the
 *                        optimum)
 * Parallelism: OpenMP over frames (pairs are independent).
 * Pinned against the numpy oracle (itself pinned to the reference's golden
 * vectors) in tests/test_oracle_c.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void center(const double* x, int n, const double* wa, double* xc) {
  double c[3] = {0, 0, 0};
  for (int j = 0; j < n; ++j)
    for (int a = 0; a < 3; ++a) c[a] += wa[j] * x[3 * j + a];
  for (int j = 0; j < n; ++j)
    for (int a = 0; a < 3; ++a) xc[3 * j + a] = x[3 * j + a] - c[a];
}

static void kearsley_matrix(const double* x, const double* a, const double* w, int n, double k[4][4]) {
  double k00 = 0, o0 = 0, o1 = 0, o2 = 0, mm[3][3] = {{0}}, pp[3][3] = {{0}}, gp = 0;
  for (int j = 0; j < n; ++j) {
    const double m0 = x[3 * j] - a[3 * j], m1 = x[3 * j + 1] - a[3 * j + 1], m2 = x[3 * j + 2] - a[3 * j + 2];
    const double p0 = x[3 * j] + a[3 * j], p1 = x[3 * j + 1] + a[3 * j + 1], p2 = x[3 * j + 2] + a[3 * j + 2];
    const double wj = w[j];
    k00 += wj * (m0 * m0 + m1 * m1 + m2 * m2);
    /* cross(p, m) */
    o0 += wj * (p1 * m2 - p2 * m1);
    o1 += wj * (p2 * m0 - p0 * m2);
    o2 += wj * (p0 * m1 - p1 * m0);
    const double m[3] = {m0, m1, m2}, p[3] = {p0, p1, p2};
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) {
        mm[r][c] += wj * m[r] * m[c];
        pp[r][c] += wj * p[r] * p[c];
      }
    gp += wj * (p0 * p0 + p1 * p1 + p2 * p2);
  }
  k[0][0] = k00;
  k[0][1] = k[1][0] = -o0;
  k[0][2] = k[2][0] = -o1;
  k[0][3] = k[3][0] = -o2;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) k[1 + r][1 + c] = mm[r][c] + (r == c ? gp : 0.0) - pp[r][c];
}

static int jacobi_eigh4(double a[4][4], double w[4], double V[4][4]) {
  double v[4][4] = {{1, 0, 0, 0}, {0, 1, 0, 0}, {0, 0, 1, 0}, {0, 0, 0, 1}};
  double fro = 0;
  for (int i = 0; i < 4; ++i)
    for (int j = 0; j < 4; ++j) fro += a[i][j] * a[i][j];
  double tol = 4e-16 * sqrt(fro);
  if (tol < 1e-14) tol = 1e-14;
  int ok = 0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0;
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j)
        if (i != j) off += a[i][j] * a[i][j];
    if (sqrt(off) < tol) { ok = 1; break; }
    for (int p = 0; p < 3; ++p)
      for (int q = p + 1; q < 4; ++q) {
        const double apq = a[p][q];
        if (apq == 0.0) continue;
        const double theta = (a[q][q] - a[p][p]) / (2.0 * apq);
        const double t = copysign(1.0, theta) / (fabs(theta) + hypot(theta, 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int r = 0; r < 4; ++r) {
          const double ap = a[r][p], aq = a[r][q];
          a[r][p] = c * ap - s * aq;
          a[r][q] = s * ap + c * aq;
        }
        for (int r = 0; r < 4; ++r) {
          const double ap = a[p][r], aq = a[q][r];
          a[p][r] = c * ap - s * aq;
          a[q][r] = s * ap + c * aq;
        }
        a[p][q] = a[q][p] = 0.0;
        for (int r = 0; r < 4; ++r) {
          const double vp = v[r][p], vq = v[r][q];
          v[r][p] = c * vp - s * vq;
          v[r][q] = s * vp + c * vq;
        }
      }
  }
  int order[4] = {0, 1, 2, 3};
  for (int i = 1; i < 4; ++i) { /* stable insertion sort */
    int k = order[i], j = i - 1;
    while (j >= 0 && a[order[j]][order[j]] > a[k][k]) { order[j + 1] = order[j]; --j; }
    order[j + 1] = k;
  }
  for (int o = 0; o < 4; ++o) {
    const int i = order[o];
    w[o] = a[i][i];
    int im = 0;
    double best = fabs(v[0][i]);
    for (int r = 1; r < 4; ++r)
      if (fabs(v[r][i]) > best) { best = fabs(v[r][i]); im = r; }
    const double sg = v[im][i] < 0.0 ? -1.0 : 1.0;
    for (int r = 0; r < 4; ++r) V[r][o] = sg * v[r][i];
  }
  return ok;
}

static void quat_to_rot(const double* q, double* r) {
  const double q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
  r[0] = q0 * q0 + q1 * q1 - q2 * q2 - q3 * q3; r[1] = 2 * (q1 * q2 - q0 * q3); r[2] = 2 * (q1 * q3 + q0 * q2);
  r[3] = 2 * (q1 * q2 + q0 * q3); r[4] = q0 * q0 - q1 * q1 + q2 * q2 - q3 * q3; r[5] = 2 * (q2 * q3 - q0 * q1);
  r[6] = 2 * (q1 * q3 - q0 * q2); r[7] = 2 * (q2 * q3 + q0 * q1); r[8] = q0 * q0 - q1 * q1 - q2 * q2 + q3 * q3;
}

/* kearsley_fit (no derivatives): returns eigvals[0]; rot optional */
double oc_fit(const double* xc, const double* ac, const double* w, int n, double* rot, double* eigvals) {
  double k[4][4], V[4][4], ev[4];
  kearsley_matrix(xc, ac, w, n, k);
  jacobi_eigh4(k, ev, V);
  if (rot) {
    const double q[4] = {V[0][0], V[1][0], V[2][0], V[3][0]};
    quat_to_rot(q, rot);
  }
  if (eigvals) memcpy(eigvals, ev, sizeof(ev));
  return ev[0];
}

static int set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
  return omp_get_max_threads();
#else
  (void)nthreads;
  return 1;
#endif
}

int oc_max_threads(void) { return set_threads(0); }

/* all-pairs MSD: frames [T,n,3], landmarks [L,n,3] (raw, fp64) -> D [T,L].
 * Every structure is centred once, then the T x L fits run in parallel over PAIRS
 * (not frames), so a small frame sample still keeps every host thread busy. */
int oc_msd_matrix(const double* frames, const double* landmarks, int T, int L, int n, const double* w,
                  const double* wa, double* D, int nthreads) {
  const int used = set_threads(nthreads);
  double* lc = (double*)malloc(sizeof(double) * 3 * n * (size_t)L);
  double* fc = (double*)malloc(sizeof(double) * 3 * n * (size_t)T);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < L; ++i) center(landmarks + (size_t)i * 3 * n, n, wa, lc + (size_t)i * 3 * n);
#pragma omp parallel for schedule(static)
  for (int t = 0; t < T; ++t) center(frames + (size_t)t * 3 * n, n, wa, fc + (size_t)t * 3 * n);
#pragma omp parallel for schedule(dynamic, 16)
  for (long long e = 0; e < (long long)T * L; ++e) {
    const int t = (int)(e / L), i = (int)(e % L);
    D[e] = oc_fit(fc + (size_t)t * 3 * n, lc + (size_t)i * 3 * n, w, n, NULL, NULL);
  }
  free(fc);
  free(lc);
  return used;
}

/* geometry.py:167-177: J[c][b*3+g] */
static void rot_quat_jacobian(const double* q, double J[4][9]) {
  const double q0 = 2 * q[0], q1 = 2 * q[1], q2 = 2 * q[2], q3 = 2 * q[3];
  const double j[4][9] = {{q0, -q3, q2, q3, q0, -q1, -q2, q1, q0},
                          {q1, q2, q3, q2, -q1, -q0, q3, q0, -q1},
                          {-q2, q1, q0, q1, q2, q3, -q0, q3, -q2},
                          {-q3, -q0, q1, q0, -q3, q2, q1, q2, q3}};
  memcpy(J, j, sizeof(j));
}

/* v^T (dK/dx_k) q0 — _kearsley_matrix_grad (geometry.py:199-224) contracted */
static void dk_contract(const double* v, const double* q, double w, const double* x, const double* y, double* out) {
  const double v0 = v[0], q0 = q[0], u[3] = {q[1], q[2], q[3]}, t[3] = {v[1], v[2], v[3]};
  const double c[3] = {v0 * u[0] + q0 * t[0], v0 * u[1] + q0 * t[1], v0 * u[2] + q0 * t[2]};
  const double cx[3] = {c[1] * y[2] - c[2] * y[1], c[2] * y[0] - c[0] * y[2], c[0] * y[1] - c[1] * y[0]};
  const double yu = y[0] * u[0] + y[1] * u[1] + y[2] * u[2], yt = y[0] * t[0] + y[1] * t[1] + y[2] * t[2];
  const double tu = t[0] * u[0] + t[1] * u[1] + t[2] * u[2];
  for (int a = 0; a < 3; ++a)
    out[a] = 2 * w * (v0 * q0 * (x[a] - y[a]) - cx[a] - t[a] * yu - u[a] * yt + (x[a] + y[a]) * tu);
}

/* Alg. 2 replay: sequential over frames, OpenMP over
 * landmarks inside a frame.  Outputs s, z, ds, dz (nullable), refresh, dxy.
 * Approximate frames use Eq. 5/6; the dR_xy term is contracted once per CV
 * with M = sum_i c_i M_i (linearity), as a good CPU port would. */
int oc_close_replay(const double* frames, const double* landmarks, int T, int L, int n, double lam,
                    const double* q, const double* w, const double* wa, double eps, double* s, double* z,
                    double* ds, double* dz, uint8_t* refresh, double* dxy, int nthreads) {
  const int used = set_threads(nthreads);
  double* lc = (double*)malloc(sizeof(double) * 3 * n * (size_t)L);
  for (int i = 0; i < L; ++i) center(landmarks + (size_t)i * 3 * n, n, wa, lc + (size_t)i * 3 * n);
  double* xc = (double*)malloc(sizeof(double) * 3 * n);
  double* y = (double*)malloc(sizeof(double) * 3 * n);
  double* Rs = (double*)malloc(sizeof(double) * 9 * (size_t)L);   /* saved R_{a_i y} */
  double* Rh = (double*)malloc(sizeof(double) * 9 * (size_t)L);   /* Rhat_i this frame */
  double* D = (double*)malloc(sizeof(double) * L);
  double* gs = (double*)malloc(sizeof(double) * 3 * n);
  double* gz = (double*)malloc(sizeof(double) * 3 * n);
  double* U = (double*)malloc(sizeof(double) * 6 * n);
  int have_y = 0;
  for (int t = 0; t < T; ++t) {
    center(frames + (size_t)t * 3 * n, n, wa, xc);
    double ev[4], V[4][4], k[4][4], rxy[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
    int fresh = 1;
    double d_xy = 0.0;
    if (have_y) {
      kearsley_matrix(xc, y, w, n, k);
      jacobi_eigh4(k, ev, V);
      d_xy = ev[0];
      fresh = d_xy > eps;
      const double q0[4] = {V[0][0], V[1][0], V[2][0], V[3][0]};
      quat_to_rot(q0, rxy);
    }
    refresh[t] = (uint8_t)fresh;
    dxy[t] = d_xy;
    if (fresh) {
      memcpy(y, xc, sizeof(double) * 3 * n);
      have_y = 1;
#pragma omp parallel for schedule(dynamic, 4)
      for (int i = 0; i < L; ++i) {
        D[i] = oc_fit(xc, lc + (size_t)i * 3 * n, w, n, Rs + 9 * (size_t)i, NULL);
        memcpy(Rh + 9 * (size_t)i, Rs + 9 * (size_t)i, sizeof(double) * 9);
      }
    } else {
#pragma omp parallel for schedule(static)
      for (int i = 0; i < L; ++i) {
        const double* r = Rs + 9 * (size_t)i;
        double* h = Rh + 9 * (size_t)i;
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) h[3 * a + b] = rxy[3 * a] * r[b] + rxy[3 * a + 1] * r[3 + b] + rxy[3 * a + 2] * r[6 + b];
        const double* a = lc + (size_t)i * 3 * n;
        double acc = 0;
        for (int j = 0; j < n; ++j)
          for (int b = 0; b < 3; ++b) {
            const double d = xc[3 * j + b] - (h[3 * b] * a[3 * j] + h[3 * b + 1] * a[3 * j + 1] + h[3 * b + 2] * a[3 * j + 2]);
            acc += w[j] * d * d;
          }
        D[i] = acc;
      }
    }
    double dmin = INFINITY;
    for (int i = 0; i < L; ++i) if (D[i] < dmin) dmin = D[i];
    double zs = 0, qs = 0;
    for (int i = 0; i < L; ++i) { const double e = exp(-lam * (D[i] - dmin)); zs += e; qs += q[i] * e; }
    const double sv = qs / zs;
    s[t] = sv;
    z[t] = dmin - log(zs) / lam;
    if (!ds) continue;
    /* U_j = sum_i c_i Rhat_i a_ij for both CVs; Mtot (approx frames) */
    memset(U, 0, sizeof(double) * 6 * n);
    double sumc[2] = {0, 0}, M[2][9] = {{0}};
    for (int i = 0; i < L; ++i) {
      const double p = exp(-lam * (D[i] - dmin)) / zs;
      const double c[2] = {-lam * p * (q[i] - sv), p};
      if (p == 0.0) continue;
      sumc[0] += c[0]; sumc[1] += c[1];
      const double* a = lc + (size_t)i * 3 * n;
      const double* h = Rh + 9 * (size_t)i;
      const double* r = Rs + 9 * (size_t)i;
      for (int j = 0; j < n; ++j) {
        double ra[3], b[3], dd[3];
        for (int bb = 0; bb < 3; ++bb) ra[bb] = h[3 * bb] * a[3 * j] + h[3 * bb + 1] * a[3 * j + 1] + h[3 * bb + 2] * a[3 * j + 2];
        for (int cv = 0; cv < 2; ++cv)
          for (int bb = 0; bb < 3; ++bb) U[6 * j + 3 * cv + bb] += c[cv] * ra[bb];
        if (!fresh) { /* M_i = -2 sum_j w d~ b^T, b = R_s a */
          for (int bb = 0; bb < 3; ++bb) {
            b[bb] = r[3 * bb] * a[3 * j] + r[3 * bb + 1] * a[3 * j + 1] + r[3 * bb + 2] * a[3 * j + 2];
            dd[bb] = xc[3 * j + bb] - ra[bb];
          }
          for (int cv = 0; cv < 2; ++cv)
            for (int aa = 0; aa < 3; ++aa)
              for (int bb = 0; bb < 3; ++bb) M[cv][3 * aa + bb] += -2.0 * c[cv] * w[j] * dd[aa] * b[bb];
        }
      }
    }
    double vv[2][4] = {{0}}, q0[4] = {0};
    if (!fresh) {
      double J[4][9];
      for (int r = 0; r < 4; ++r) q0[r] = V[r][0];
      rot_quat_jacobian(q0, J);
      for (int cv = 0; cv < 2; ++cv) {
        double g[4];
        for (int cc = 0; cc < 4; ++cc) { g[cc] = 0; for (int e = 0; e < 9; ++e) g[cc] += M[cv][e] * J[cc][e]; }
        for (int m = 1; m < 4; ++m) {
          const double h = (V[0][m] * g[0] + V[1][m] * g[1] + V[2][m] * g[2] + V[3][m] * g[3]) / (ev[0] - ev[m]);
          for (int r = 0; r < 4; ++r) vv[cv][r] += h * V[r][m];
        }
      }
    }
    double sum[2][3] = {{0}};
    for (int j = 0; j < n; ++j)
      for (int cv = 0; cv < 2; ++cv) {
        double g[3];
        for (int bb = 0; bb < 3; ++bb) g[bb] = 2.0 * w[j] * (sumc[cv] * xc[3 * j + bb] - U[6 * j + 3 * cv + bb]);
        if (!fresh) {
          double d3[3];
          dk_contract(vv[cv], q0, w[j], xc + 3 * j, y + 3 * j, d3);
          for (int bb = 0; bb < 3; ++bb) g[bb] += d3[bb];
        }
        double* o = cv == 0 ? gs : gz;
        for (int bb = 0; bb < 3; ++bb) { o[3 * j + bb] = g[bb]; sum[cv][bb] += g[bb]; }
      }
    for (int j = 0; j < n; ++j)
      for (int bb = 0; bb < 3; ++bb) {
        ds[((size_t)t * n + j) * 3 + bb] = gs[3 * j + bb] - wa[j] * sum[0][bb];
        dz[((size_t)t * n + j) * 3 + bb] = gz[3 * j + bb] - wa[j] * sum[1][bb];
      }
  }
  free(lc); free(xc); free(y); free(Rs); free(Rh); free(D); free(gs); free(gz); free(U);
  return used;
}

/* Alg. 1 path-CV: s, z [T]; ds, dz [T,n,3] (nullable).
 * Three parallel phases so every host thread is busy even for a handful of frames:
 * (1) the T x L exact fits (geometry.py:227-249) in parallel over PAIRS, keeping D and R;
 * (2) per frame the shifted softmax s, z (PAPER Eq. 2); (3) the
 * gradients (Eq. 4 summed with the K4 coefficients) in parallel over (frame, atom block),
 * each landmark's translation term sum_j 2 w_j d_j = 2 (Sx - R Sa) from per-structure sums. */
int oc_path_cv_exact(const double* frames, const double* landmarks, int T, int L, int n, double lam, const double* q,
                     const double* w, const double* wa, double* s, double* z, double* ds, double* dz, int nthreads) {
  const int used = set_threads(nthreads);
  double* lc = (double*)malloc(sizeof(double) * 3 * n * (size_t)L);
  double* fc = (double*)malloc(sizeof(double) * 3 * n * (size_t)T);
  double* D = (double*)malloc(sizeof(double) * (size_t)T * L);
  double* R = (double*)malloc(sizeof(double) * 9 * (size_t)T * L);
  double* Sa = (double*)malloc(sizeof(double) * 3 * (size_t)L);
  double* Sx = (double*)malloc(sizeof(double) * 3 * (size_t)T);
#pragma omp parallel for schedule(static)
  for (int i = 0; i < L; ++i) {
    double* a = lc + (size_t)i * 3 * n;
    center(landmarks + (size_t)i * 3 * n, n, wa, a);
    double acc[3] = {0, 0, 0};
    for (int j = 0; j < n; ++j)
      for (int b = 0; b < 3; ++b) acc[b] += w[j] * a[3 * j + b];
    for (int b = 0; b < 3; ++b) Sa[3 * i + b] = acc[b];
  }
#pragma omp parallel for schedule(static)
  for (int t = 0; t < T; ++t) {
    double* x = fc + (size_t)t * 3 * n;
    center(frames + (size_t)t * 3 * n, n, wa, x);
    double acc[3] = {0, 0, 0};
    for (int j = 0; j < n; ++j)
      for (int b = 0; b < 3; ++b) acc[b] += w[j] * x[3 * j + b];
    for (int b = 0; b < 3; ++b) Sx[3 * t + b] = acc[b];
  }
  /* (1) fits */
#pragma omp parallel for schedule(dynamic, 16)
  for (long long e = 0; e < (long long)T * L; ++e) {
    const int t = (int)(e / L), i = (int)(e % L);
    D[e] = oc_fit(fc + (size_t)t * 3 * n, lc + (size_t)i * 3 * n, w, n, R + 9 * (size_t)e, NULL);
  }
  /* (2) softmax weights -> s, z; D is overwritten with the coefficient p_i */
  double* cs = (double*)malloc(sizeof(double) * (size_t)T * L);
#pragma omp parallel for schedule(static)
  for (int t = 0; t < T; ++t) {
    double* Dt = D + (size_t)t * L;
    double dmin = INFINITY;
    for (int i = 0; i < L; ++i)
      if (Dt[i] < dmin) dmin = Dt[i];
    double zs = 0, qs = 0;
    for (int i = 0; i < L; ++i) {
      const double e = exp(-lam * (Dt[i] - dmin));
      zs += e;
      qs += q[i] * e;
    }
    const double sv = qs / zs;
    s[t] = sv;
    z[t] = dmin - log(zs) / lam;
    for (int i = 0; i < L; ++i) {
      const double p = exp(-lam * (Dt[i] - dmin)) / zs;
      cs[(size_t)t * L + i] = -lam * p * (q[i] - sv);
      Dt[i] = p;
    }
  }
  /* (3) gradients over (frame, block of 64 atoms) */
  if (ds) {
    const int AB = 64, nb = (n + AB - 1) / AB;
#pragma omp parallel for schedule(dynamic, 1)
    for (long long e = 0; e < (long long)T * nb; ++e) {
      const int t = (int)(e / nb), j0 = (int)(e % nb) * AB, j1 = j0 + AB < n ? j0 + AB : n;
      const double* xc = fc + (size_t)t * 3 * n;
      double gs[3 * 64], gz[3 * 64];
      memset(gs, 0, sizeof(gs));
      memset(gz, 0, sizeof(gz));
      for (int i = 0; i < L; ++i) {
        const double c_s = cs[(size_t)t * L + i], c_z = D[(size_t)t * L + i];
        const double* a = lc + (size_t)i * 3 * n;
        const double* r = R + 9 * ((size_t)t * L + i);
        double sum[3];
        for (int b = 0; b < 3; ++b)
          sum[b] = 2.0 * (Sx[3 * t + b] - (r[3 * b] * Sa[3 * i] + r[3 * b + 1] * Sa[3 * i + 1] + r[3 * b + 2] * Sa[3 * i + 2]));
        for (int j = j0; j < j1; ++j)
          for (int b = 0; b < 3; ++b) {
            const double d = xc[3 * j + b] - (r[3 * b] * a[3 * j] + r[3 * b + 1] * a[3 * j + 1] + r[3 * b + 2] * a[3 * j + 2]);
            const double g = 2.0 * w[j] * d - wa[j] * sum[b];
            gs[3 * (j - j0) + b] += c_s * g;
            gz[3 * (j - j0) + b] += c_z * g;
          }
      }
      memcpy(ds + ((size_t)t * n + j0) * 3, gs, sizeof(double) * 3 * (j1 - j0));
      memcpy(dz + ((size_t)t * n + j0) * 3, gz, sizeof(double) * 3 * (j1 - j0));
    }
  }
  free(cs); free(Sx); free(Sa); free(R); free(D); free(fc); free(lc);
  return used;
}
