/*
 * TEST INFRASTRUCTURE ONLY -- C restatement of the reference's sLSLU loop,
 * used as the timed CPU baseline (bench.py cpu_baseline / --impl reference)
 * and as a fast CPU checker at sizes the numpy port cannot reach.
 * Never linked into, or called by, the product package.
 *
 * Restates (reference paths under pkg/src/hessketch/):
 *   co_tomo_*         problems.py:276-331  ray tracer / tomography_matrix
 *                     (detector count generalised, as oracle/tomo_oracle.py)
 *   co_csr_transpose  linops.py:139        M.T.tocsr() (rows sorted by source row)
 *   co_slslu_f32      solvers.py:410-539 + hessenberg.py:275-390 (sketched,
 *                     lam = 0) in float32 vector arithmetic ("oracle32"):
 *                     CSR row sums sequential without FMA (scipy csr_matvec),
 *                     in-order elimination u -= c*d_j (one pass per j, as numpy
 *                     does), argmax |u| with smallest-index ties, u / pivot,
 *                     sketch S2 u in float64, projected LS re-factored from
 *                     scratch every iteration (Householder QR, float64) and
 *                     x = L_k y recomputed every iteration.
 * Parallelism: OpenMP over rows / elements (the reference is single-threaded
 * in csr_matvec; this port uses every host core it is given).
 *
 * Build: oracle/build_coracle.py  (gcc -O3 -fopenmp -ffp-contract=off)
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

/* ------------------------------------------------------------------------ */
/* ray tracer (problems.py:276-308)                                          */

typedef struct {
  int grid;
  double ox, oy, dx, dy;
} ray_t;

static double cross_t(int k, double o, double d) { return ((double)k - o) / d; }

/* calls emit(pix, len, ctx) in traversal order with consecutive duplicate pixels merged;
   returns count. If out_col/out_val non-NULL, writes entries there (traversal order). */
static int64_t trace(const ray_t* r, int32_t* out_col, double* out_val) {
  const int grid = r->grid;
  double t0 = -INFINITY, t1 = INFINITY;
  const double o[2] = {r->ox, r->oy}, d[2] = {r->dx, r->dy};
  for (int ax = 0; ax < 2; ++ax) {
    if (fabs(d[ax]) < 1e-12) {
      if (o[ax] <= 0.0 || o[ax] >= (double)grid) return 0;
    } else {
      double ta = (0.0 - o[ax]) / d[ax], tb = ((double)grid - o[ax]) / d[ax];
      if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
      if (ta > t0) t0 = ta;
      if (tb < t1) t1 = tb;
    }
  }
  if (!(t1 > t0)) return 0;
  /* axis walks in ascending t */
  int act[2], k[2], step[2];
  double tc[2];
  for (int ax = 0; ax < 2; ++ax) {
    act[ax] = fabs(d[ax]) >= 1e-12;
    tc[ax] = INFINITY;
    if (!act[ax]) continue;
    step[ax] = d[ax] > 0 ? 1 : -1;
    double p = o[ax] + t0 * d[ax];
    long kk = step[ax] > 0 ? (long)floor(p) + 1 : (long)ceil(p) - 1;
    if (kk < 1) kk = 1;
    if (kk > grid - 1) kk = grid - 1;
    k[ax] = (int)kk;
    while (k[ax] - step[ax] >= 1 && k[ax] - step[ax] <= grid - 1 && cross_t(k[ax] - step[ax], o[ax], d[ax]) > t0)
      k[ax] -= step[ax];
    while (k[ax] >= 1 && k[ax] <= grid - 1 && !(cross_t(k[ax], o[ax], d[ax]) > t0)) k[ax] += step[ax];
    if (k[ax] >= 1 && k[ax] <= grid - 1) {
      double tt = cross_t(k[ax], o[ax], d[ax]);
      tc[ax] = tt < t1 ? tt : INFINITY;
    }
  }
  double prev = t0;
  int64_t count = 0;
  long long last = -1;
  double lastlen = 0.0;
  int done = 0;
  while (!done) {
    double nxt = tc[0] < tc[1] ? tc[0] : tc[1];
    if (nxt == INFINITY) {
      nxt = t1;
      done = 1;
    }
    double len = nxt - prev;
    if (len > 1e-12) {
      double mt = 0.5 * (prev + nxt);
      double mx = r->ox + mt * r->dx, my = r->oy + mt * r->dy;
      long long ci = (long long)floor(mx), rj = (long long)floor(my);
      if (ci < 0) ci = 0;
      if (ci > grid - 1) ci = grid - 1;
      if (rj < 0) rj = 0;
      if (rj > grid - 1) rj = grid - 1;
      long long pix = rj * grid + ci;
      if (pix == last) {
        lastlen = lastlen + len;
        if (out_val) out_val[count - 1] = lastlen;
      } else {
        if (out_col) {
          out_col[count] = (int32_t)pix;
          out_val[count] = len;
        }
        last = pix;
        lastlen = len;
        ++count;
      }
    }
    if (!done) {
      int a0 = tc[0] == nxt, a1 = tc[1] == nxt;
      for (int ax = 0; ax < 2; ++ax) {
        if (!(ax == 0 ? a0 : a1)) continue;
        k[ax] += step[ax];
        if (k[ax] >= 1 && k[ax] <= grid - 1) {
          double tt = cross_t(k[ax], o[ax], d[ax]);
          tc[ax] = tt < t1 ? tt : INFINITY;
        } else {
          tc[ax] = INFINITY;
        }
      }
    }
    prev = nxt;
  }
  return count;
}

static void make_ray(int grid, const double* cos_t, const double* sin_t, const double* offs, int n_bins, int64_t r,
                     ray_t* out) {
  int a = (int)(r / n_bins), j = (int)(r % n_bins);
  double half = (double)grid / 2.0;
  out->grid = grid;
  out->ox = half + offs[j] * (-sin_t[a]);
  out->oy = half + offs[j] * cos_t[a];
  out->dx = cos_t[a];
  out->dy = sin_t[a];
}

/* per-ray counts; rowptr[m+1] is filled (exclusive scan) */
void co_tomo_rowptr(int grid, int n_angles, int n_bins, const double* cos_t, const double* sin_t,
                    const double* offs, int64_t* rowptr, int nthreads) {
  int64_t m = (int64_t)n_angles * n_bins;
#pragma omp parallel for schedule(dynamic, 256) num_threads(nthreads)
  for (int64_t r = 0; r < m; ++r) {
    ray_t ray;
    make_ray(grid, cos_t, sin_t, offs, n_bins, r, &ray);
    rowptr[r + 1] = trace(&ray, NULL, NULL);
  }
  rowptr[0] = 0;
  for (int64_t r = 0; r < m; ++r) rowptr[r + 1] += rowptr[r];
}

/* fill: per row, traversal order then ascending column (run reversal for -x rays) */
void co_tomo_fill(int grid, int n_angles, int n_bins, const double* cos_t, const double* sin_t, const double* offs,
                  const int64_t* rowptr, int32_t* col, float* val, int nthreads) {
  int64_t m = (int64_t)n_angles * n_bins;
#pragma omp parallel num_threads(nthreads)
  {
    double* tmpv = (double*)malloc(sizeof(double) * (size_t)(4 * grid + 8));
    int32_t* tmpc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(4 * grid + 8));
#pragma omp for schedule(dynamic, 256)
    for (int64_t r = 0; r < m; ++r) {
      ray_t ray;
      make_ray(grid, cos_t, sin_t, offs, n_bins, r, &ray);
      int64_t n = trace(&ray, tmpc, tmpv);
      if (ray.dx < 0.0) {
        int64_t s = 0;
        while (s < n) {
          int32_t rowid = tmpc[s] / grid;
          int64_t e = s + 1;
          while (e < n && tmpc[e] / grid == rowid) ++e;
          for (int64_t lo = s, hi = e - 1; lo < hi; ++lo, --hi) {
            int32_t tc = tmpc[lo]; tmpc[lo] = tmpc[hi]; tmpc[hi] = tc;
            double tv = tmpv[lo]; tmpv[lo] = tmpv[hi]; tmpv[hi] = tv;
          }
          s = e;
        }
      }
      int64_t b = rowptr[r];
      for (int64_t i = 0; i < n; ++i) {
        col[b + i] = tmpc[i];
        val[b + i] = (float)tmpv[i];
      }
    }
    free(tmpv);
    free(tmpc);
  }
}

/* A^T as CSR with rows sorted by source row (stable, chunked counting sort) */
void co_csr_transpose(int64_t m, int64_t n, const int64_t* rp, const int32_t* ci, const float* cv, int64_t* trp,
                      int32_t* tci, float* tcv, int nthreads) {
  /* T fixed row chunks, each handled by one loop iteration: correct whatever
     team size the runtime grants (chunk t must not depend on thread ids) */
  int T = nthreads > 0 ? nthreads : 1;
  int64_t* cnt = (int64_t*)calloc((size_t)T * (size_t)n, sizeof(int64_t));
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int t = 0; t < T; ++t) {
    int64_t r0 = m * t / T, r1 = m * (t + 1) / T;
    int64_t* c = cnt + (size_t)t * n;
    for (int64_t p = rp[r0]; p < rp[r1]; ++p) c[ci[p]]++;
  }
  /* column-major prefix over (column, chunk) */
  int64_t run = 0;
  for (int64_t j = 0; j < n; ++j) {
    trp[j] = run;
    for (int t = 0; t < T; ++t) {
      int64_t v = cnt[(size_t)t * n + j];
      cnt[(size_t)t * n + j] = run;
      run += v;
    }
  }
  trp[n] = run;
#pragma omp parallel for schedule(static, 1) num_threads(T)
  for (int t = 0; t < T; ++t) {
    int64_t r0 = m * t / T, r1 = m * (t + 1) / T;
    int64_t* c = cnt + (size_t)t * n;
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t p = rp[r]; p < rp[r + 1]; ++p) {
        int64_t dst = c[ci[p]]++;
        tci[dst] = (int32_t)r;
        tcv[dst] = cv[p];
      }
  }
  free(cnt);
}

/* ------------------------------------------------------------------------ */
/* the loop                                                                  */

static void spmv_f32(int64_t rows, const int64_t* rp, const int32_t* ci, const float* cv, const float* x, float* y,
                     int T) {
#pragma omp parallel for schedule(dynamic, 1024) num_threads(T)
  for (int64_t i = 0; i < rows; ++i) {
    float acc = 0.0f;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      float prod = cv[p] * x[ci[p]];
      acc = acc + prod;
    }
    y[i] = acc;
  }
}

static void sketch_csr(int64_t ell, const int64_t* sp, const int32_t* sc, const double* sv, const float* v,
                       double* z, int T) {
#pragma omp parallel for schedule(static) num_threads(T)
  for (int64_t i = 0; i < ell; ++i) {
    double acc = 0.0;
    for (int64_t p = sp[i]; p < sp[i + 1]; ++p) acc += sv[p] * (double)v[sc[p]];
    z[i] = acc;
  }
}

/* eliminate against basis[0..k-1] at positions pos[], one pass per column */
static void eliminate(float* u, int64_t len, float* const* basis, const int64_t* pos, int k, double* hcol, int T) {
  for (int j = 0; j < k; ++j) {
    float c = u[pos[j]];
    hcol[j] = c;
    const float* b = basis[j];
#pragma omp parallel for schedule(static) num_threads(T)
    for (int64_t e = 0; e < len; ++e) {
      float prod = c * b[e];
      u[e] = u[e] - prod;
    }
  }
}

static void argmax_abs(const float* u, int64_t len, int64_t* idx, float* val, int T) {
  int64_t bi = -1;
  float bm = -1.0f;
#pragma omp parallel num_threads(T)
  {
    int64_t li = -1;
    float lm = -1.0f;
#pragma omp for schedule(static) nowait
    for (int64_t e = 0; e < len; ++e) {
      float a = fabsf(u[e]);
      if (a > lm) {
        lm = a;
        li = e;
      }
    }
#pragma omp critical
    {
      if (lm > bm || (lm == bm && li < bi)) {
        bm = lm;
        bi = li;
      }
    }
  }
  *idx = bi;
  *val = bi >= 0 ? u[bi] : 0.0f;
}

/* min ||M y - rhs|| by Householder QR from scratch (M: l x k column-major, copied) */
static void ls_qr(const double* M, int64_t l, int k, const double* rhs, double* y, double* work) {
  double* A = work;                     /* l*k */
  double* b = work + (size_t)l * k;     /* l */
  memcpy(A, M, sizeof(double) * (size_t)l * k);
  memcpy(b, rhs, sizeof(double) * (size_t)l);
  for (int j = 0; j < k; ++j) {
    double* a = A + (size_t)j * l;
    double nrm = 0.0;
    for (int64_t i = j; i < l; ++i) nrm += a[i] * a[i];
    nrm = sqrt(nrm);
    if (nrm == 0.0) continue;
    double alpha = a[j] > 0 ? -nrm : nrm;
    a[j] -= alpha;
    double vnorm2 = 0.0;
    for (int64_t i = j; i < l; ++i) vnorm2 += a[i] * a[i];
    for (int jj = j + 1; jj < k; ++jj) {
      double* c = A + (size_t)jj * l;
      double s = 0.0;
      for (int64_t i = j; i < l; ++i) s += a[i] * c[i];
      s = 2.0 * s / vnorm2;
      for (int64_t i = j; i < l; ++i) c[i] -= s * a[i];
    }
    double s = 0.0;
    for (int64_t i = j; i < l; ++i) s += a[i] * b[i];
    s = 2.0 * s / vnorm2;
    for (int64_t i = j; i < l; ++i) b[i] -= s * a[i];
    a[j] = alpha; /* R diagonal */
  }
  for (int j = k - 1; j >= 0; --j) {
    double s = b[j];
    for (int jj = j + 1; jj < k; ++jj) s -= A[(size_t)jj * l + j] * y[jj];
    double rjj = A[(size_t)j * l + j];
    y[j] = rjj != 0.0 ? s / rjj : 0.0;
  }
}

/*
 * sLSLU, lam = 0, float32 vectors.  Runs until maxiter, a breakdown, or until
 * `budget_s` seconds have elapsed (bounded sample).  Outputs: t/g pivots
 * (maxiter+1 each), per-iteration sres and wall seconds, x of the last
 * iteration.  Returns the number of iterations done.
 */
int co_slslu_f32(int64_t m, int64_t n, const int64_t* Arp, const int32_t* Aci, const float* Acv, const int64_t* Trp,
                 const int32_t* Tci, const float* Tcv, int64_t ell, const int64_t* Srp, const int32_t* Sci,
                 const double* Scv, const double* b, int maxiter, int nthreads, double budget_s, int64_t* t_out,
                 int64_t* g_out, double* sres_out, double* iter_s_out, double* x_out) {
  int T = nthreads > 0 ? nthreads : omp_get_max_threads();
  int K = maxiter;
  float** D = (float**)calloc((size_t)K + 2, sizeof(float*));
  float** L = (float**)calloc((size_t)K + 2, sizeof(float*));
  int64_t* t = (int64_t*)calloc((size_t)K + 2, sizeof(int64_t));
  int64_t* g = (int64_t*)calloc((size_t)K + 2, sizeof(int64_t));
  double* hcol = (double*)malloc(sizeof(double) * ((size_t)K + 2));
  float* r0 = (float*)malloc(sizeof(float) * (size_t)m);
  float* u = (float*)malloc(sizeof(float) * (size_t)m);
  float* q = (float*)malloc(sizeof(float) * (size_t)n);
  double* Z = (double*)malloc(sizeof(double) * (size_t)ell * K);
  double* sr0 = (double*)malloc(sizeof(double) * (size_t)ell);
  double* y = (double*)calloc((size_t)K + 1, sizeof(double));
  double* work = (double*)malloc(sizeof(double) * ((size_t)ell * K + ell));
  for (int64_t i = 0; i < m; ++i) r0[i] = (float)b[i];
  int64_t idx;
  float val;
  int done = 0;
  argmax_abs(r0, m, &idx, &val, T);
  if (val == 0.0f) goto out;
  t[0] = idx;
  D[0] = (float*)malloc(sizeof(float) * (size_t)m);
  for (int64_t i = 0; i < m; ++i) D[0][i] = r0[i] / val;
  spmv_f32(n, Trp, Tci, Tcv, r0, q, T);
  argmax_abs(q, n, &idx, &val, T);
  if (val == 0.0f) goto out;
  g[0] = idx;
  L[0] = (float*)malloc(sizeof(float) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) L[0][i] = q[i] / val;
  spmv_f32(n, Trp, Tci, Tcv, D[0], q, T); /* W(1,1) (not needed further) */
  sketch_csr(ell, Srp, Sci, Scv, r0, sr0, T);
  double t_start = now_s();
  for (int k = 1; k <= K; ++k) {
    double tic = now_s();
    int bd = 0;
    spmv_f32(m, Arp, Aci, Acv, L[k - 1], u, T);
    sketch_csr(ell, Srp, Sci, Scv, u, Z + (size_t)(k - 1) * ell, T);
    eliminate(u, m, D, t, k, hcol, T);
    argmax_abs(u, m, &idx, &val, T);
    if (k >= m || val == 0.0f) bd = 1;
    if (!bd) {
      t[k] = idx;
      D[k] = (float*)malloc(sizeof(float) * (size_t)m);
      float* dk = D[k];
#pragma omp parallel for schedule(static) num_threads(T)
      for (int64_t i = 0; i < m; ++i) dk[i] = u[i] / val;
      spmv_f32(n, Trp, Tci, Tcv, dk, q, T);
      eliminate(q, n, L, g, k, hcol, T);
      argmax_abs(q, n, &idx, &val, T);
      if (k >= n || val == 0.0f) bd = 1;
      if (!bd) {
        g[k] = idx;
        L[k] = (float*)malloc(sizeof(float) * (size_t)n);
        float* lk = L[k];
#pragma omp parallel for schedule(static) num_threads(T)
        for (int64_t i = 0; i < n; ++i) lk[i] = q[i] / val;
      }
    }
    ls_qr(Z, ell, k, sr0, y, work);
    /* sres = |Z y - sr0| */
    double s2 = 0.0;
    for (int64_t i = 0; i < ell; ++i) {
      double a = -sr0[i];
      for (int j = 0; j < k; ++j) a += Z[(size_t)j * ell + i] * y[j];
      s2 += a * a;
    }
    sres_out[k - 1] = sqrt(s2);
    /* x = L_k y (recomputed every iteration, as solvers.py:510) */
#pragma omp parallel for schedule(static) num_threads(T)
    for (int64_t e = 0; e < n; ++e) {
      double a = 0.0;
      for (int j = 0; j < k; ++j) a += y[j] * (double)L[j][e];
      x_out[e] = a;
    }
    iter_s_out[k - 1] = now_s() - tic;
    done = k;
    if (bd) break;
    if (now_s() - t_start > budget_s) break;
  }
out:
  if (t_out) memcpy(t_out, t, sizeof(int64_t) * ((size_t)K + 1));
  if (g_out) memcpy(g_out, g, sizeof(int64_t) * ((size_t)K + 1));
  for (int i = 0; i <= K + 1; ++i) {
    free(D[i]);
    free(L[i]);
  }
  free(D); free(L); free(t); free(g); free(hcol); free(r0); free(u); free(q); free(Z); free(sr0); free(y); free(work);
  return done;
}

int co_max_threads(void) { return omp_get_max_threads(); }

/* y = A x in float32, sequential no-FMA row sums (scipy csr_matvec order): the
   full-size operator checker for the device SpMV */
void co_spmv_f32_export(int64_t rows, const int64_t* rp, const int32_t* ci, const float* cv, const float* x, float* y,
                        int nthreads) {
  spmv_f32(rows, rp, ci, cv, x, y, nthreads);
}

/* y = A x with float values and float64 x / y (input generation: b = A x_true) */
void co_spmv_f32_f64(int64_t rows, const int64_t* rp, const int32_t* ci, const float* cv, const double* x, double* y,
                     int nthreads) {
#pragma omp parallel for schedule(dynamic, 1024) num_threads(nthreads)
  for (int64_t i = 0; i < rows; ++i) {
    double acc = 0.0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) acc = acc + (double)cv[p] * x[ci[p]];
    y[i] = acc;
  }
}

/* ---- square process on the PSF operator (BASELINE config 5, fp32 storage) ----
   out[r, c] = sum over a (outer), b (inner) of K[a, b] * x[r + ry - a, c + rx - b]
   (zero outside; each product rounded, then added to the running sum from +0):
   the order-specified stencil of oracle/tomo_oracle.py:psf_stencil (transpose
   = False), which the device stencil reproduces bit for bit. */
static void psf_conv_f32(int Hh, int Ww, const float* K, int kh, int kw, const float* x, float* out, int T) {
  const int ry = kh / 2, rx = kw / 2;
#pragma omp parallel num_threads(T)
  {
    float* acc = (float*)malloc(sizeof(float) * (size_t)Ww);
#pragma omp for schedule(static)
    for (int r = 0; r < Hh; ++r) {
      for (int c = 0; c < Ww; ++c) acc[c] = 0.0f;
      for (int a = 0; a < kh; ++a) {
        const int rr = r + ry - a;
        for (int b = 0; b < kw; ++b) {
          const float kab = K[a * kw + b];
          const int off = rx - b;
          if (rr < 0 || rr >= Hh) {
            /* zero row: every product is +0 or -0 times kab; acc + (+-0) keeps acc
               unless acc is -0, which it never is (it starts at +0) */
            continue;
          }
          const float* xr = x + (size_t)rr * Ww;
          const int c0 = off < 0 ? -off : 0, c1 = Ww - (off > 0 ? off : 0);
          for (int c = 0; c < c0; ++c) acc[c] = acc[c] + kab * 0.0f;
          for (int c = c0; c < c1; ++c) {
            float prod = kab * xr[c + off];
            acc[c] = acc[c] + prod;
          }
          for (int c = c1; c < Ww; ++c) acc[c] = acc[c] + kab * 0.0f;
        }
      }
      memcpy(out + (size_t)r * Ww, acc, sizeof(float) * (size_t)Ww);
    }
    free(acc);
  }
}

void co_psf_conv_f32(int Hh, int Ww, const float* K, int kh, int kw, const float* x, float* out, int nthreads) {
  psf_conv_f32(Hh, Ww, K, kh, kw, x, out, nthreads > 0 ? nthreads : omp_get_max_threads());
}

/* hessenberg.py:160-226 (full pivoting), float32 vectors and basis: pivots t
   (maxiter + 1) and H columns (h_out[j * (maxiter + 1) + i], column-major).
   Returns the number of steps done. */
int co_scmrh_psf_f32(int Hh, int Ww, const float* K, int kh, int kw, const double* b, int maxiter, int nthreads,
                     int64_t* t_out, double* h_out) {
  const int T = nthreads > 0 ? nthreads : omp_get_max_threads();
  const int64_t n = (int64_t)Hh * Ww;
  const int KK = maxiter;
  float** L = (float**)calloc((size_t)KK + 2, sizeof(float*));
  int64_t* t = (int64_t*)calloc((size_t)KK + 2, sizeof(int64_t));
  double* hcol = (double*)calloc((size_t)KK + 2, sizeof(double));
  float* u = (float*)malloc(sizeof(float) * (size_t)n);
  int64_t idx;
  float val;
  int done = 0;
  for (int64_t i = 0; i < n; ++i) u[i] = (float)b[i];
  argmax_abs(u, n, &idx, &val, T);
  if (val == 0.0f) goto out2;
  t[0] = idx;
  L[0] = (float*)malloc(sizeof(float) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) L[0][i] = u[i] / val;
  for (int k = 1; k <= KK; ++k) {
    psf_conv_f32(Hh, Ww, K, kh, kw, L[k - 1], u, T);
    for (int i = 0; i <= KK; ++i) hcol[i] = 0.0;
    eliminate(u, n, L, t, k, hcol, T);
    argmax_abs(u, n, &idx, &val, T);
    const int bd = (k >= n || val == 0.0f);
    hcol[k] = bd ? 0.0 : (double)val;
    if (h_out) memcpy(h_out + (size_t)(k - 1) * (KK + 1), hcol, sizeof(double) * ((size_t)KK + 1));
    done = k;
    if (bd) break;
    t[k] = idx;
    L[k] = (float*)malloc(sizeof(float) * (size_t)n);
    float* lk = L[k];
#pragma omp parallel for schedule(static) num_threads(T)
    for (int64_t i = 0; i < n; ++i) lk[i] = u[i] / val;
  }
out2:
  if (t_out) memcpy(t_out, t, sizeof(int64_t) * ((size_t)KK + 1));
  for (int i = 0; i <= KK + 1; ++i) free(L[i]);
  free(L); free(t); free(hcol); free(u);
  return done;
}

/* ---- reference-arm cost probe: one sLSLU iteration of co_slslu_f32 at step k ----
   The loop's per-iteration work depends on k (k-pass eliminations on both
   sides, the from-scratch QR of the l x k sketched matrix, the iterate
   x = L_k y), not on the basis values, so the rate of a full K-iteration run is
   the mean over k of one iteration's time at each k.  The probe holds a
   K-column stand-in basis (pseudo-random fp32 columns, distinct pivot
   positions) and times the body of co_slslu_f32's loop at any k without
   running the k - 1 iterations before it. */
typedef struct {
  int64_t m, n, ell;
  int kmax;
  float **D, **L;
  int64_t *t, *g;
  double *Z, *sr0, *y, *work, *hcol, *x;
  float *u, *q;
} co_probe;

static float prand(uint64_t* s) {
  *s = *s * 6364136223846793005ULL + 1442695040888963407ULL;
  return (float)((double)(*s >> 40) / (double)(1ULL << 24)) * 2.0f - 1.0f;
}

void* co_probe_create(int64_t m, int64_t n, int64_t ell, int kmax, int nthreads) {
  const int T = nthreads > 0 ? nthreads : omp_get_max_threads();
  co_probe* p = (co_probe*)calloc(1, sizeof(co_probe));
  p->m = m; p->n = n; p->ell = ell; p->kmax = kmax;
  p->D = (float**)calloc((size_t)kmax + 2, sizeof(float*));
  p->L = (float**)calloc((size_t)kmax + 2, sizeof(float*));
  p->t = (int64_t*)calloc((size_t)kmax + 2, sizeof(int64_t));
  p->g = (int64_t*)calloc((size_t)kmax + 2, sizeof(int64_t));
  for (int j = 0; j <= kmax; ++j) {
    p->D[j] = (float*)malloc(sizeof(float) * (size_t)m);
    p->L[j] = (float*)malloc(sizeof(float) * (size_t)n);
    p->t[j] = (int64_t)(((uint64_t)j * 2654435761ULL) % (uint64_t)m);
    p->g[j] = (int64_t)(((uint64_t)j * 40503ULL + 17) % (uint64_t)n);
#pragma omp parallel num_threads(T)
    {
      uint64_t sd = 0x9E3779B97F4A7C15ULL ^ ((uint64_t)j << 20) ^ (uint64_t)omp_get_thread_num();
#pragma omp for schedule(static)
      for (int64_t i = 0; i < m; ++i) p->D[j][i] = prand(&sd);
#pragma omp for schedule(static)
      for (int64_t i = 0; i < n; ++i) p->L[j][i] = prand(&sd);
    }
  }
  /* unit pivots, zeros at the other pivot rows (as partial pivoting leaves
     them): the elimination coefficients stay the size of u's entries */
  for (int j = 0; j <= kmax; ++j)
    for (int i = 0; i <= kmax; ++i) {
      p->D[j][p->t[i]] = i == j ? 1.0f : 0.0f;
      p->L[j][p->g[i]] = i == j ? 1.0f : 0.0f;
    }
  p->Z = (double*)malloc(sizeof(double) * (size_t)ell * (kmax + 1));
  uint64_t sd = 12345;
  for (int64_t i = 0; i < ell * (kmax + 1); ++i) p->Z[i] = (double)prand(&sd);
  p->sr0 = (double*)malloc(sizeof(double) * (size_t)ell);
  for (int64_t i = 0; i < ell; ++i) p->sr0[i] = (double)prand(&sd);
  p->y = (double*)calloc((size_t)kmax + 1, sizeof(double));
  p->work = (double*)malloc(sizeof(double) * ((size_t)ell * (kmax + 1) + ell));
  p->hcol = (double*)calloc((size_t)kmax + 2, sizeof(double));
  p->x = (double*)malloc(sizeof(double) * (size_t)n);
  p->u = (float*)malloc(sizeof(float) * (size_t)m);
  p->q = (float*)malloc(sizeof(float) * (size_t)n);
  return p;
}

void co_probe_destroy(void* vp) {
  co_probe* p = (co_probe*)vp;
  if (!p) return;
  for (int j = 0; j <= p->kmax; ++j) {
    free(p->D[j]);
    free(p->L[j]);
  }
  free(p->D); free(p->L); free(p->t); free(p->g); free(p->Z); free(p->sr0); free(p->y); free(p->work);
  free(p->hcol); free(p->x); free(p->u); free(p->q);
  free(p);
}

/* seconds for one iteration of co_slslu_f32's loop body at step k (1 <= k <= kmax) */
double co_probe_iter(void* vp, int k, const int64_t* Arp, const int32_t* Aci, const float* Acv, const int64_t* Trp,
                     const int32_t* Tci, const float* Tcv, const int64_t* Srp, const int32_t* Sci, const double* Scv,
                     int nthreads) {
  co_probe* p = (co_probe*)vp;
  const int T = nthreads > 0 ? nthreads : omp_get_max_threads();
  const int64_t m = p->m, n = p->n, ell = p->ell;
  int64_t idx;
  float val;
  const double tic = now_s();
  spmv_f32(m, Arp, Aci, Acv, p->L[k - 1], p->u, T);
  sketch_csr(ell, Srp, Sci, Scv, p->u, p->Z + (size_t)(k - 1) * ell, T);
  eliminate(p->u, m, p->D, p->t, k, p->hcol, T);
  argmax_abs(p->u, m, &idx, &val, T);
  if (val == 0.0f) val = 1.0f;
  {
    float* dk = p->D[k];
    const float* u = p->u;
#pragma omp parallel for schedule(static) num_threads(T)
    for (int64_t i = 0; i < m; ++i) dk[i] = u[i] / val;
  }
  spmv_f32(n, Trp, Tci, Tcv, p->D[k], p->q, T);
  eliminate(p->q, n, p->L, p->g, k, p->hcol, T);
  argmax_abs(p->q, n, &idx, &val, T);
  if (val == 0.0f) val = 1.0f;
  {
    float* lk = p->L[k];
    const float* q = p->q;
#pragma omp parallel for schedule(static) num_threads(T)
    for (int64_t i = 0; i < n; ++i) lk[i] = q[i] / val;
  }
  ls_qr(p->Z, ell, k, p->sr0, p->y, p->work);
  double s2 = 0.0;
  for (int64_t i = 0; i < ell; ++i) {
    double a = -p->sr0[i];
    for (int j = 0; j < k; ++j) a += p->Z[(size_t)j * ell + i] * p->y[j];
    s2 += a * a;
  }
  p->hcol[0] = s2;
  double* x = p->x;
  const double* y = p->y;
  float** L = p->L;
#pragma omp parallel for schedule(static) num_threads(T)
  for (int64_t e = 0; e < n; ++e) {
    double a = 0.0;
    for (int j = 0; j < k; ++j) a += y[j] * (double)L[j][e];
    x[e] = a;
  }
  return now_s() - tic;
}
