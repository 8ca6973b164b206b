/*
 * spotfit_oracle.c -- CPU restatement of the reference fit path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker for the CUDA product
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product (paper_2106_02045_b200/)
 * never links or calls it.
 *
 * What is restated, and from where (all citations into /root/reference):
 *   npexp_f32        numpy 2.3.5 float32 exp (AVX512F/AVX2 simd_exp_f32), the
 *                    np.exp called at pkg/src/spotfit/model.py:177,193.
 *                    Constants / op order: SURVEY.md App. B.2 (third-party
 *                    dependency numpy>=1.24, pyproject.toml:12).  Pinned by
 *                    tests/test_oracle_numerics.py against this host's np.exp.
 *   pw_sum           numpy float64 pairwise add-reduce of a float32 array
 *                    (x.sum(dtype=np.float64), model.py:222-225,250,263-265,314)
 *                    SURVEY.md App. B.3.  Pinned against np.sum in tests.
 *   sf_oracle_eval   model.py:154-315 (profile_and_gradient, alpha_beta,
 *                    chi_squared, gradient_sums, coefficient_gradients,
 *                    chi_gradient) + the normal matrix of SPEC.md:173-176.
 *                    Pinned bit-for-bit against the reference model.py via
 *                    the tests/golden npz fixtures (tests/golden/make_golden.py).
 *   sf_oracle_fit    LM state machine of PAPER.md:126-180 / SPEC.md:209-262 as
 *                    pinned in SURVEY.md App. A (and DESIGN.md section 3).
 *   elliptical (P=4) SURVEY.md App. B.5 -- no reference exists (SPEC.md:152
 *                    lists it as a non-goal): parity for P=4 is unpinned.
 *
 * Build: oracle/Makefile  (-O2 -ffp-contract=off: no FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <float.h>
#include <pthread.h>

#include "spotfit_oracle.h"

/* ------------------------------------------------------------------ */
/* numpy float32 exp                                 */
/* ------------------------------------------------------------------ */
static float ldexp_single_round(float r, int q) {
  /* r in [0.7, 1.42]; one rounding of r * 2^q, denormals kept */
  if (q >= -126 && q <= 127) {
    union { uint32_t u; float f; } s; s.u = (uint32_t)(q + 127) << 23;
    return r * s.f;
  }
  if (q > 127) {                       /* r*2*2^127: first product exact */
    union { uint32_t u; float f; } s; s.u = (uint32_t)(127 + 127) << 23;
    return (r * 2.0f) * s.f;
  }
  { /* q < -126: r*2^(q+64) exact (normal), then *2^-64 rounds once */
    union { uint32_t u; float f; } s; s.u = (uint32_t)(q + 64 + 127) << 23;
    union { uint32_t u; float f; } t; t.u = (uint32_t)(-64 + 127) << 23;
    return (r * s.f) * t.f;
  }
}

/* The fit kernel's packed exp (sf_device.cuh:npexp2) drops the underflow guard and clamps
 * the argument instead: max.NaN(x, -104) followed by the unguarded formula.  This restates
 * that form; npexp_clamp_mismatches() counts the float32 x in [lo, hi] where it differs from
 * npexp_f32 (tests/test_oracle_numerics.py: must be none on the kernel's domain x <= 0). */
float npexp_f32_clamped(float x) {
  if (x != x) return x;
  if (x < -104.0f) x = -104.0f;
  volatile float t = x * 1.442695040888963407359924681001892137f;
  float q = (t + 0x1.8p23f) - 0x1.8p23f;
  float y = fmaf(q, -6.93145752e-1f, x);
  y = fmaf(q, -1.42860677e-6f, y);
  float n = fmaf(5.082762527590693718096e-4f, y, 6.757896990527504603057e-3f);
  n = fmaf(n, y, 5.114512081637298353406e-2f);
  n = fmaf(n, y, 2.473615434895520810817e-1f);
  n = fmaf(n, y, 7.257664613233124478488e-1f);
  n = fmaf(n, y, 9.999999999980870924916e-1f);
  float d = fmaf(2.159509375685829852307e-2f, y, -2.742335390411667452936e-1f);
  d = fmaf(d, y, 1.0f);
  float r = n / d;
  return ldexp_single_round(r, (int)q);
}

int64_t npexp_clamp_mismatches(float lo, float hi) {
  int64_t bad = 0;
  for (float x = lo; x <= hi; x = nextafterf(x, INFINITY)) {
    const float a = npexp_f32(x), b = npexp_f32_clamped(x);
    uint32_t ua, ub;
    memcpy(&ua, &a, 4);
    memcpy(&ub, &b, 4);
    bad += ua != ub;
    if (x == hi) break;
  }
  return bad;
}

float npexp_f32(float x) {
  if (x != x) return x;
  if (x >= 88.72283935546875f) return INFINITY;
  if (x <= -103.97208404541015625f) return 0.0f;
  volatile float t = x * 1.442695040888963407359924681001892137f; /* rounded mul */
  float q = (t + 0x1.8p23f) - 0x1.8p23f;                            /* RNE to int */
  float y = fmaf(q, -6.93145752e-1f, x);
  y = fmaf(q, -1.42860677e-6f, y);
  float n = fmaf(5.082762527590693718096e-4f, y, 6.757896990527504603057e-3f);
  n = fmaf(n, y, 5.114512081637298353406e-2f);
  n = fmaf(n, y, 2.473615434895520810817e-1f);
  n = fmaf(n, y, 7.257664613233124478488e-1f);
  n = fmaf(n, y, 9.999999999980870924916e-1f);
  float d = fmaf(2.159509375685829852307e-2f, y, -2.742335390411667452936e-1f);
  d = fmaf(d, y, 1.0f);
  float r = n / d;
  return ldexp_single_round(r, (int)q);
}

typedef struct { const float* x; float* y; int64_t n; } npexp_job_t;

static void* npexp_job(void* a) {
  npexp_job_t* j = (npexp_job_t*)a;
  for (int64_t i = 0; i < j->n; ++i) j->y[i] = npexp_f32(j->x[i]);
  return NULL;
}

void npexp_f32_array(const float* x, float* y, int64_t n) {
  enum { T = 16 };
  if (n < (1 << 20)) {
    npexp_job_t j = {x, y, n};
    npexp_job(&j);
    return;
  }
  pthread_t tid[T];
  npexp_job_t jobs[T];
  for (int t = 0; t < T; ++t) {
    const int64_t lo = n * t / T, hi = n * (t + 1) / T;
    jobs[t].x = x + lo; jobs[t].y = y + lo; jobs[t].n = hi - lo;
    pthread_create(&tid[t], NULL, npexp_job, &jobs[t]);
  }
  for (int t = 0; t < T; ++t) pthread_join(tid[t], NULL);
}

/* ------------------------------------------------------------------ */
/* numpy pairwise float64 sum of float32             */
/* ------------------------------------------------------------------ */
static double pw_rec(const float* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += (double)a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = (double)a[k];
    int i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] += (double)a[i + k];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += (double)a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return pw_rec(a, n2) + pw_rec(a + n2, n - n2);
}

double pw_sum(const float* a, int n) { return 0.0 + pw_rec(a, n); }

/* ------------------------------------------------------------------ */
/* model evaluation (model.py:154-315)                */
/* ------------------------------------------------------------------ */
#define DENOM_GUARD 1e-12 /* model.py:28 */

/* Explicit 5-parameter model (the Gpufit-like baseline; no
 * reference code -- pinned here in the same numeric style): p = (x, y, sigma,
 * alpha, beta), h = alpha*f + beta, model derivatives
 * d = (alpha*df/dx, alpha*df/dy, alpha*df/dsigma, f, 1) in f32, chi^2, rhs = sum r*d
 * and JtJ = sum d_j*d_k as f64 numpy-order sums of f32 products. */
static int eval_explicit5(const float* g, int W, int H, const float* p, sf_oracle_eval_t* e) {
  const int N = W * H;
  float t[SF_ORACLE_MAXPIX], d[5][SF_ORACLE_MAXPIX], r[SF_ORACLE_MAXPIX];
  const float x0 = p[0], y0 = p[1], inv = 1.0f / p[2], a32 = p[3], b32 = p[4];
  for (int i = 0; i < N; ++i) {
    const float xi = (float)(i % W), yi = (float)(i / W);
    const float u = (xi - x0) * inv, v = (yi - y0) * inv;
    const float uu = u * u, vv = v * v;
    const float q = uu + vv;
    const float f = npexp_f32(-0.5f * q);
    const float fs = f * inv;
    const float f0 = u * fs, f1 = v * fs, f2 = q * fs;
    const float h = a32 * f + b32;
    r[i] = g[i] - h;
    d[0][i] = a32 * f0; d[1][i] = a32 * f1; d[2][i] = a32 * f2; d[3][i] = f; d[4][i] = 1.0f;
  }
  for (int i = 0; i < N; ++i) t[i] = r[i] * r[i];
  e->chi = (float)pw_sum(t, N);
  e->alpha = a32; e->beta = b32;
  for (int j = 0; j < 5; ++j) {
    for (int i = 0; i < N; ++i) t[i] = r[i] * d[j][i];
    e->rhs[j] = pw_sum(t, N);
  }
  int m = 0;
  for (int j = 0; j < 5; ++j)
    for (int k = j; k < 5; ++k) {
      for (int i = 0; i < N; ++i) t[i] = d[j][i] * d[k][i];
      e->jtj[m++] = pw_sum(t, N);
    }
  return 0;
}

int sf_oracle_eval(const float* g, int W, int H, int P, const float* p, sf_oracle_eval_t* e) {
  const int N = W * H;
  float f[SF_ORACLE_MAXPIX], fg[4][SF_ORACLE_MAXPIX], t[SF_ORACLE_MAXPIX];
  float d[4][SF_ORACLE_MAXPIX], r[SF_ORACLE_MAXPIX];
  memset(e, 0, sizeof(*e));
  if (N < 1 || N > SF_ORACLE_MAXPIX || P < 3 || P > 5) return -1;
  if (P == 5) return eval_explicit5(g, W, H, p, e);
  /* _scaled_offsets (model.py:154-165) / profile_and_gradient (model.py:180-199) */
  if (P == 3) {
    const float x0 = p[0], y0 = p[1], inv = 1.0f / p[2];
    for (int i = 0; i < N; ++i) {
      const float xi = (float)(i % W), yi = (float)(i / W);
      const float u = (xi - x0) * inv, v = (yi - y0) * inv;
      const float uu = u * u, vv = v * v;
      const float q = uu + vv;
      f[i] = npexp_f32(-0.5f * q);
      const float fs = f[i] * inv;
      fg[0][i] = u * fs; fg[1][i] = v * fs; fg[2][i] = q * fs;
    }
  } else { /* SURVEY App. B.5 (no reference) */
    const float x0 = p[0], y0 = p[1], ix = 1.0f / p[2], iy = 1.0f / p[3];
    for (int i = 0; i < N; ++i) {
      const float xi = (float)(i % W), yi = (float)(i / W);
      const float u = (xi - x0) * ix, v = (yi - y0) * iy;
      const float uu = u * u, vv = v * v;
      const float q = uu + vv;
      f[i] = npexp_f32(-0.5f * q);
      const float fx = f[i] * ix, fy = f[i] * iy;
      fg[0][i] = u * fx; fg[1][i] = v * fy;
      fg[2][i] = u * fg[0][i]; fg[3][i] = v * fg[1][i];
    }
  }
  const double n = (double)N;
  /* alpha_beta (model.py:207-234) */
  e->F = pw_sum(f, N);
  e->G = pw_sum(g, N);
  for (int i = 0; i < N; ++i) t[i] = f[i] * f[i];
  e->FF = pw_sum(t, N);
  for (int i = 0; i < N; ++i) t[i] = f[i] * g[i];
  e->FG = pw_sum(t, N);
  e->denom = n * e->FF - e->F * e->F;
  if (e->denom <= DENOM_GUARD * n * e->FF) { e->singular = 1; return 0; }
  const double alpha = (n * e->FG - e->F * e->G) / e->denom;
  const double beta = (e->G * e->FF - e->F * e->FG) / e->denom;
  e->alpha = (float)alpha; e->beta = (float)beta;
  /* chi_squared (model.py:237-250) */
  const float a32 = e->alpha, b32 = e->beta;
  for (int i = 0; i < N; ++i) { const float h = a32 * f[i] + b32; r[i] = g[i] - h; t[i] = r[i] * r[i]; }
  e->chi = (float)pw_sum(t, N);
  /* gradient_sums (model.py:253-267) */
  for (int j = 0; j < P; ++j) {
    e->dF[j] = pw_sum(fg[j], N);
    for (int i = 0; i < N; ++i) t[i] = f[i] * fg[j][i];
    e->dFF[j] = 2.0 * pw_sum(t, N);
    for (int i = 0; i < N; ++i) t[i] = g[i] * fg[j][i];
    e->dFG[j] = pw_sum(t, N);
    e->gamma[j] = n * e->dFF[j] - 2.0 * e->F * e->dF[j];
  }
  /* coefficient_gradients (model.py:270-288) */
  for (int j = 0; j < P; ++j) {
    e->dalpha[j] = (n * e->dFG[j] - e->G * e->dF[j] - (double)a32 * e->gamma[j]) / e->denom;
    e->dbeta[j] = (e->G * e->dFF[j] - e->FG * e->dF[j] - e->F * e->dFG[j] - (double)b32 * e->gamma[j]) / e->denom;
  }
  /* chi_gradient (model.py:291-315): d_ij, rhs_j = sum r*d_j = -grad_j/2 */
  for (int j = 0; j < P; ++j) {
    const float da = (float)e->dalpha[j], db = (float)e->dbeta[j];
    for (int i = 0; i < N; ++i) {
      const float t1 = da * f[i], t2 = a32 * fg[j][i];
      d[j][i] = (t1 + t2) + db;
    }
    for (int i = 0; i < N; ++i) t[i] = r[i] * d[j][i];
    e->rhs[j] = pw_sum(t, N);
  }
  /* normal matrix: f32 products, f64 pairwise sums */
  int m = 0;
  for (int j = 0; j < P; ++j)
    for (int k = j; k < P; ++k) {
      for (int i = 0; i < N; ++i) t[i] = d[j][i] * d[k][i];
      e->jtj[m++] = pw_sum(t, N);
    }
  return 0;
}

/* ------------------------------------------------------------------ */
/* damped LDL^T solve (pinned in DESIGN.md 3.2)       */
/* ------------------------------------------------------------------ */
static inline int sym_idx(int P, int i, int j) { /* upper-packed row-major */
  if (i > j) { int t = i; i = j; j = t; }
  return i * P - (i * (i - 1)) / 2 + (j - i);
}

/* explicit-5 step ("a 5x5 damped system solved by elimination with
 * partial pivoting"): f64, no FMA, first maximal |pivot| on ties; StepFailed on a
 * zero pivot or |det| <= 1e-12 * prod(damped diagonal). */
static int solve_pivot5(const double* jtj, const double* rhs, double lam, double* delta) {
  enum { P = 5 };
  double M[P][P], b[P];
  for (int i = 0; i < P; ++i) {
    for (int j = 0; j < P; ++j) M[i][j] = jtj[sym_idx(P, i, j)];
    b[i] = rhs[i];
  }
  for (int i = 0; i < P; ++i) M[i][i] = M[i][i] + lam * M[i][i];
  double dprod = M[0][0];
  for (int i = 1; i < P; ++i) dprod = dprod * M[i][i];
  double det = 1.0;
  for (int col = 0; col < P; ++col) {
    int pr = col;
    double best = fabs(M[col][col]);
    for (int r = col + 1; r < P; ++r)
      if (fabs(M[r][col]) > best) { best = fabs(M[r][col]); pr = r; }
    if (!(best > 0.0)) return 0;
    if (pr != col) {
      for (int c = 0; c < P; ++c) { double t = M[col][c]; M[col][c] = M[pr][c]; M[pr][c] = t; }
      double t = b[col]; b[col] = b[pr]; b[pr] = t;
    }
    det = det * M[col][col];
    for (int r = col + 1; r < P; ++r) {
      const double fct = M[r][col] / M[col][col];
      for (int c = col; c < P; ++c) M[r][c] = M[r][c] - fct * M[col][c];
      b[r] = b[r] - fct * b[col];
    }
  }
  if (!(fabs(det) > SF_STEP_GUARD * fabs(dprod))) return 0;
  for (int r = P - 1; r >= 0; --r) {
    double s = b[r];
    for (int c = r + 1; c < P; ++c) s = s - M[r][c] * delta[c];
    delta[r] = s / M[r][r];
  }
  return 1;
}

int sf_oracle_solve(int P, const double* jtj, const double* rhs, double lam, double* delta) {
  if (P == 5) return solve_pivot5(jtj, rhs, lam, delta);
  double A[4][4] = {{0}}, L[4][4] = {{0}}, C[4][4] = {{0}}, D[4] = {0}, z[4] = {0};
  for (int i = 0; i < P; ++i)
    for (int j = 0; j < P; ++j) A[i][j] = jtj[sym_idx(P, i, j)];
  for (int i = 0; i < P; ++i) A[i][i] = A[i][i] + lam * A[i][i];
  for (int i = 0; i < P; ++i) {
    for (int j = 0; j < i; ++j) {
      double s = A[i][j];
      for (int k = 0; k < j; ++k) s = s - C[i][k] * L[j][k];
      C[i][j] = s;
      L[i][j] = s / D[j];
    }
    double s = A[i][i];
    for (int k = 0; k < i; ++k) s = s - C[i][k] * L[i][k];
    D[i] = s;
    if (!(D[i] > 0.0)) return 0;
  }
  double det = D[0], dprod = A[0][0];
  for (int i = 1; i < P; ++i) { det = det * D[i]; dprod = dprod * A[i][i]; }
  if (!(det > SF_STEP_GUARD * dprod)) return 0;
  for (int i = 0; i < P; ++i) {
    double s = rhs[i];
    for (int k = 0; k < i; ++k) s = s - L[i][k] * z[k];
    z[i] = s;
  }
  for (int i = 0; i < P; ++i) z[i] = z[i] / D[i];
  for (int i = P - 1; i >= 0; --i) {
    double s = z[i];
    for (int k = i + 1; k < P; ++k) s = s - L[k][i] * delta[k];
    delta[i] = s;
  }
  return 1;
}

/* ------------------------------------------------------------------ */
/* limit and the LM state machine    */
/* ------------------------------------------------------------------ */
static inline double clampd(double v, double lo, double hi) {
  return v < lo ? lo : (v > hi ? hi : v); /* NaN passes through */
}

static void limit_params(int P, int W, int H, const sf_oracle_config_t* c, const double* v, float* out) {
  out[0] = (float)clampd(v[0], -c->margin_x, (double)(W - 1) + c->margin_x);
  out[1] = (float)clampd(v[1], -c->margin_y, (double)(H - 1) + c->margin_y);
  if (P == 5) {  /* explicit-5: sigma free in sign, |sigma| bounded; alpha, beta free */
    out[2] = (float)(v[2] < 0.0 ? -clampd(-v[2], c->sigma_min, c->sigma_max) : clampd(v[2], c->sigma_min, c->sigma_max));
    out[3] = (float)v[3];
    out[4] = (float)v[4];
    return;
  }
  for (int j = 2; j < P; ++j) out[j] = (float)clampd(v[j], c->sigma_min, c->sigma_max);
}

static void set_result(int P, int N, const float* p, const sf_oracle_eval_t* e, sf_oracle_result_t* res) {
  for (int j = 0; j < P; ++j) res->params[j] = p[j];
  if (e->singular) {
    res->alpha = NAN; res->beta = NAN; res->nchi2 = NAN;
  } else {
    res->alpha = e->alpha; res->beta = e->beta;
    res->nchi2 = N > 5 ? (float)((double)e->chi / (double)(N - 5)) : e->chi;
  }
}

int sf_oracle_fit(const float* g, int W, int H, int P, const float* init, const sf_oracle_config_t* c,
                  sf_oracle_result_t* res) {
  const int N = W * H;
  memset(res, 0, sizeof(*res));
  if (N < 1 || N > SF_ORACLE_MAXPIX || P < 3 || P > 5) return -1;
  /* InvalidInput: per-image status, not a batch failure */
  int bad = 0;
  for (int i = 0; i < N; ++i) bad |= !isfinite(g[i]);
  for (int j = 0; j < P; ++j) bad |= !isfinite(init[j]);
  if (bad) {
    for (int j = 0; j < P; ++j) res->params[j] = init[j];
    res->alpha = res->beta = res->nchi2 = NAN;
    res->status = SF_STOP_NOT_CONVERGED | SF_FLAG_INVALID;
    res->iterations = 0;
    return 0;
  }
  float p[5], best[5], trial[5];
  double v[5], delta[5], thr[5];
  sf_oracle_eval_t Eb, Et;
  {
    for (int j = 0; j < P; ++j) v[j] = (double)init[j];
    limit_params(P, W, H, c, v, p);
  }
  double lam = c->lambda_init;
  int it = 0, stop = SF_STOP_MAX_ITERATIONS, noimp = 0;
  const sf_oracle_eval_t* final_e = NULL;
  const float* final_p = p;
  int have_trial = 0;
  while (it < c->max_iterations) {
    it += 1;
    sf_oracle_eval(g, W, H, P, p, &Eb);                 /* G-eval */
    if (Eb.singular || !isfinite(Eb.chi)) { stop = SF_STOP_NOT_CONVERGED; final_e = &Eb; final_p = p; break; }
    if ((double)Eb.chi < c->max_error) { stop = SF_STOP_MAX_ERROR; final_e = &Eb; final_p = p; break; }
    const float chib = Eb.chi;
    for (int j = 0; j < P; ++j) {
      best[j] = p[j];
      const double a = fabs((double)best[j]);
      thr[j] = c->min_step * (a > 1.0 ? a : 1.0);
    }
    float chit;
    int small;
    /* one trial: solve -> limit -> T-eval; StepFailed => chit=+inf, not small */
#define SF_TRIAL()                                                                  \
    do {                                                                            \
      if (sf_oracle_solve(P, Eb.jtj, Eb.rhs, lam, delta)) {                         \
        for (int j = 0; j < P; ++j) v[j] = (double)best[j] + delta[j];              \
        limit_params(P, W, H, c, v, trial);                                         \
        sf_oracle_eval(g, W, H, P, trial, &Et);                                     \
        have_trial = 1;                                                             \
        chit = Et.singular ? NAN : Et.chi;                                          \
        small = 1;                                                                  \
        for (int j = 0; j < P; ++j) small &= fabs(delta[j]) < thr[j];               \
      } else {                                                                      \
        chit = INFINITY; small = 0; have_trial = 0;                                 \
      }                                                                             \
    } while (0)
    SF_TRIAL();
    if (chib > chit) lam = lam / c->lambda_down;
    while (!small && chib < chit && lam < c->lambda_max) {
      lam = lam * c->lambda_up;
      SF_TRIAL();
    }
#undef SF_TRIAL
    if (isnan(chit) || (chib < chit && lam >= c->lambda_max)) {
      stop = SF_STOP_NOT_CONVERGED; final_e = &Eb; final_p = best; break;
    }
    if (chib < chit) { stop = SF_STOP_MIN_DELTA; noimp = 1; final_e = &Eb; final_p = best; break; } /* [A2] */
    /* accepted: current := trial */
    for (int j = 0; j < P; ++j) p[j] = trial[j];
    (void)have_trial;
    final_e = &Et; final_p = p;
    if ((double)chit < c->max_error) { stop = SF_STOP_MAX_ERROR; break; }
    if ((double)chib * (1.0 - c->min_delta) < (double)chit) { stop = SF_STOP_MIN_DELTA; break; } /* :172 */
    if (small) { stop = SF_STOP_MIN_STEP; break; }                                      /* :174 */
  }
  set_result(P, N, final_p, final_e, res);
  res->status = (uint8_t)(stop | (noimp ? SF_FLAG_NOIMP : 0));
  res->iterations = (uint8_t)it;
  return 0;
}

/* batch drivers: contiguous chunks per pthread */
typedef struct {
  const float* images; int W, H, P; int64_t lo, hi; const float* inits; const sf_oracle_config_t* c;
  const float* params; sf_oracle_eval_t* eout;
  float *out_params, *out_alpha, *out_beta, *out_nchi2; uint8_t *out_status, *out_iters; int err;
} sf_chunk_t;

static void* fit_chunk(void* arg) {
  sf_chunk_t* k = (sf_chunk_t*)arg;
  const int N = k->W * k->H, P = k->P;
  for (int64_t s = k->lo; s < k->hi; ++s) {
    sf_oracle_result_t r;
    k->err |= sf_oracle_fit(k->images + s * N, k->W, k->H, P, k->inits + s * P, k->c, &r);
    for (int j = 0; j < P; ++j) k->out_params[s * P + j] = r.params[j];
    k->out_alpha[s] = r.alpha; k->out_beta[s] = r.beta; k->out_nchi2[s] = r.nchi2;
    k->out_status[s] = r.status; k->out_iters[s] = r.iterations;
  }
  return NULL;
}

static void* eval_chunk(void* arg) {
  sf_chunk_t* k = (sf_chunk_t*)arg;
  const int N = k->W * k->H, P = k->P;
  for (int64_t s = k->lo; s < k->hi; ++s)
    k->err |= sf_oracle_eval(k->images + s * N, k->W, k->H, P, k->params + s * P, k->eout + s);
  return NULL;
}

static int run_chunks(sf_chunk_t* proto, int64_t count, int threads, void* (*fn)(void*)) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  if ((int64_t)threads > count) threads = count > 0 ? (int)count : 1;
  pthread_t tid[256];
  sf_chunk_t ks[256];
  int err = 0;
  for (int t = 0; t < threads; ++t) {
    ks[t] = *proto;
    ks[t].lo = count * t / threads; ks[t].hi = count * (t + 1) / threads; ks[t].err = 0;
    if (t > 0) pthread_create(&tid[t], NULL, fn, &ks[t]);
  }
  fn(&ks[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
  for (int t = 0; t < threads; ++t) err |= ks[t].err;
  return err ? -1 : 0;
}

int sf_oracle_fit_batch(const float* images, int W, int H, int64_t count, int P, const float* inits,
                        const sf_oracle_config_t* c, float* out_params, float* out_alpha, float* out_beta,
                        float* out_nchi2, uint8_t* out_status, uint8_t* out_iters, int threads) {
  const int N = W * H;
  if (N < 1 || N > SF_ORACLE_MAXPIX || P < 3 || P > 5 || c->max_iterations < 1 || c->max_iterations > 255)
    return -1;
  sf_chunk_t k;
  memset(&k, 0, sizeof(k));
  k.images = images; k.W = W; k.H = H; k.P = P; k.inits = inits; k.c = c;
  k.out_params = out_params; k.out_alpha = out_alpha; k.out_beta = out_beta; k.out_nchi2 = out_nchi2;
  k.out_status = out_status; k.out_iters = out_iters;
  return run_chunks(&k, count, threads, fit_chunk);
}

int sf_oracle_eval_batch(const float* images, int W, int H, int64_t count, int P, const float* params,
                         sf_oracle_eval_t* out, int threads) {
  sf_chunk_t k;
  memset(&k, 0, sizeof(k));
  k.images = images; k.W = W; k.H = H; k.P = P; k.params = params; k.eout = out;
  return run_chunks(&k, count, threads, eval_chunk);
}

int sf_oracle_eval_size(void) { return (int)sizeof(sf_oracle_eval_t); }
