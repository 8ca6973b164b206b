/* spotfit_oracle.h -- CPU restatement of the reference fit path (TEST INFRASTRUCTURE ONLY).
 * See spotfit_oracle.c for what is restated and the reference file:line of each piece. */
#ifndef SPOTFIT_ORACLE_H
#define SPOTFIT_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define SF_ORACLE_MAXPIX 1024 /* model.py:25 MAX_PIXELS */
#define SF_STEP_GUARD 1e-12   /* SPEC.md:193 StepFailed guard, pinned */

/* StopReason codes -- identical values to include/spotfit.h */
#define SF_STOP_MAX_ERROR 0
#define SF_STOP_MIN_DELTA 1
#define SF_STOP_MIN_STEP 2
#define SF_STOP_NOT_CONVERGED 3
#define SF_STOP_MAX_ITERATIONS 4
#define SF_FLAG_INVALID 0x40 /* InvalidInput */
#define SF_FLAG_NOIMP 0x80   /* no improvement after the retry loop (SURVEY App. A [A2]) */

typedef struct {
  int max_iterations;
  double max_error, min_delta, min_step;
  double lambda_init, lambda_up, lambda_down, lambda_max;
  double margin_x, margin_y, sigma_min, sigma_max;
} sf_oracle_config_t;

typedef struct {
  int singular;
  float alpha, beta, chi;
  double F, G, FF, FG, denom;
  double dF[4], dFF[4], dFG[4], gamma[4], dalpha[4], dbeta[4];
  double rhs[5];   /* P = 5: explicit (x, y, sigma, alpha, beta) model */
  double jtj[15];
} sf_oracle_eval_t;

typedef struct {
  float params[5];
  float alpha, beta, nchi2;
  uint8_t status, iterations;
} sf_oracle_result_t;

float npexp_f32(float x);
float npexp_f32_clamped(float x);
int64_t npexp_clamp_mismatches(float lo, float hi);
void npexp_f32_array(const float* x, float* y, int64_t n);
double pw_sum(const float* a, int n);
int sf_oracle_eval(const float* g, int W, int H, int P, const float* p, sf_oracle_eval_t* e);
int sf_oracle_solve(int P, const double* jtj, const double* rhs, double lam, double* delta);
int sf_oracle_fit(const float* g, int W, int H, int P, const float* init, const sf_oracle_config_t* c,
                  sf_oracle_result_t* res);
int sf_oracle_fit_batch(const float* images, int W, int H, int64_t count, int P, const float* inits,
                        const sf_oracle_config_t* c, float* out_params, float* out_alpha, float* out_beta,
                        float* out_nchi2, uint8_t* out_status, uint8_t* out_iters, int threads);
int sf_oracle_eval_batch(const float* images, int W, int H, int64_t count, int P, const float* params,
                         sf_oracle_eval_t* out, int threads);
int sf_oracle_eval_size(void);

#ifdef __cplusplus
}
#endif
#endif
