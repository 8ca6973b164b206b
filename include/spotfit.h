/*
 * spotfit.h -- C-ABI of the B200-native implicit-amplitude LM spot fitter.
 *
 * Drop-in boundary for the reference's batch fit path.  The
 * reference (arXiv 2106.02045, /root/reference) exposes this path as Python:
 *
 *   fit_batch(BatchRequest{images, inits|None, config, engine, workers})
 *       -> [FitResult]
 *   fit_single(image, init, config) -> FitResult
 *   the model arithmetic spotfit.model.*                   pkg/src/spotfit/model.py:154-315
 *   estimate_initial(image, bounds)
 *   simulate_spot / simulate_batch
 *
 * Each entry point below cites the reference interface it replaces.  Plain
 * pointers and sizes only; no torch types.  All functions are reentrant and
 * blocking; the library keeps per-device streams and scratch memory in an
 * internal context guarded by a mutex per device.  A non-zero return code is
 * reserved for argument, CUDA or launch failures (message: sf_last_error());
 * per-spot failures are reported in out_status.
 *
 * Result layout per spot: shape params
 * (x, y, sigma) or (x, y, sigma_x, sigma_y), alpha, beta, normalised chi^2,
 * status byte (StopReason in the low 3 bits + flags), iterations used.
 */
#ifndef SPOTFIT_H
#define SPOTFIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SF_ABI_VERSION 1

/* StopReason in the low 3 bits of the status byte */
#define SF_STOP_MAX_ERROR 0
#define SF_STOP_MIN_DELTA 1
#define SF_STOP_MIN_STEP 2
#define SF_STOP_NOT_CONVERGED 3
#define SF_STOP_MAX_ITERATIONS 4
#define SF_FLAG_INVALID 0x40 /* InvalidInput: non-finite pixel or init */
#define SF_FLAG_NOIMP 0x80   /* no chi^2 decrease after the lambda retries (SURVEY App. A [A2]) */

/* model selector */
#define SF_MODEL_SYMMETRIC 3  /* (x, y, sigma)            model.py:100-115 */
#define SF_MODEL_ELLIPTICAL 4 /* (x, y, sigma_x, sigma_y) SURVEY App. B.5, no reference */
/* explicit 5-parameter baseline fit_explicit5: LM over (x, y, sigma, alpha,
 * beta), 5x5 pivoted solve, sigma free in sign; inits and out_params are [count][5] */
#define SF_MODEL_EXPLICIT5 5

/* FitConfig + ParameterBounds (defaults) */
typedef struct sf_config {
  int32_t model;          /* SF_MODEL_SYMMETRIC | SF_MODEL_ELLIPTICAL */
  int32_t max_iterations; /* 1..255, default 20 */
  double max_error;       /* chi^2 early stop, default 0 = disabled */
  double min_delta;       /* relative chi^2 improvement, default 1e-6 */
  double min_step;        /* relative parameter change, default 1e-4 */
  double lambda_init;     /* 0.01 */
  double lambda_up;       /* 10 */
  double lambda_down;     /* 10 */
  double lambda_max;      /* 1e4 */
  double margin_x;        /* centre may leave the grid by this much, default W/2 */
  double margin_y;        /* default H/2 */
  double sigma_min;       /* default 0.3 */
  double sigma_max;       /* default max(W, H) */
} sf_config;

/* Evaluation counters and timings of one sf_fit_batch call. */
typedef struct sf_stats {
  uint64_t n_gradient_evals; /* reference-accounted G-evals (= sum of iterations) */
  uint64_t n_trial_evals;    /* reference-accounted T-evals (trial chi^2 evaluations) */
  uint64_t n_kernel_evals;   /* full evaluations the fused kernel executed */
  double h2d_ms, kernel_ms, d2h_ms, total_ms; /* device-event times (summed over chunks / devices) */
  int32_t n_devices;
  int32_t n_chunks;
  int32_t n_chunks_u16; /* host chunks that crossed PCIe as 16-bit counts (u16 input, or narrowed f32) */
  uint64_t h2d_bytes;   /* bytes copied host -> device (pixels + inits), 0 for device-resident input */
} sf_stats;

/*
 * sf_fit_batch -- replaces fit_batch / per-spot fit_single
 * (SPEC.md:209).  images: [count][H][W] f32 row-major (SpotImage values,
 * model.py:70-93); inits: [count][P] f32 (ShapeParams; estimate_initial output).
 * Pointers may be host (pageable or pinned) or device memory of devices[0];
 * the library detects which.  Host inputs are streamed in chunks over copy/compute
 * streams; with n_devices > 1 the batch is split into contiguous shards, one
 * host thread per device, results written into disjoint slices.
 * out_params: [count][P]; out_alpha/out_beta/out_nchi2: [count]; out_status,
 * out_iters: [count] bytes.  stats may be NULL.  Host f32 chunks whose pixels are all
 * integers in [0, 65535] cross PCIe as u16, narrowed losslessly by the host (results unchanged;
 * SPOTFIT_NARROW).
 */
int sf_fit_batch(const float* images, int32_t width, int32_t height, int64_t count, const float* inits,
                 const sf_config* cfg, float* out_params, float* out_alpha, float* out_beta, float* out_nchi2,
                 uint8_t* out_status, uint8_t* out_iters, const int32_t* devices, int32_t n_devices,
                 sf_stats* stats);

/*
 * sf_fit_batch_u16 -- sf_fit_batch for 16-bit camera counts: images [count][H][W]
 * uint16 (host pointers).  Each chunk is copied as u16 (half the PCIe bytes of
 * f32) and staged as u16 by the fit kernel, which widens each pixel exactly, so results are identical to
 * sf_fit_batch on the same values as float32.
 */
int sf_fit_batch_u16(const uint16_t* images, int32_t width, int32_t height, int64_t count, const float* inits,
                     const sf_config* cfg, float* out_params, float* out_alpha, float* out_beta, float* out_nchi2,
                     uint8_t* out_status, uint8_t* out_iters, const int32_t* devices, int32_t n_devices,
                     sf_stats* stats);

/*
 * sf_fit_batch_device -- the same fit with every pointer in device memory of
 * the current device, launched on `stream` (cudaStream_t, 0 = legacy default),
 * asynchronous.  Used by bench.py for the HBM-resident measurement and by
 * callers that already hold spots on the GPU.  evals_out: device u64[3]
 * accumulating (G-evals, T-evals, kernel evals) or NULL.  Any device-accessible
 * address works, including pinned host memory (device-mapped under UVA): small
 * latency-bound frames read the spots and write the results over PCIe directly
 * (bench.py realtime, zero copy).  sf_estimate_initial_device likewise.
 * Each launch holds one of 256 work-claim counters until it ends (round robin),
 * so at most 256 fit launches may be in flight at once.  A launch captured in a
 * CUDA graph keeps its counter: replays of one graph must not overlap (replays
 * on one stream never do).
 */
int sf_fit_batch_device(const float* d_images, int32_t width, int32_t height, int64_t count, const float* d_inits,
                        const sf_config* cfg, float* d_params, float* d_alpha, float* d_beta, float* d_nchi2,
                        uint8_t* d_status, uint8_t* d_iters, uint64_t* d_evals, void* stream);

/*
 * sf_fit_batch_device_u16 -- sf_fit_batch_device for 16-bit camera counts
 * [count][H][W] uint16 in device-accessible memory: the fit kernel stages the
 * u16 pixels itself and widens them exactly (no f32 copy), so results equal
 * sf_fit_batch_device on the same values as float32.  Extension (not in the
 * reference interface), the device-side twin of sf_fit_batch_u16.
 */
int sf_fit_batch_device_u16(const uint16_t* d_images, int32_t width, int32_t height, int64_t count,
                            const float* d_inits, const sf_config* cfg, float* d_params, float* d_alpha,
                            float* d_beta, float* d_nchi2, uint8_t* d_status, uint8_t* d_iters, uint64_t* d_evals,
                            void* stream);

/*
 * sf_eval_batch_device -- model-level evaluation at given shape parameters
 * (one evaluation per spot, no LM): replaces the spotfit.model call chain
 * profile_and_gradient -> alpha_beta -> chi_squared -> gradient_sums ->
 * coefficient_gradients -> chi_gradient (model.py:180-315) plus the normal
 * matrix.  out: [count] records of sf_eval_record below.
 */
typedef struct sf_eval_record {
  int32_t singular; /* SingularProfile raised (model.py:228-231) */
  float alpha, beta, chi;
  double F, G, FF, FG, denom;
  double dF[4], dFF[4], dFG[4], gamma[4], dalpha[4], dbeta[4];
  double rhs[4];  /* sum r*d_j = -grad_j/2 (model.py:314) */
  double jtj[10]; /* upper-packed normal matrix */
} sf_eval_record;

int sf_eval_batch_device(const float* d_images, int32_t width, int32_t height, int64_t count, int32_t model,
                         const float* d_params, sf_eval_record* d_out, void* stream);

/*
 * spotfit.model function surface (pkg/src/spotfit/model.py:168-315), batched:
 * each entry point replaces one reference function and takes / returns the
 * per-pixel arrays that function does, so a caller can chain them as model.py
 * does (also on f / fgrad arrays that did not come from the profile).  All
 * pointers are device-accessible memory; asynchronous on `stream`.  n = pixels
 * per spot (1..1024); model 3 (x, y, sigma) or 4 (x, y, sigma_x, sigma_y) sets
 * the column count P of fgrad / dmat / gradient arrays.  Bit-identical to the
 * reference (f32 per-pixel ops, numpy float32 exp, numpy-order f64 sums).
 */
/* profile (model.py:168-177) / profile_and_gradient (180-199): params [count][P];
 * f [count][n]; fgrad [count][n][P] or NULL. */
int sf_model_profile_device(const float* d_params, int32_t width, int32_t height, int64_t count, int32_t model,
                            float* d_f, float* d_fgrad, void* stream);
/* alpha_beta (model.py:207-234): f, g [count][n] -> alpha, beta [count] (f32-quantised,
 * NaN where SingularProfile is raised), sums [count][5] = (F, G, FF, FG, denom), singular [count]. */
int sf_model_alpha_beta_device(const float* d_f, const float* d_g, int32_t n, int64_t count, float* d_alpha,
                               float* d_beta, double* d_sums, int32_t* d_singular, void* stream);
/* model_values (237-239), residuals (242-244), chi_squared (247-250): h, r [count][n] or NULL; chi [count]. */
int sf_model_chi_squared_device(const float* d_g, const float* d_f, const float* d_alpha, const float* d_beta,
                                int32_t n, int64_t count, float* d_h, float* d_r, float* d_chi, void* stream);
/* gradient_sums (253-267): gsums [count][4][P] = df, dff, dfg, gamma. */
int sf_model_gradient_sums_device(const float* d_f, const float* d_fgrad, const float* d_g, const double* d_sums,
                                  int32_t n, int32_t model, int64_t count, double* d_gsums, void* stream);
/* coefficient_gradients (270-288): dalpha, dbeta [count][P] (NaN + singular where the reference raises). */
int sf_model_coefficient_gradients_device(const double* d_sums, const double* d_gsums, const float* d_alpha,
                                          const float* d_beta, int32_t n, int32_t model, int64_t count,
                                          double* d_dalpha, double* d_dbeta, int32_t* d_singular, void* stream);
/* chi_gradient (291-315): grad [count][P] f64, dmat [count][n][P] f32 or NULL. */
int sf_model_chi_gradient_device(const float* d_g, const float* d_f, const float* d_fgrad, const float* d_alpha,
                                 const float* d_beta, const double* d_dalpha, const double* d_dbeta, int32_t n,
                                 int32_t model, int64_t count, double* d_grad, float* d_dmat, void* stream);

/*
 * sf_estimate_initial_device -- replaces estimate_initial (SPEC.md:286-290,
 * PAPER.md:212) for a whole batch on the GPU: 3x3 truncated moving average,
 * argmax -> centre, min -> beta, max-beta -> alpha, sigma = sqrt(M/pi) clamped.
 * out_inits: [count][model] f32 (elliptical: sigma_x = sigma_y); out_amps:
 * [count][2] (alpha, beta) or NULL.  Asynchronous on `stream`.
 */
int sf_estimate_initial_device(const float* d_images, int32_t width, int32_t height, int64_t count, int32_t model,
                               double sigma_min, double sigma_max, float* d_inits, float* d_amps, void* stream);

/*
 * sf_simulate_host -- replaces simulate_batch: synthetic
 * spots with a counter-based RNG keyed by (seed, index), so any
 * index can be regenerated alone.  images: [count][H][W]; truth: [count][P+2]
 * (shape params, alpha, beta).  Runs on host threads (threads <= 0: all cores).
 */
typedef struct sf_sim_config {
  int32_t model;      /* 3 or 4 */
  double n_signal;    /* 400 */
  double n_background;/* 40 (per image; beta = n_background / (W*H)) */
  double sigma_lo, sigma_hi; /* [1, 2] */
  double spread;      /* centre std in px; <= 0 means S/20 per axis */
  int32_t noise;      /* 1: N(0, lambda) noise, rounded, clamped at 0 */
  int32_t rounding;   /* 1: round half away from zero */
  uint64_t seed;
} sf_sim_config;

int sf_simulate_host(const sf_sim_config* cfg, int32_t width, int32_t height, int64_t first_index, int64_t count,
                     float* images, float* truth, int32_t threads);

/*
 * sf_simulate_device -- the same generator on the GPU: writes
 * d_images [count][H][W] and d_truth [count][P+2] (or NULL) in device memory on
 * `stream`.  Integer draws are identical to sf_simulate_host; pixels match it
 * except where CUDA's f64 libm and glibc round a .5 boundary differently.
 */
int sf_simulate_device(const sf_sim_config* cfg, int32_t width, int32_t height, int64_t first_index, int64_t count,
                       float* d_images, float* d_truth, void* stream);

/* pinned host allocations (so that callers' buffers DMA directly) */
void* sf_host_alloc(size_t bytes);
void sf_host_free(void* p);

/*
 * sf_lane_geometry -- diagnostic: how a W x H spot maps onto chain lanes
 * (numpy's pairwise-sum tree).  Writes slots (1..16) and, per
 * lane (8*slots entries, up to 128), the chain-pixel count nc, tail-pixel count
 * nt, first chain pixel base and first tail pixel tbase.  Host-only.
 */
int sf_lane_geometry(int32_t width, int32_t height, int32_t* slots, int32_t* ppl, int16_t* nc, int16_t* nt,
                     int16_t* base, int16_t* tbase);

/*
 * sf_debug_npexp_device -- diagnostic: the kernel's float32 exp (numpy's
 * simd_exp_f32 restated; model.py:177,193 call np.exp) on a device array.
 * variant 0: production (fast-path IEEE division); 1: CUDA __fdiv_rn;
 * 2: the packed f32x2 form used by the fit kernel's chain loops.
 */
int sf_debug_npexp_device(const float* d_x, float* d_y, int64_t n, int32_t variant, void* stream);

/*
 * sf_debug_ddiv_device -- diagnostic: the kernel's shared-divisor f64 division
 * (the LDL^T pivots and the alpha/beta denominator of SPEC.md:189-197 and
 * model.py:226-233, 281-287) on device arrays; must equal IEEE a / b.
 */
int sf_debug_ddiv_device(const double* d_a, const double* d_b, double* d_out, int64_t n, void* stream);

/*
 * sf_debug_tame_div_device -- diagnostic: counts (into *d_mismatches, device u64, accumulated)
 * the integers s in [0, 9 * 2^20] and window counts c in {1, 2, 3, 4, 6, 9} for which the
 * initializer's integer-path division (sf_init_core.cuh:tame_div) differs from IEEE s / c.
 */
int sf_debug_tame_div_device(uint64_t* d_mismatches, void* stream);

/*
 * ParamsCSV / truth CSV (cmd_fit writes, cmd_assess reads, SPEC.md:536-549;
 * round trip SPEC.md:554).  Host-only, multi-threaded (threads <= 0: all hardware threads).
 * The reference CLI is SPEC-only (no code under /root/reference); its Python restatement in
 * paper_2106_02045_b200/io_formats.py (fmt32: numpy's format_float_positional(unique=True,
 * trim='-')) is the checker.  Floats are rendered as the shortest decimal that round-trips the
 * float32 value, positional notation.  Every row is `index,<cells>` with index = first_index + r.
 */
enum sf_csv_kind {
  SF_CSV_F32 = 0,   /* float32, shortest round-trip positional */
  SF_CSV_U8 = 1,    /* uint8 as a decimal integer (iterations) */
  SF_CSV_STOP = 2,  /* status byte & 7 as the StopReason name (MaxError .. MaxIterations) */
  SF_CSV_FLAGS = 3, /* status byte & 0xf8 as a decimal integer (0x40 invalid, 0x80 no-improvement) */
  SF_CSV_SKIP = 4   /* reader only: ignore the column */
};
typedef struct sf_csv_col {
  int32_t kind;   /* sf_csv_kind */
  void* data;     /* element r of the column is data[r * stride] */
  int64_t stride; /* in elements */
} sf_csv_col;

/* write `header` + '\n' then `rows` rows; returns 0 or -1 (message: sf_csv_last_error()) */
int sf_csv_write(const char* path, const char* header, int64_t first_index, int64_t rows, int ncols,
                 const sf_csv_col* cols, int threads);
/* parse the rows after the header line: *rows_out = row count; capacity < 0 counts only; index may be
 * NULL; a row whose cells do not match `cols` exactly fails with its row number */
int sf_csv_read(const char* path, int64_t* rows_out, int64_t* index, int ncols, const sf_csv_col* cols,
                int64_t capacity, int threads);
/* diagnostic: the float32 rendering alone, one value per line into out (capacity bytes) */
int sf_format_f32(const float* values, int64_t count, char* out, int64_t capacity, int64_t* out_len);
const char* sf_csv_last_error(void);

/*
 * sf_shard_range -- the contiguous spot range [*lo, *hi) of shard `shard` of `n_shards` (the split
 * sf_fit_batch applies over its devices and a torchrun rank applies over the job): independent,
 * order-preserving shards, sizes differing by at most one.  Host-only.
 */
int sf_shard_range(int64_t count, int32_t shard, int32_t n_shards, int64_t* lo, int64_t* hi);

/*
 * sf_debug_narrow_u16 -- diagnostic: the host pipeline's lossless narrowing of f32 pixel chunks for
 * the PCIe leg (sf_fit_batch sends a pageable f32 chunk as u16 when every pixel is an integer in
 * [0, 65535] with a clear sign bit; SPOTFIT_NARROW).  Returns 1 if all n values narrowed (dst
 * holds them), 0 if some value did not, -1 on bad arguments.  Host-only.
 */
int sf_debug_narrow_u16(const float* src, int64_t n, uint16_t* dst, int32_t threads);

/*
 * sf_debug_par_copy -- diagnostic: the host pipeline's staging copy of pageable input (threads,
 * streaming stores into a 32-byte aligned destination).  Returns 0, or -1 on bad arguments.  Host-only.
 */
int sf_debug_par_copy(void* dst, const void* src, int64_t bytes, int32_t threads);

int sf_device_count(void);
const char* sf_last_error(void);
int sf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SPOTFIT_H */
