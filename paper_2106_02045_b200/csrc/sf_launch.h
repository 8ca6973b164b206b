// sf_launch.h -- internal (C++) interface between the C-ABI layer and the
// template instantiation units (sf_inst.cu compiled once per (P, SLOTS)).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "sf_fit_kernel.cuh"

namespace sf {

struct LaunchFit {
  const float* images;
  const uint16_t* images16 = nullptr;  // non-null: 16-bit pixels (fit_kernel<..., uint16_t>), images unused
  const float* inits;
  int64_t count;
  Geom geom;
  Cfg cfg;
  FitOut out;
  cudaStream_t stream;
  int sm_count;
};

struct LaunchEval {
  const float* images;
  const float* params;
  int64_t count;
  Geom geom;
  sf_eval_record* out;
  cudaStream_t stream;
};

// Each returns the number of CTAs launched; a CUDA error is reported through *err.
#define SF_DECLARE_UNIT(P, S)                                          \
  int launch_fit_P##P##_S##S(const LaunchFit& a, cudaError_t* err);   \
  int launch_eval_P##P##_S##S(const LaunchEval& a, cudaError_t* err);
SF_DECLARE_UNIT(3, 1)
SF_DECLARE_UNIT(3, 2)
SF_DECLARE_UNIT(3, 4)
SF_DECLARE_UNIT(3, 8)
SF_DECLARE_UNIT(3, 16)
SF_DECLARE_UNIT(4, 1)
SF_DECLARE_UNIT(4, 2)
SF_DECLARE_UNIT(4, 4)
SF_DECLARE_UNIT(4, 8)
SF_DECLARE_UNIT(4, 16)
#undef SF_DECLARE_UNIT
// explicit 5-parameter model (fit only)
int launch_fit_P5_S1(const LaunchFit& a, cudaError_t* err);
int launch_fit_P5_S2(const LaunchFit& a, cudaError_t* err);
int launch_fit_P5_S4(const LaunchFit& a, cudaError_t* err);
int launch_fit_P5_S8(const LaunchFit& a, cudaError_t* err);
int launch_fit_P5_S16(const LaunchFit& a, cudaError_t* err);

// initializer kernel launchers (sf_init.cu): float pixels, 16-bit counts
cudaError_t launch_estimate_initial(const float* images, int W, int H, int64_t count, int P, double sigma_min,
                                    double sigma_max, float* inits, float* amps, cudaStream_t stream);
cudaError_t launch_estimate_initial_u16(const uint16_t* images, int W, int H, int64_t count, int P,
                                        double sigma_min, double sigma_max, float* inits, float* amps,
                                        cudaStream_t stream);
// Batches up to this many spots with inits == NULL use the fit kernel's fused initializer (one
// kernel, the latency path); larger ones run the standalone initializer in front of the fit on the
// same stream, which keeps the fit kernel's instruction working set small (the fused path costs
// ~20% of fit time at 15x15 in i-cache misses: profiles/r02_fused_init.txt).
constexpr int64_t kFusedInitMaxSpots = 16384;

// spotfit.model function surface (sf_model.cu)
cudaError_t launch_model_profile(const float* params, int W, int H, int64_t count, int P, float* f, float* fgrad,
                                 cudaStream_t st);
cudaError_t launch_model_alpha_beta(const float* f, const float* g, int N, int64_t count, float* alpha, float* beta,
                                    double* sums, int32_t* singular, cudaStream_t st);
cudaError_t launch_model_chi(const float* g, const float* f, const float* alpha, const float* beta, int N,
                             int64_t count, float* h, float* r, float* chi, cudaStream_t st);
cudaError_t launch_model_gradient_sums(const float* f, const float* fgrad, const float* g, const double* sums, int N,
                                       int P, int64_t count, double* out, cudaStream_t st);
cudaError_t launch_model_coefficient_gradients(const double* sums, const double* gsums, const float* alpha,
                                               const float* beta, int N, int P, int64_t count, double* dalpha,
                                               double* dbeta, int32_t* singular, cudaStream_t st);
cudaError_t launch_model_chi_gradient(const float* g, const float* f, const float* fgrad, const float* alpha,
                                      const float* beta, const double* dalpha, const double* dbeta, int N, int P,
                                      int64_t count, double* grad, float* dmat, cudaStream_t st);

// lossless f32 -> u16 narrowing of a host chunk for the PCIe leg (sf_host_narrow.cpp): true iff every
// value is an integer in [0, 65535] with a clear sign bit
bool par_narrow_u16(uint16_t* dst, const float* src, size_t n, int threads);
// memcpy over `threads` threads, streaming stores into an aligned destination (sf_host_narrow.cpp)
void par_copy(void* dst, const void* src, size_t bytes, int threads);

// device simulator (sf_sim.cu)
cudaError_t launch_simulate(const sf_sim_config& c, int W, int H, int64_t first, int64_t count, float* images,
                            float* truth, cudaStream_t stream);


// shared-divisor f64 division check (sf_init.cu)
cudaError_t launch_ddiv(const double* a, const double* b, double* out, int64_t n, cudaStream_t stream);

// initializer integer-path division check (sf_init.cu)
cudaError_t launch_tame_div(unsigned long long* mismatches, cudaStream_t stream);

// exhaustive-check helper (sf_init.cu)
cudaError_t launch_npexp(const float* x, float* y, int64_t n, int variant, cudaStream_t stream);

}  // namespace sf
