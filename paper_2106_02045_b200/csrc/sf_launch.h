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

// initializer kernel launcher (sf_init.cu)
cudaError_t launch_estimate_initial(const float* images, int W, int H, int64_t count, int P, double sigma_min,
                                    double sigma_max, float* inits, float* amps, cudaStream_t stream);

// device simulator (sf_sim.cu)
cudaError_t launch_simulate(const sf_sim_config& c, int W, int H, int64_t first, int64_t count, float* images,
                            float* truth, cudaStream_t stream);


// shared-divisor f64 division check (sf_init.cu)
cudaError_t launch_ddiv(const double* a, const double* b, double* out, int64_t n, cudaStream_t stream);

// exhaustive-check helper (sf_init.cu)
cudaError_t launch_npexp(const float* x, float* y, int64_t n, int variant, cudaStream_t stream);

}  // namespace sf
