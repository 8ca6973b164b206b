// sf_model.cu -- the spotfit.model function surface on the GPU
// (pkg/src/spotfit/model.py:154-315), one batched kernel per reference function,
// taking and returning the per-pixel arrays the reference functions do (f,
// fgrad, h, r, dmat) so that callers can chain them exactly as model.py does --
// including on arrays that did not come from profile().  The fit kernel fuses
// this whole chain; these kernels are the model-level API (include/spotfit.h:
// sf_model_*), bit-identical to the reference:
//   * per-pixel values: individually rounded f32 ops in model.py order
//     (-fmad=false, explicit __f*_rn), numpy's float32 exp (sf_device.cuh:npexp);
//   * sums: ndarray.sum(dtype=float64) of f32 addends in numpy's pairwise order
//     (SURVEY App. B.3), one thread per quantity over the addends staged in
//     shared memory;
//   * scalar f64 formulas in model.py's association order.
#include <cstdint>

#include "sf_device.cuh"
#include "sf_launch.h"

namespace sf {

namespace {

// numpy pairwise_sum (numpy/_core/src/umath/loops_utils.h.src) of a float32 array
// cast to float64, for n <= 1024: leaves of <= 128 with 8 strided accumulators,
// split n2 = n/2 - (n/2)%8.  D bounds the recursion depth (4 suffices for n <= 1024).
template <int D>
__device__ double pw_t(const float* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, (double)a[i]);
    return res;
  }
  if (D == 0 || n <= 128) {
    double r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = (double)a[k];
    int i;
    for (i = 8; i < n - (n % 8); i += 8)
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], (double)a[i + k]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, (double)a[i]);
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return __dadd_rn(pw_t<(D > 0 ? D - 1 : 0)>(a, n2), pw_t<(D > 0 ? D - 1 : 0)>(a + n2, n - n2));
}

// x.sum(dtype=np.float64) == 0.0 + pairwise(x)
__device__ __forceinline__ double np_sum(const float* a, int n) { return __dadd_rn(0.0, pw_t<4>(a, n)); }

constexpr int kTPB = 128;

// profile (model.py:168-177) and profile_and_gradient (180-199); elliptical: SURVEY App. B.5.
template <int P>
__global__ void profile_kernel(const float* __restrict__ params, int W, int H, int64_t count, float* __restrict__ f,
                               float* __restrict__ fgrad) {
  const int N = W * H;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * N) return;
  const int64_t spot = t / N;
  const int i = (int)(t - spot * N);
  float pe[P];
#pragma unroll
  for (int k = 0; k < P; ++k) pe[k] = params[spot * P + k];
  const float ix = __frcp_rn(pe[2]);  // np.float32(1.0) / np.float32(sigma), IEEE (model.py:162)
  const float iy = P == 4 ? __frcp_rn(pe[P - 1]) : ix;
  float fv, fg[P];
  pixel_profile<P>(make_float2((float)(i % W), (float)(i / W)), pe, ix, iy, true, fv, fg);
  f[t] = fv;
  if (fgrad != nullptr) {
#pragma unroll
    for (int k = 0; k < P; ++k) fgrad[t * P + k] = fg[k];
  }
}

// alpha_beta (model.py:207-234): F, G, FF, FG, denom; SingularProfile guard; Eq. (6).
// out: alpha, beta (f32-quantised, Amplitudes model.py:118-127; NaN when singular),
// sums[count][5] = (F, G, FF, FG, denom), singular[count].
__global__ void alpha_beta_kernel(const float* __restrict__ f, const float* __restrict__ g, int N, int64_t count,
                                  float* __restrict__ alpha, float* __restrict__ beta, double* __restrict__ sums,
                                  int32_t* __restrict__ singular) {
  extern __shared__ float sm[];  // [4][N]: f, g, f*f, f*g
  const int64_t spot = blockIdx.x;
  const float* fs = f + spot * N;
  const float* gs = g + spot * N;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const float fv = fs[i], gv = gs[i];
    sm[i] = fv;
    sm[N + i] = gv;
    sm[2 * N + i] = __fmul_rn(fv, fv);
    sm[3 * N + i] = __fmul_rn(fv, gv);
  }
  __syncthreads();
  __shared__ double s[4];
  if (threadIdx.x < 4) s[threadIdx.x] = np_sum(sm + threadIdx.x * N, N);
  __syncthreads();
  if (threadIdx.x == 0) {
    const double n = (double)N, F = s[0], G = s[1], FF = s[2], FG = s[3];
    const double denom = __dsub_rn(__dmul_rn(n, FF), __dmul_rn(F, F));
    const bool sing = denom <= __dmul_rn(__dmul_rn(1e-12, n), FF);
    double* o = sums + spot * 5;
    o[0] = F;
    o[1] = G;
    o[2] = FF;
    o[3] = FG;
    o[4] = denom;
    singular[spot] = sing ? 1 : 0;
    const float nan = __int_as_float(0x7fc00000);
    alpha[spot] = sing ? nan : (float)(__dsub_rn(__dmul_rn(n, FG), __dmul_rn(F, G)) / denom);
    beta[spot] = sing ? nan : (float)(__dsub_rn(__dmul_rn(G, FF), __dmul_rn(F, FG)) / denom);
  }
}

// model_values (model.py:237-239), residuals (242-244), chi_squared (247-250).
// h, r: [count][N] or NULL; chi: [count] f32.
__global__ void chi_kernel(const float* __restrict__ g, const float* __restrict__ f, const float* __restrict__ alpha,
                           const float* __restrict__ beta, int N, int64_t count, float* __restrict__ h,
                           float* __restrict__ r, float* __restrict__ chi) {
  extern __shared__ float sm[];  // [N]: r*r
  const int64_t spot = blockIdx.x;
  const float a32 = alpha[spot], b32 = beta[spot];
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const int64_t k = spot * N + i;
    const float hv = __fadd_rn(__fmul_rn(a32, f[k]), b32);
    const float rv = __fsub_rn(g[k], hv);
    if (h != nullptr) h[k] = hv;
    if (r != nullptr) r[k] = rv;
    sm[i] = __fmul_rn(rv, rv);
  }
  __syncthreads();
  if (threadIdx.x == 0) chi[spot] = (float)np_sum(sm, N);
}

// gradient_sums (model.py:253-267): out[count][4][P] = df, dff, dfg, gamma.
template <int P>
__global__ void gradient_sums_kernel(const float* __restrict__ f, const float* __restrict__ fgrad,
                                     const float* __restrict__ g, const double* __restrict__ sums, int N,
                                     int64_t count, double* __restrict__ out) {
  extern __shared__ float sm[];  // [3P][N]: fgrad_j | f*fgrad_j | g*fgrad_j
  const int64_t spot = blockIdx.x;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const int64_t k = spot * N + i;
    const float fv = f[k], gv = g[k];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const float c = fgrad[k * P + j];
      sm[j * N + i] = c;
      sm[(P + j) * N + i] = __fmul_rn(fv, c);
      sm[(2 * P + j) * N + i] = __fmul_rn(gv, c);
    }
  }
  __syncthreads();
  __shared__ double s[3 * P];
  if (threadIdx.x < 3 * P) s[threadIdx.x] = np_sum(sm + threadIdx.x * N, N);
  __syncthreads();
  if (threadIdx.x < P) {
    const int j = threadIdx.x;
    const double n = (double)N, F = sums[spot * 5 + 0];
    const double df = s[j], dff = __dmul_rn(2.0, s[P + j]), dfg = s[2 * P + j];
    double* o = out + spot * 4 * P;
    o[j] = df;
    o[P + j] = dff;
    o[2 * P + j] = dfg;
    o[3 * P + j] = __dsub_rn(__dmul_rn(n, dff), __dmul_rn(__dmul_rn(2.0, F), df));  // n dff - (2 F) df
  }
}

// coefficient_gradients (model.py:270-288), Eq. (8): one thread per spot.
template <int P>
__global__ void coefficient_gradients_kernel(const double* __restrict__ sums, const double* __restrict__ gsums,
                                             const float* __restrict__ alpha, const float* __restrict__ beta, int N,
                                             int64_t count, double* __restrict__ dalpha, double* __restrict__ dbeta,
                                             int32_t* __restrict__ singular) {
  const int64_t spot = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (spot >= count) return;
  const double* s = sums + spot * 5;
  const double n = (double)N, F = s[0], G = s[1], FF = s[2], FG = s[3], D = s[4];
  const bool sing = D <= __dmul_rn(__dmul_rn(1e-12, n), FF);
  singular[spot] = sing ? 1 : 0;
  const double a = (double)alpha[spot], b = (double)beta[spot];
  const double* gs = gsums + spot * 4 * P;
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const double df = gs[j], dff = gs[P + j], dfg = gs[2 * P + j], gam = gs[3 * P + j];
    const double na = __dsub_rn(__dsub_rn(__dmul_rn(n, dfg), __dmul_rn(G, df)), __dmul_rn(a, gam));
    const double nb = __dsub_rn(__dsub_rn(__dsub_rn(__dmul_rn(G, dff), __dmul_rn(FG, df)), __dmul_rn(F, dfg)),
                                __dmul_rn(b, gam));
    dalpha[spot * P + j] = sing ? __longlong_as_double(0x7ff8000000000000ll) : na / D;
    dbeta[spot * P + j] = sing ? __longlong_as_double(0x7ff8000000000000ll) : nb / D;
  }
}

// chi_gradient (model.py:291-315), Eq. (9): d_ij = (f32(dalpha_j) f_i + alpha fgrad_ij) + f32(dbeta_j),
// grad_j = -2 sum r_i d_ij.  grad: [count][P] f64; dmat: [count][N][P] f32 or NULL.
template <int P>
__global__ void chi_gradient_kernel(const float* __restrict__ g, const float* __restrict__ f,
                                    const float* __restrict__ fgrad, const float* __restrict__ alpha,
                                    const float* __restrict__ beta, const double* __restrict__ dalpha,
                                    const double* __restrict__ dbeta, int N, int64_t count,
                                    double* __restrict__ grad, float* __restrict__ dmat) {
  extern __shared__ float sm[];  // [P][N]: r * d_j
  const int64_t spot = blockIdx.x;
  const float a32 = alpha[spot], b32 = beta[spot];
  float da[P], db[P];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    da[j] = (float)dalpha[spot * P + j];
    db[j] = (float)dbeta[spot * P + j];
  }
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    const int64_t k = spot * N + i;
    const float fv = f[k];
    const float rv = __fsub_rn(g[k], __fadd_rn(__fmul_rn(a32, fv), b32));
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const float d = __fadd_rn(__fadd_rn(__fmul_rn(da[j], fv), __fmul_rn(a32, fgrad[k * P + j])), db[j]);
      if (dmat != nullptr) dmat[k * P + j] = d;
      sm[j * N + i] = __fmul_rn(rv, d);
    }
  }
  __syncthreads();
  if (threadIdx.x < P) grad[spot * P + threadIdx.x] = __dmul_rn(-2.0, np_sum(sm + threadIdx.x * N, N));
}

}  // namespace

cudaError_t launch_model_profile(const float* params, int W, int H, int64_t count, int P, float* f, float* fgrad,
                                 cudaStream_t st) {
  const int64_t n = count * W * H;
  if (n <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((n + kTPB - 1) / kTPB);
  if (P == 4)
    profile_kernel<4><<<blocks, kTPB, 0, st>>>(params, W, H, count, f, fgrad);
  else
    profile_kernel<3><<<blocks, kTPB, 0, st>>>(params, W, H, count, f, fgrad);
  return cudaGetLastError();
}

cudaError_t launch_model_alpha_beta(const float* f, const float* g, int N, int64_t count, float* alpha, float* beta,
                                    double* sums, int32_t* singular, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  alpha_beta_kernel<<<(unsigned)count, kTPB, 4 * N * sizeof(float), st>>>(f, g, N, count, alpha, beta, sums,
                                                                          singular);
  return cudaGetLastError();
}

cudaError_t launch_model_chi(const float* g, const float* f, const float* alpha, const float* beta, int N,
                             int64_t count, float* h, float* r, float* chi, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  chi_kernel<<<(unsigned)count, kTPB, N * sizeof(float), st>>>(g, f, alpha, beta, N, count, h, r, chi);
  return cudaGetLastError();
}

cudaError_t launch_model_gradient_sums(const float* f, const float* fgrad, const float* g, const double* sums, int N,
                                       int P, int64_t count, double* out, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const size_t smem = 3 * P * N * sizeof(float);
  if (P == 4) {
    cudaError_t e = cudaFuncSetAttribute(gradient_sums_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    gradient_sums_kernel<4><<<(unsigned)count, kTPB, smem, st>>>(f, fgrad, g, sums, N, count, out);
  } else {
    gradient_sums_kernel<3><<<(unsigned)count, kTPB, smem, st>>>(f, fgrad, g, sums, N, count, out);
  }
  return cudaGetLastError();
}

cudaError_t launch_model_coefficient_gradients(const double* sums, const double* gsums, const float* alpha,
                                               const float* beta, int N, int P, int64_t count, double* dalpha,
                                               double* dbeta, int32_t* singular, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((count + kTPB - 1) / kTPB);
  if (P == 4)
    coefficient_gradients_kernel<4><<<blocks, kTPB, 0, st>>>(sums, gsums, alpha, beta, N, count, dalpha, dbeta,
                                                             singular);
  else
    coefficient_gradients_kernel<3><<<blocks, kTPB, 0, st>>>(sums, gsums, alpha, beta, N, count, dalpha, dbeta,
                                                             singular);
  return cudaGetLastError();
}

cudaError_t launch_model_chi_gradient(const float* g, const float* f, const float* fgrad, const float* alpha,
                                      const float* beta, const double* dalpha, const double* dbeta, int N, int P,
                                      int64_t count, double* grad, float* dmat, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const size_t smem = P * N * sizeof(float);
  if (P == 4)
    chi_gradient_kernel<4><<<(unsigned)count, kTPB, smem, st>>>(g, f, fgrad, alpha, beta, dalpha, dbeta, N, count,
                                                                grad, dmat);
  else
    chi_gradient_kernel<3><<<(unsigned)count, kTPB, smem, st>>>(g, f, fgrad, alpha, beta, dalpha, dbeta, N, count,
                                                                grad, dmat);
  return cudaGetLastError();
}

}  // namespace sf
