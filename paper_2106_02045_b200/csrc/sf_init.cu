// sf_init.cu -- GPU initializer: estimate_initial for a whole batch
// (SURVEY 8f item 1).  One warp per spot.
//
// Pinned arithmetic (oracle/initializer.py restates it):
//   smoothed_i = f32( sum_f64(in-bounds 3x3 neighbours, row-major order) / count )
//   (x, y)     = coordinates of the first maximum of smoothed (row-major ties)
//   beta       = min smoothed;  alpha = f32(f64(max) - f64(beta))
//   M          = #{ i : f64(g_i) > f64(alpha) * exp(-0.5) + f64(beta) }  (original pixels)
//   sigma      = f32( clamp( sqrt(M / pi), sigma_min, sigma_max ) )
#include <cfloat>
#include <climits>

#include "sf_launch.h"

namespace sf {

namespace {
constexpr double kExpMinusHalf = 0x1.368b2fc6f960ap-1;  // exp(-0.5), correctly rounded
constexpr double kPi = 3.141592653589793115997963468544185161590576171875;

// One warp per spot; the spot is staged in shared memory with coalesced loads (the 3x3 means
// read it 9x), and pixel coordinates come from the exact float reciprocal (idx + 0.5) / W
// instead of integer division.  Arithmetic exactly as pinned above.
constexpr int kInitWarps = 8;
__global__ void __launch_bounds__(32 * kInitWarps) init_kernel(const float* __restrict__ images, int W, int H,
                                                              int64_t count, int P, double smin, double smax,
                                                              float* __restrict__ inits, float* __restrict__ amps) {
  extern __shared__ float init_smem[];  // [kInitWarps][N]
  const int warp = threadIdx.x >> 5;
  const int64_t spot = (int64_t)blockIdx.x * kInitWarps + warp;
  const int lane = threadIdx.x & 31;
  if (spot >= count) return;
  const int N = W * H;
  float* sg = init_smem + warp * N;
  const float* g = images + spot * (int64_t)N;
  for (int i = lane; i < N; i += 32) sg[i] = __ldg(g + i);
  __syncwarp();
  const float Wf = (float)W, invW = 1.0f / Wf;
  float best = -INFINITY, lo = INFINITY;
  int bidx = INT_MAX;
  for (int i = lane; i < N; i += 32) {
    // y = floor((i + 0.5) / W) exactly (small integers, never a tie), x = i - y W
    const int y = (int)(((float)i + 0.5f) * invW);
    const int x = i - y * W;
    double s = 0.0;
    int cnt = 0;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
      const int yy = y + dy;
      const bool vy = yy >= 0 && yy < H;
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int xx = x + dx;
        const bool v = vy && xx >= 0 && xx < W;
        const float val = v ? sg[yy * W + xx] : 0.0f;
        if (v) {
          s = s + (double)val;
          ++cnt;
        }
      }
    }
    const float v = (float)(s / (double)cnt);
    if (v > best || (v == best && i < bidx)) {
      best = v;
      bidx = i;
    }
    lo = fminf(lo, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ob > best || (ob == best && oi < bidx)) {
      best = ob;
      bidx = oi;
    }
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
  }
  if (bidx == INT_MAX) bidx = 0;
  const float alpha = (float)((double)best - (double)lo);
  const double thr = (double)alpha * kExpMinusHalf + (double)lo;
  int m = 0;
  for (int i = lane; i < N; i += 32) m += ((double)sg[i] > thr) ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m += __shfl_xor_sync(0xffffffffu, m, o);
  double sgm = sqrt((double)m / kPi);
  sgm = sgm < smin ? smin : (sgm > smax ? smax : sgm);
  if (lane == 0) {
    float* o = inits + spot * P;
    o[0] = (float)(bidx % W);
    o[1] = (float)(bidx / W);
    o[2] = (float)sgm;
    if (P == 4) o[3] = (float)sgm;
    if (amps != nullptr) {
      amps[2 * spot] = alpha;
      amps[2 * spot + 1] = lo;
    }
  }
}
}  // namespace

cudaError_t launch_estimate_initial(const float* images, int W, int H, int64_t count, int P, double sigma_min,
                                    double sigma_max, float* inits, float* amps, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const int64_t blocks = (count + kInitWarps - 1) / kInitWarps;
  const size_t smem = (size_t)kInitWarps * W * H * sizeof(float);  // <= 32 KB (N <= 1024)
  init_kernel<<<(unsigned)blocks, 32 * kInitWarps, smem, stream>>>(images, W, H, count, P, sigma_min, sigma_max,
                                                                   inits, amps);
  return cudaGetLastError();
}

// Exhaustive-check helper: numpy exp on the device (variant 0: production
// scalar npexp, 1: the same with CUDA's IEEE __fdiv_rn, 2: the packed f32x2
// npexp2 of the chain loops, on element pairs (x[2i], x[2i+1])).
__global__ void npexp_kernel(const float* __restrict__ x, float* __restrict__ y, int64_t n, int variant,
                             unsigned long long nz2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (variant == 2) {
    const int64_t a = 2 * i;
    if (a < n) {
      const float xa = x[a], xb = a + 1 < n ? x[a + 1] : 0.0f;
      float ya, yb;
      up2(npexp2(pk2(xa, xb), f2{nz2}), ya, yb);
      y[a] = ya;
      if (a + 1 < n) y[a + 1] = yb;
    }
    return;
  }
  if (i < n) y[i] = variant == 0 ? npexp(x[i]) : npexp_ieee_div(x[i]);
}

// Shared-divisor f64 division check: out = ddiv_with(a, b, ddiv_rcp(b)) (should equal a / b).
__global__ void ddiv_kernel(const double* __restrict__ a, const double* __restrict__ b, double* __restrict__ out,
                            int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {  // both forms: ddiv_with, and ddiv_fast with the solve's fall-back to a / b
    bool ok = true;
    const double q = ddiv_fast(a[i], b[i], ddiv_rcp(b[i]), ok);
    const double w = ddiv_with(a[i], b[i], ddiv_rcp(b[i]));
    const double f = ok ? q : a[i] / b[i];
    // report ddiv_with; flag a disagreement between the two forms with a NaN of a distinct payload
    out[i] = (__double_as_longlong(w) == __double_as_longlong(f) || (w != w && f != f)) ? w
                                                                                    : __longlong_as_double(0x7ff8dead0000beefull);
  }
}

cudaError_t launch_ddiv(const double* a, const double* b, double* out, int64_t n, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  ddiv_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(a, b, out, n);
  return cudaGetLastError();
}

cudaError_t launch_npexp(const float* x, float* y, int64_t n, int variant, cudaStream_t stream) {
  if (n <= 0) return cudaSuccess;
  const int64_t threads = variant == 2 ? (n + 1) / 2 : n;
  npexp_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, stream>>>(x, y, n, variant, 0x8000000080000000ull);
  return cudaGetLastError();
}

}  // namespace sf
