// sf_init_core.cuh -- the initializer arithmetic (estimate_initial, SPEC.md:276-305,
// PAPER.md:212), shared by the standalone initializer kernel (sf_init.cu) and
// the fit kernel's fused initializer (sf_fit_kernel.cuh, inits == NULL).
//
// Pinned arithmetic (oracle/initializer.py restates it):
//   smoothed_i = f32( sum_f64(in-bounds 3x3 neighbours, row-major order) / count )
//   (x, y)     = coordinates of the first maximum of smoothed (row-major scan with a strict
//                ">" from smoothed_0: NaN never wins, and a NaN smoothed_0 wins for good)
//   beta       = min smoothed (NaN if any smoothed value is NaN, as numpy's min)
//   alpha      = f32(f64(max) - f64(beta))
//   M          = #{ i : f64(g_i) > f64(alpha) * exp(-0.5) + f64(beta) }  (original pixels)
//   sigma      = f32( clamp( sqrt(M / pi), sigma_min, sigma_max ) )
#pragma once
#include <climits>
#include <cstdint>

namespace sf {

constexpr double kExpMinusHalf = 0x1.368b2fc6f960ap-1;  // exp(-0.5), correctly rounded
constexpr double kPi = 3.141592653589793115997963468544185161590576171875;

// A lane's partial scan: first maximum (best, idx), minimum, NaN flags
// (bit 0: some smoothed value is NaN; bit 1: smoothed_0 is NaN).
struct InitPart {
  float best, lo;
  int idx, nan;
};

__device__ __forceinline__ void init_part_reset(InitPart& p) {
  p.best = -__int_as_float(0x7f800000);
  p.lo = __int_as_float(0x7f800000);
  p.idx = INT_MAX;
  p.nan = 0;
}

// Order-independent merge: the surviving maximum is the non-NaN maximum with the
// smallest index, which is what the row-major strict-">" scan finds unless
// smoothed_0 is NaN (resolved in init_finish).
__device__ __forceinline__ void init_part_merge(InitPart& a, float best, int idx, float lo, int nan) {
  if (best > a.best || (best == a.best && idx < a.idx)) {
    a.best = best;
    a.idx = idx;
  }
  a.lo = fminf(a.lo, lo);
  a.nan |= nan;
}

// Pixel value i of a staged spot (float or 16-bit counts, widened exactly).
template <typename PX>
__device__ __forceinline__ float init_px(const PX* st, int i) {
  return (float)st[i];
}

// smoothed_i: the truncated 3x3 mean, summed in f64 in row-major neighbour order.
// y = floor((i + 0.5) / W) from the float reciprocal (small integers, never a tie).
template <typename PX>
__device__ __forceinline__ float init_smoothed(const PX* st, int W, int H, float invW, int i) {
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
      if (vy && xx >= 0 && xx < W) {
        s = __dadd_rn(s, (double)init_px(st, yy * W + xx));
        ++cnt;
      }
    }
  }
  return (float)(s / (double)cnt);
}

// Scan pixels i = first, first + stride, ... < N of a staged spot into p.
template <typename PX>
__device__ __forceinline__ void init_scan(const PX* st, int W, int H, int N, float invW, int first, int stride,
                                          InitPart& p) {
#pragma unroll 1
  for (int i = first; i < N; i += stride) {
    const float v = init_smoothed(st, W, H, invW, i);
    if (v != v) p.nan |= i == 0 ? 3 : 1;
    init_part_merge(p, v, i, v, 0);
  }
}

// The merged scan -> (idx, alpha, beta) with numpy's NaN semantics, and the M threshold.
__device__ __forceinline__ void init_finish(const InitPart& p, int& idx, float& alpha, float& beta, double& thr) {
  float best = p.best;
  idx = p.idx;
  if ((p.nan & 2) || idx == INT_MAX) {  // smoothed_0 is NaN: the scan never moves off it
    best = __int_as_float(0x7fc00000);
    idx = 0;
  }
  beta = (p.nan & 1) ? __int_as_float(0x7fc00000) : p.lo;
  alpha = (float)__dadd_rn((double)best, -(double)beta);
  thr = __dadd_rn(__dmul_rn((double)alpha, kExpMinusHalf), (double)beta);
}

// M over pixels i = first, first + stride, ... < N.
template <typename PX>
__device__ __forceinline__ int init_count(const PX* st, int N, double thr, int first, int stride) {
  int m = 0;
#pragma unroll 1
  for (int i = first; i < N; i += stride) m += ((double)init_px(st, i) > thr) ? 1 : 0;
  return m;
}

// sigma = f32(clamp(sqrt(M / pi), smin, smax)).
__device__ __forceinline__ float init_sigma(int m, double smin, double smax) {
  double sg = sqrt((double)m / kPi);
  sg = sg < smin ? smin : (sg > smax ? smax : sg);
  return (float)sg;
}

}  // namespace sf
