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
//
// A lane scans some pixels into an InitScan; lanes merge with an order-
// independent max / min / or, so any pixel-to-lane mapping gives the row-major
// scan's answer.
#pragma once
#include <climits>
#include <cstdint>

namespace sf {

constexpr double kExpMinusHalf = 0x1.368b2fc6f960ap-1;  // exp(-0.5), correctly rounded
constexpr double kPi = 3.141592653589793115997963468544185161590576171875;

// (value, index) -> a 64-bit key whose maximum is the first maximum: the value's bits mapped
// to an order-preserving unsigned integer (smoothed values are never -0.0: their sums start at
// +0.0), then ~index so that ties go to the first pixel.  0 is below every key.
__device__ __forceinline__ unsigned long long scan_key(float v, int idx) {
  const unsigned u = __float_as_uint(v);
  const unsigned o = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
  return ((unsigned long long)o << 32) | (unsigned)(~idx);
}
__device__ __forceinline__ unsigned long long key_max(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}

// A lane's partial scan: the first maximum over the non-NaN smoothed values (key), their
// minimum, NaN flags (bit 0: some smoothed value is NaN; bit 1: smoothed_0 is NaN).
struct InitScan {
  unsigned long long key;
  float lo;
  int nan;
};

__device__ __forceinline__ void scan_reset(InitScan& a) {
  a.key = 0ull;
  a.lo = __int_as_float(0x7f800000);
  a.nan = 0;
}

__device__ __forceinline__ void scan_take(InitScan& a, float v, int i) {
  if (v == v)
    a.key = key_max(a.key, scan_key(v, i));
  else
    a.nan |= i == 0 ? 3 : 1;
  a.lo = fminf(a.lo, v);
}

__device__ __forceinline__ void scan_merge(InitScan& a, unsigned long long key, float lo, int nan) {
  a.key = key_max(a.key, key);
  a.lo = fminf(a.lo, lo);
  a.nan |= nan;
}

// Merge across `width` lanes (xor butterfly, width a power of two <= 32); every lane of the
// warp calls it.
template <int WIDTH>
__device__ __forceinline__ void scan_reduce(InitScan& a) {
#pragma unroll
  for (int o = 1; o < WIDTH; o <<= 1)
    scan_merge(a, __shfl_xor_sync(0xffffffffu, a.key, o), __shfl_xor_sync(0xffffffffu, a.lo, o),
               __shfl_xor_sync(0xffffffffu, a.nan, o));
}

// The merged scan -> (idx, alpha, beta) with numpy's NaN semantics, and the M threshold.
__device__ __forceinline__ void init_finish(const InitScan& a, int& idx, float& alpha, float& beta, double& thr) {
  float best;
  if ((a.nan & 2) || a.key == 0ull) {  // smoothed_0 is NaN (or every value is): the scan never leaves it
    best = __int_as_float(0x7fc00000);
    idx = 0;
  } else {
    const unsigned o = (unsigned)(a.key >> 32);
    best = __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
    idx = ~(int)(unsigned)a.key;
  }
  beta = (a.nan & 1) ? __int_as_float(0x7fc00000) : a.lo;
  alpha = (float)__dadd_rn((double)best, -(double)beta);
  thr = __dadd_rn(__dmul_rn((double)alpha, kExpMinusHalf), (double)beta);
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

// General scan of pixels i = first, first + stride, ... < N of a staged spot.
template <typename PX>
__device__ __forceinline__ void init_scan(const PX* st, int W, int H, int N, float invW, int first, int stride,
                                          InitScan& a) {
#pragma unroll 1
  for (int i = first; i < N; i += stride) scan_take(a, init_smoothed(st, W, H, invW, i), i);
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

// ---------------------------------------------------------------------------
// Integer fast path, for spots whose pixel values are all integers in [0, 2^20]
// (camera counts; every u16 spot).  Every 3x3 partial sum is then an integer below
// 9 * 2^20 < 2^24, exact in f32 (or int) in any order, so it equals the pinned
// row-major f64 sum; and since numerator and count are exact in f32,
// f32(f64(s) / count) is the correctly rounded s / count (a double-precision
// intermediate (53 >= 2*24 + 2 bits) rounds innocuously), computed by tame_div.
// Each lane walks down a column (a segment of one when the grid is narrower than
// the group), two rows per trip, keeping the horizontal 3-sums of the rows above
// and below, so a pixel costs three loads and four adds instead of nine
// converted f64 taps.  M: for integer g, g > thr  <=>  g >= floor(thr) + 1.
// ---------------------------------------------------------------------------
template <typename PX>
struct TameAcc {
  using T = float;  // f32 pixels: exact f32 sums
};
template <>
struct TameAcc<uint16_t> {
  using T = int;  // 16-bit counts: integer sums
};

// s / c correctly rounded for an integer s in [0, 9 * 2^20] and c in {1, 2, 3, 4, 6, 9} (the
// truncated-window counts): q0 = RN(s rc), exact residual, one correction with rc = RN(1/c).
// Checked on the device for every such (s, c) (tests: sf_debug_tame_div_device).
__device__ __forceinline__ float tame_div(float s, float c, float rc) {
  const float q0 = __fmul_rn(s, rc);
  return __fmaf_rn(__fmaf_rn(-q0, c, s), rc, q0);
}

template <int LANES, typename PX>
__device__ __forceinline__ void init_scan_tame(const PX* st, int W, int H, int gl, InitScan& a) {
  using Acc = typename TameAcc<PX>::T;
  int S = W >= LANES ? 1 : LANES / W;  // row segments per column when the grid is narrow
  if (S > H) S = H;
  const int x0 = W >= LANES ? gl : gl % W;
  const int seg = W >= LANES ? 0 : gl / W;
  if (seg >= S) return;
  const int y0 = seg * H / S, y1 = (seg + 1) * H / S;
  const int xstep = W >= LANES ? LANES : W;
  unsigned long long key = a.key;
  float lo = a.lo;
#pragma unroll 1
  for (int x = x0; x < W; x += xstep) {
    // neighbour offsets: a missing neighbour reads the pixel itself and is masked by a 0/1 factor
    // (exact for integers), so the row loop has no branches
    const int ol = x > 0 ? -1 : 0, orr = x < W - 1 ? 1 : 0;
    const Acc ml = (Acc)(x > 0 ? 1 : 0), mr = (Acc)(x < W - 1 ? 1 : 0);
    const int cxi = 1 + (x > 0) + (x < W - 1);
    const float ci = (float)(3 * cxi), ce = (float)((H > 1 ? 2 : 1) * cxi);  // counts: inner / edge rows
    const float rci = __frcp_rn(ci), rce = __frcp_rn(ce);
    const PX* col = st + x;
    auto hsum = [&](int y) -> Acc {
      const PX* r = col + y * W;
      return (Acc)r[0] + ml * (Acc)r[ol] + mr * (Acc)r[orr];
    };
    auto value = [&](int y, Acc s) {
      const bool edge = y == 0 || y == H - 1;  // count 1, 2, 3, 4, 6 or 9
      return tame_div((float)s, edge ? ce : ci, edge ? rce : rci);
    };
    Acc prev = y0 > 0 ? hsum(y0 - 1) : (Acc)0;
    Acc cur = hsum(y0);
    // down the column the pixel index increases, so a strict ">" keeps the first maximum; the
    // column's (best, row) joins the lane's key once.  Two rows per trip for independent work.
    float best = -1.0f;  // below every tame value
    int brow = y0;
    int y = y0;
#pragma unroll 1
    for (; y + 1 < y1; y += 2) {
      const Acc n1 = hsum(y + 1);
      const Acc n2 = y + 2 < H ? hsum(y + 2) : (Acc)0;
      const float va = value(y, prev + cur + n1);
      const float vb = value(y + 1, cur + n1 + n2);
      const bool tb = vb > va;  // the pair's first maximum
      const float vm = tb ? vb : va;
      if (vm > best) {
        best = vm;
        brow = tb ? y + 1 : y;
      }
      lo = fminf(lo, fminf(va, vb));
      prev = n1;
      cur = n2;
    }
    if (y < y1) {
      const Acc n1 = y + 1 < H ? hsum(y + 1) : (Acc)0;
      const float va = value(y, prev + cur + n1);
      if (va > best) {
        best = va;
        brow = y;
      }
      lo = fminf(lo, va);
    }
    key = key_max(key, scan_key(best, brow * W + x));
  }
  a.key = key;
  a.lo = lo;
}

// M for a tame spot: #{g_i >= floor(thr) + 1} over pixels first, first + stride, ...
template <typename PX>
__device__ __forceinline__ int init_count_tame(const PX* st, int N, double thr, int first, int stride) {
  double t = floor(thr) + 1.0;  // integer-valued; clamped where the answer no longer depends on it
  t = t < -1.0 ? -1.0 : (t > 2097152.0 ? 2097152.0 : t);
  using Acc = typename TameAcc<PX>::T;
  const Acc tt = (Acc)t;
  int m = 0;
#pragma unroll 4
  for (int i = first; i < N; i += stride) m += ((Acc)st[i] >= tt) ? 1 : 0;
  return m;
}

}  // namespace sf
