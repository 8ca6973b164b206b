// sf_init.cu -- GPU initializer: estimate_initial for a whole batch
// (SURVEY 8f item 1).  One warp per spot.
// The arithmetic is pinned in sf_init_core.cuh (shared with the fit kernel's
// fused initializer) and restated in oracle/initializer.py.
#include <cfloat>
#include <climits>

#include "sf_init_core.cuh"
#include "sf_launch.h"

namespace sf {

namespace {

// Standalone initializer.  A warp takes G = 32 / L spots at a time (L lanes per
// spot: the smallest of 8, 16, 32 that covers a row, so every lane walks a
// column), persistent over the batch.  The next G spots stream into the warp's
// second staging buffer with cp.async while the current ones are scanned (one
// coalesced window per G spots: 16-byte copies, element copies only where the
// window pokes out of the caller's array), so the HBM latency is hidden and the
// per-spot reductions are shared by G spots per instruction.  A tame spot (every
// pixel an integer in [0, 2^20]: camera counts) takes the exact integer column
// walk of sf_init_core.cuh; any other spot the general f64 scan.
#ifndef SF_INIT_WARPS
#define SF_INIT_WARPS 8
#endif
#ifndef SF_INIT_MINB
#define SF_INIT_MINB 3
#endif
constexpr int kInitWarps = SF_INIT_WARPS;
#ifndef SF_INIT_QUAD
#define SF_INIT_QUAD 1  // odd-N f32 grids of width 9..32: four adjacent columns per lane
#endif
#ifndef SF_INIT_WARPS4
#define SF_INIT_WARPS4 3
#endif
#ifndef SF_INIT_MINB4
#define SF_INIT_MINB4 5
#endif
// warps per CTA and launch-bound CTAs per SM: the quad walk stages 7-8 KB of spots per warp and
// buffer, so it runs fewer warps per CTA
template <bool QUAD>
__host__ __device__ constexpr int init_warps() {
  return QUAD ? SF_INIT_WARPS4 : kInitWarps;
}
template <bool QUAD>
__host__ __device__ constexpr int init_minb() {
  return QUAD ? SF_INIT_MINB4 : SF_INIT_MINB;
}

#ifndef SF_INIT_PAIR
#define SF_INIT_PAIR 1  // L < W <= 2L: a lane walks two adjacent columns off one set of row loads
#endif
#ifndef SF_INIT_CCOUNT
#define SF_INIT_CCOUNT 1  // M of a tame spot over its contiguous pixels with 16-byte loads
#endif
#ifndef SF_INIT_TMA
#define SF_INIT_TMA 1  // stage a task's window with one bulk async copy (mbarrier completion)
#endif

// Bulk async copy (the TMA engine's non-tensor form) and its mbarrier.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT;\n}\n" ::"r"(
          smem_addr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_to_smem(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(b))
               : "memory");
}

template <typename PX>
__host__ __device__ constexpr int init_buf_elems(int G, int N) {
  // the 16-B aligned window around G*N pixels, in PX units (+ one 16-B line of slack each side)
  return ((G * N * (int)sizeof(PX) + 47) & ~15) / (int)sizeof(PX);
}

// A lane's column of the tame walk when the grid is no wider than the spot's lanes (W <= L, every
// 2D grid of the fitter): column x, rows [y0, y1) (several row segments per column when W < L / 2),
// with its window counts -- the geometry of sf_init_core.cuh's
// init_scan_tame, computed once per kernel instead of once per spot.
struct TameCol {
  bool active;
  int x, y0, y1;
  float ci, ce, rci, rce;
};

// Column k (0 or 1) of lane gl: when W <= L one column per lane, split into S row segments when
// W < L / 2; when L < W <= 2L two adjacent full-height columns per lane (x = 2 gl + k).
template <int L>
__device__ __forceinline__ TameCol tame_col(int W, int H, int gl, int k) {
  TameCol c;
  if (W <= L) {
    int S = L / W;  // row segments per column
    if (S > H) S = H;
    c.x = gl % W;
    const int seg = gl / W;
    c.active = k == 0 && seg < S;
    c.y0 = seg * H / S;
    c.y1 = (seg + 1) * H / S;
  } else {
#if SF_INIT_PAIR
    c.x = 2 * gl + k;  // adjacent columns: walk_pair shares the row loads
#else
    c.x = gl + k * L;
#endif
    c.active = c.x < W;
    c.y0 = 0;
    c.y1 = H;
  }
  const int cxi = 1 + (c.x > 0) + (c.x < W - 1);
  c.ci = (float)(3 * cxi);
  c.ce = (float)((H > 1 ? 2 : 1) * cxi);
  c.rci = __frcp_rn(c.ci);
  c.rce = __frcp_rn(c.ce);
  return c;
}

// The tame walk of NC columns in lockstep (the arithmetic of sf_init_core.cuh:init_scan_tame: same
// values, same first maximum and minimum; NC = 2 gives the walk two independent chains), which also
// checks the tame condition on every pixel it centres: the walk runs speculatively and its result is
// used only when the whole spot turns out tame, so the spot is read once for both.  Integer-valued
// pixels below 2^20 keep every partial sum exact in f32, so the order of the three taps does not
// matter.  Neighbours are read at constant offsets -1 / +1 from the row pointer (the staging area has
// a guard in front, see init_kernel) and a missing one (grid edge) is dropped by a select, never
// multiplied, so whatever lies there cannot leak in.  The top and bottom grid rows (window count
// 2 cxi) are peeled off the interior loop (3 cxi).  All columns share the rows [y0, y1) of cs[0].
template <int NC, typename PX>
__device__ __forceinline__ void walk_tame(const PX* st, int W, int H, const TameCol (&cs)[NC], InitScan& a,
                                          bool& tame) {
  using Acc = typename TameAcc<PX>::T;
  bool hl[NC] = {}, hr[NC] = {};
  const PX* p[NC];
  Acc prev[NC], cur[NC];
  float best[NC] = {};
  int brow[NC] = {};
  unsigned mx = 0u;   // max pixel bit pattern (negative, -0, inf, NaN and > 2^20 all exceed 0x49800000)
  bool frac = false;  // some pixel is not an integer
  float lo = a.lo;
  const int y0 = cs[0].y0, y1 = cs[0].y1;
  auto hsum = [&](int k, const PX* r) -> Acc {
    const PX v = r[0];
    if constexpr (sizeof(PX) == 4) {  // u16 counts are tame by construction
      const float f = (float)v;
      mx = max(mx, __float_as_uint(f));
      frac |= __fsub_rn(__fadd_rn(f, 8388608.0f), 8388608.0f) != f;
    }
    const Acc l = (Acc)r[-1], rr = (Acc)r[1];
    return ((Acc)v + (hl[k] ? l : (Acc)0)) + (hr[k] ? rr : (Acc)0);
  };
  auto take = [&](int k, float v, int y) {
    if (v > best[k]) {  // rows ascend: a strict ">" keeps the column's first maximum
      best[k] = v;
      brow[k] = y;
    }
    lo = fminf(lo, v);
  };
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    hl[k] = cs[k].x > 0;
    hr[k] = cs[k].x < W - 1;
    p[k] = st + cs[k].x + y0 * W;
    best[k] = -1.0f;  // below every tame value
    brow[k] = y0;
    prev[k] = y0 > 0 ? hsum(k, p[k] - W) : (Acc)0;
    cur[k] = hsum(k, p[k]);
  }
  int y = y0;
  if (y == 0) {  // top grid row
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const Acc nx = H > 1 ? hsum(k, p[k] + W) : (Acc)0;
      take(k, tame_div((float)(prev[k] + cur[k] + nx), cs[k].ce, cs[k].rce), 0);
      prev[k] = cur[k];
      cur[k] = nx;
      p[k] += W;
    }
    ++y;
  }
  const int yi = y1 < H - 1 ? y1 : H - 1;  // interior rows [y, yi): row y + 1 exists
#pragma unroll 2
  for (; y < yi; ++y) {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const Acc nx = hsum(k, p[k] + W);
      take(k, tame_div((float)(prev[k] + cur[k] + nx), cs[k].ci, cs[k].rci), y);
      prev[k] = cur[k];
      cur[k] = nx;
      p[k] += W;
    }
  }
  if (y < y1) {  // bottom grid row (y = H - 1 > 0)
#pragma unroll
    for (int k = 0; k < NC; ++k) take(k, tame_div((float)(prev[k] + cur[k]), cs[k].ce, cs[k].rce), y);
  }
  unsigned long long key = a.key;
#pragma unroll
  for (int k = 0; k < NC; ++k) key = key_max(key, scan_key(best[k], brow[k] * W + cs[k].x));
  a.key = key;
  a.lo = lo;
  if constexpr (sizeof(PX) == 4) tame = tame && mx <= 0x49800000u && !frac;
}

// M of a tame spot over the lane's NC columns (init_count_tame's test, g >= floor(thr) + 1, with the
// threshold clamped the same way), in lockstep; column k counts only when live[k].
template <int NC, typename PX>
__device__ __forceinline__ int count_columns(const PX* st, int W, const TameCol (&cs)[NC], const bool (&live)[NC],
                                             double thr) {
  double t = floor(thr) + 1.0;
  t = t < -1.0 ? -1.0 : (t > 2097152.0 ? 2097152.0 : t);
  using Acc = typename TameAcc<PX>::T;
  const Acc tt = (Acc)t;
  // f32 tame pixels are non-negative, so float order is the order of the bit patterns: compare bits
  // (a threshold <= 0 counts every pixel: +0 is the smallest tame bit pattern)
  const unsigned tb = __float_as_uint(fmaxf((float)t, 0.0f));
  const PX* p[NC];
  int m[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    p[k] = st + cs[k].x + cs[0].y0 * W;
    m[k] = 0;
  }
#pragma unroll 4
  for (int y = cs[0].y0; y < cs[0].y1; ++y) {
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      if constexpr (sizeof(PX) == 4)
        m[k] += (__float_as_uint((float)p[k][0]) >= tb) ? 1 : 0;
      else
        m[k] += ((Acc)p[k][0] >= tt) ? 1 : 0;
      p[k] += W;
    }
  }
  int r = 0;
#pragma unroll
  for (int k = 0; k < NC; ++k) r += live[k] ? m[k] : 0;
  return r;
}

// Two adjacent columns x = cs[0].x and x + 1 of one lane (L < W <= 2L), in lockstep: a row's four
// loads r[-1 .. 2] give both columns' horizontal 3-sums (four shared loads per row instead of six),
// otherwise walk_tame<2>'s arithmetic (integer sums exact in any order).  Column x + 1 exists iff
// liveB (= x < W - 1); without it its values are dropped from the scan and the tame check.
template <typename PX>
__device__ __forceinline__ void walk_pair(const PX* st, int W, int H, const TameCol (&cs)[2], bool liveB, InitScan& a,
                                          bool& tame) {
  using Acc = typename TameAcc<PX>::T;
  const int x = cs[0].x;
  const bool hlA = x > 0, hrB = x + 2 < W;
  unsigned mx = 0u;
  bool frac = false;
  float lo = a.lo, best0 = -1.0f, best1 = -1.0f;
  int brow0 = 0, brow1 = 0;
  auto row = [&](const PX* r, Acc& hA, Acc& hB) {
    const PX l = r[-1], c0 = r[0], c1 = r[1], rr = r[2];
    if constexpr (sizeof(PX) == 4) {
      const float f0 = (float)c0, f1 = liveB ? (float)c1 : 0.0f;
      mx = max(mx, max(__float_as_uint(f0), __float_as_uint(f1)));
      frac |= (__fsub_rn(__fadd_rn(f0, 8388608.0f), 8388608.0f) != f0) |
              (__fsub_rn(__fadd_rn(f1, 8388608.0f), 8388608.0f) != f1);
    }
    hA = ((Acc)c0 + (hlA ? (Acc)l : (Acc)0)) + (liveB ? (Acc)c1 : (Acc)0);
    hB = ((Acc)c1 + (Acc)c0) + (hrB ? (Acc)rr : (Acc)0);
  };
  auto take = [&](float vA, float vB, int y) {
    if (vA > best0) {
      best0 = vA;
      brow0 = y;
    }
    if (vB > best1) {
      best1 = vB;
      brow1 = y;
    }
    lo = fminf(lo, liveB ? fminf(vA, vB) : vA);
  };
  const PX* p = st + x;
  Acc pA = (Acc)0, pB = (Acc)0, cA, cB, nA, nB;
  row(p, cA, cB);
  int y = 0;
  {  // top grid row
    if (H > 1) row(p + W, nA, nB);
    else nA = nB = (Acc)0;
    take(tame_div((float)(pA + cA + nA), cs[0].ce, cs[0].rce), tame_div((float)(pB + cB + nB), cs[1].ce, cs[1].rce), 0);
    pA = cA; pB = cB; cA = nA; cB = nB;
    p += W;
    ++y;
  }
#pragma unroll 2
  for (; y < H - 1; ++y) {
    row(p + W, nA, nB);
    take(tame_div((float)(pA + cA + nA), cs[0].ci, cs[0].rci), tame_div((float)(pB + cB + nB), cs[1].ci, cs[1].rci), y);
    pA = cA; pB = cB; cA = nA; cB = nB;
    p += W;
  }
  if (y < H)  // bottom grid row (y = H - 1 > 0)
    take(tame_div((float)(pA + cA), cs[0].ce, cs[0].rce), tame_div((float)(pB + cB), cs[1].ce, cs[1].rce), y);
  unsigned long long key = key_max(a.key, scan_key(best0, brow0 * W + x));
  if (liveB) key = key_max(key, scan_key(best1, brow1 * W + x + 1));
  a.key = key;
  a.lo = lo;
  if constexpr (sizeof(PX) == 4) tame = tame && mx <= 0x49800000u && !frac;
}

// walk_pair for f32 pixels with the two columns in the halves of f32x2 registers: the horizontal
// sums, the vertical sums, the tame check's rounding and tame_div run as FADD2 / FFMA2 / FMUL2 (the
// same IEEE operation on each half).  A missing neighbour (grid edge, or column x + 1 when !liveB)
// is read from the row's own pixel x and multiplied by 0: exact, and finite whenever the spot is tame
// (a tame spot's pixels are integers), so nothing from outside the spot can reach a tame result.
__device__ __forceinline__ void walk_pair_f32(const float* st, int W, int H, const TameCol (&cs)[2], bool liveB,
                                              InitScan& a, bool& tame) {
  const int x = cs[0].x;
  // neighbour offsets of the top and bottom grid rows, where a missing neighbour would lie outside
  // the spot; inside the grid the row above / below is the same spot's, so the interior rows read at
  // constant offsets -1 .. 2 and the 0 factor alone drops a missing neighbour
  const int oL = x > 0 ? -1 : 0, o1 = liveB ? 1 : 0, o2 = x + 2 < W ? 2 : 0;
  const f2 mL = pk2(x > 0 ? 1.0f : 0.0f, 1.0f), mR = pk2(liveB ? 1.0f : 0.0f, x + 2 < W ? 1.0f : 0.0f);
  const f2 nci = pk2(-cs[0].ci, -cs[1].ci), rci = pk2(cs[0].rci, cs[1].rci);
  const f2 nce = pk2(-cs[0].ce, -cs[1].ce), rce = pk2(cs[0].rce, cs[1].rce);
  const f2 big = bc2(8388608.0f), nbig = bc2(-8388608.0f), nz = bc2(-0.0f);
  unsigned mx = 0u, fr = 0u;
  float loA = a.lo, loB = a.lo, best0 = -1.0f, best1 = -1.0f;
  int brow0 = 0, brow1 = 0;
  auto hsum = [&](float l, float c0, float c1, float rr) -> f2 {
    mx = __vimax3_u32(mx, __float_as_uint(c0), __float_as_uint(c1));
    const f2 c = pk2(c0, c1);
    // tame check: __fsub_rn(__fadd_rn(g, 2^23), 2^23) == g bitwise for both halves (-0.0 fails it,
    // as it fails the bound on mx)
    const f2 i = add2(add2(c, big), nbig);
    fr |= (unsigned)(i.v ^ c.v) | (unsigned)((i.v ^ c.v) >> 32);
    return fma2(pk2(c1, rr), mR, fma2(pk2(l, c0), mL, c));  // (g + l [x > 0]) + r [x < W - 1] per half
  };
  auto row_edge = [&](const float* r) { return hsum(r[oL], r[0], r[o1], r[o2]); };
  auto row = [&](const float* r) { return hsum(r[-1], r[0], r[1], r[2]); };
  auto div = [&](f2 sum, f2 nc, f2 rc) -> f2 {  // tame_div per half
    const f2 q0 = mul2(sum, rc, nz);
    return fma2(fma2(q0, nc, sum), rc, q0);
  };
  auto take = [&](f2 v, int y) {
    float vA, vB;
    up2(v, vA, vB);
    if (vA > best0) {
      best0 = vA;
      brow0 = y;
    }
    if (vB > best1) {
      best1 = vB;
      brow1 = y;
    }
    loA = fminf(loA, vA);
    loB = fminf(loB, vB);
  };
  const float* p = st + x;
  f2 pv = bc2(0.0f), cu = row_edge(p), nx = bc2(0.0f);
  if (H > 1) nx = H > 2 ? row(p + W) : row_edge(p + W);
  take(div(add2(add2(pv, cu), nx), nce, rce), 0);  // top grid row
  pv = cu;
  cu = nx;
  p += W;
  int y = 1;
  for (; y < H - 2; ++y) {  // interior rows whose row below is interior too
    nx = row(p + W);
    take(div(add2(add2(pv, cu), nx), nci, rci), y);
    pv = cu;
    cu = nx;
    p += W;
  }
  if (y < H - 1) {  // the last interior row: the row below is the bottom grid row
    nx = row_edge(p + W);
    take(div(add2(add2(pv, cu), nx), nci, rci), y);
    pv = cu;
    cu = nx;
    ++y;
  }
  if (y < H) take(div(add2(pv, cu), nce, rce), y);  // bottom grid row (y = H - 1 > 0)
  unsigned long long key = key_max(a.key, scan_key(best0, brow0 * W + x));
  if (liveB) key = key_max(key, scan_key(best1, brow1 * W + x + 1));
  a.key = key;
  a.lo = liveB ? fminf(loA, loB) : loA;
  tame = tame && mx <= 0x49800000u && fr == 0u;
}

// The tame walk of four adjacent columns x .. x + 3 of one lane (8 < W <= 16, L = 4), the columns in
// the halves of two f32x2 registers: a row's six loads r[-1 .. 4] give all four horizontal 3-sums,
// otherwise walk_pair_f32's arithmetic and edge handling (a missing neighbour or a column beyond the
// grid reads a pixel of the row itself in the top and bottom grid rows, a pixel of the same spot
// elsewhere, and is multiplied by 0 or dropped from the scan).
__device__ __forceinline__ void walk_quad_f32(const float* st, int W, int H, int x, InitScan& a, bool& tame) {
  bool live[4];
  float cif[4], cef[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    live[k] = x + k < W;
    const int xc = live[k] ? x + k : x;
    const int cxi = 1 + (xc > 0) + (xc < W - 1);
    cif[k] = (float)(3 * cxi);
    cef[k] = (float)((H > 1 ? 2 : 1) * cxi);
  }
  const f2 nciA = pk2(-cif[0], -cif[1]), nciB = pk2(-cif[2], -cif[3]);
  const f2 rciA = pk2(__frcp_rn(cif[0]), __frcp_rn(cif[1])), rciB = pk2(__frcp_rn(cif[2]), __frcp_rn(cif[3]));
  const f2 nceA = pk2(-cef[0], -cef[1]), nceB = pk2(-cef[2], -cef[3]);
  const f2 rceA = pk2(__frcp_rn(cef[0]), __frcp_rn(cef[1])), rceB = pk2(__frcp_rn(cef[2]), __frcp_rn(cef[3]));
  const int oL = x > 0 ? -1 : 0, o1 = live[1] ? 1 : 0, o2 = live[2] ? 2 : 0, o3 = live[3] ? 3 : 0,
            o4 = x + 4 < W ? 4 : 0;
  const f2 mLa = pk2(x > 0 ? 1.0f : 0.0f, 1.0f);
  const f2 mRa = pk2(live[1] ? 1.0f : 0.0f, live[2] ? 1.0f : 0.0f);
  const f2 mRb = pk2(live[3] ? 1.0f : 0.0f, x + 4 < W ? 1.0f : 0.0f);
  const f2 big = bc2(8388608.0f), nbig = bc2(-8388608.0f), nz = bc2(-0.0f);
  unsigned mx = 0u, fr = 0u;
  float lo0 = a.lo, lo1 = a.lo, lo2 = a.lo, lo3 = a.lo;
  float b0 = -1.0f, b1 = -1.0f, b2 = -1.0f, b3 = -1.0f;
  int y0r = 0, y1r = 0, y2r = 0, y3r = 0;
  auto hsum = [&](float l, float r0, float r1, float r2, float r3, float r4, f2& hA, f2& hB) {
    mx = __vimax3_u32(mx, __float_as_uint(r0), __float_as_uint(r1));
    mx = __vimax3_u32(mx, __float_as_uint(r2), __float_as_uint(r3));
    const f2 cA = pk2(r0, r1), cB = pk2(r2, r3);
    const f2 iA = add2(add2(cA, big), nbig), iB = add2(add2(cB, big), nbig);  // tame check per half
    const unsigned long long d = (iA.v ^ cA.v) | (iB.v ^ cB.v);
    fr |= (unsigned)d | (unsigned)(d >> 32);
    const f2 p12 = pk2(r1, r2);
    hA = fma2(p12, mRa, fma2(pk2(l, r0), mLa, cA));  // (r0 + l [x > 0] + r1 [.], r1 + r0 + r2 [.])
    hB = fma2(pk2(r3, r4), mRb, add2(p12, cB));      // (r2 + r1 + r3 [.], r3 + r2 + r4 [.])
  };
  auto row_edge = [&](const float* r, f2& hA, f2& hB) { hsum(r[oL], r[0], r[o1], r[o2], r[o3], r[o4], hA, hB); };
  auto row = [&](const float* r, f2& hA, f2& hB) { hsum(r[-1], r[0], r[1], r[2], r[3], r[4], hA, hB); };
  auto div = [&](f2 sum, f2 nc, f2 rc) -> f2 {  // tame_div per half
    const f2 q0 = mul2(sum, rc, nz);
    return fma2(fma2(q0, nc, sum), rc, q0);
  };
  auto take = [&](f2 vA, f2 vB, int y) {
    float v0, v1, v2, v3;
    up2(vA, v0, v1);
    up2(vB, v2, v3);
    if (v0 > b0) { b0 = v0; y0r = y; }
    if (v1 > b1) { b1 = v1; y1r = y; }
    if (v2 > b2) { b2 = v2; y2r = y; }
    if (v3 > b3) { b3 = v3; y3r = y; }
    lo0 = fminf(lo0, v0);
    lo1 = fminf(lo1, v1);
    lo2 = fminf(lo2, v2);
    lo3 = fminf(lo3, v3);
  };
  const float* p = st + x;
  const f2 z = bc2(0.0f);
  f2 pA = z, pB = z, cA, cB, nA = z, nB = z;
  row_edge(p, cA, cB);
  if (H > 1) {
    if (H > 2) row(p + W, nA, nB);
    else row_edge(p + W, nA, nB);
  }
  take(div(add2(add2(pA, cA), nA), nceA, rceA), div(add2(add2(pB, cB), nB), nceB, rceB), 0);  // top grid row
  pA = cA; pB = cB; cA = nA; cB = nB;
  p += W;
  int y = 1;
  for (; y < H - 2; ++y) {  // interior rows whose row below is interior too
    row(p + W, nA, nB);
    take(div(add2(add2(pA, cA), nA), nciA, rciA), div(add2(add2(pB, cB), nB), nciB, rciB), y);
    pA = cA; pB = cB; cA = nA; cB = nB;
    p += W;
  }
  if (y < H - 1) {  // the last interior row: the row below is the bottom grid row
    row_edge(p + W, nA, nB);
    take(div(add2(add2(pA, cA), nA), nciA, rciA), div(add2(add2(pB, cB), nB), nciB, rciB), y);
    pA = cA; pB = cB; cA = nA; cB = nB;
    ++y;
  }
  if (y < H) take(div(add2(pA, cA), nceA, rceA), div(add2(pB, cB), nceB, rceB), y);  // bottom grid row
  unsigned long long key = key_max(a.key, scan_key(b0, y0r * W + x));
  float lo = lo0;
  if (live[1]) { key = key_max(key, scan_key(b1, y1r * W + x + 1)); lo = fminf(lo, lo1); }
  if (live[2]) { key = key_max(key, scan_key(b2, y2r * W + x + 2)); lo = fminf(lo, lo2); }
  if (live[3]) { key = key_max(key, scan_key(b3, y3r * W + x + 3)); lo = fminf(lo, lo3); }
  a.key = key;
  a.lo = lo;
  tame = tame && mx <= 0x49800000u && fr == 0u;
}

// M of a tame spot (init_count_tame's test, g >= floor(thr) + 1, the threshold clamped the same
// way) over its N contiguous staged pixels: 16-byte loads strided over the spot's L lanes.  The
// first and last chunk reach outside the spot (into valid staging memory) and are masked by index
// (u16: every chunk is counted whole, and the lanes holding those two take back what lies outside).
template <int L, typename PX>
__device__ __forceinline__ int count_contig(const PX* sp, int N, double thr, int sl) {
  double t = floor(thr) + 1.0;
  t = t < -1.0 ? -1.0 : (t > 2097152.0 ? 2097152.0 : t);
  constexpr int E = 16 / (int)sizeof(PX);
  const int h = (int)(((uintptr_t)sp & 15) / sizeof(PX));
  const uint4* q = reinterpret_cast<const uint4*>(sp - h);
  const int nc = (h + N + E - 1) / E, tail = nc * E - (h + N);  // h elements before, tail after
  (void)tail;
  int m = 0;
  if constexpr (sizeof(PX) == 4) {
    // Inner chunks (wholly inside the spot, integer pixels): g >= t <=> sat(g + (1 - t)) = 1, else 0
    // (every operand an integer below 2^22: exact), summed in f32x2 pairs (exact below 2^24).  The
    // first and last chunk (partly outside the spot) compare bit patterns under an index mask (tame
    // f32 pixels are non-negative, so float order is bit-pattern order; t <= 0 counts every one).
    const float k1 = (float)(1.0 - t);
    const unsigned tb = __float_as_uint(fmaxf((float)t, 0.0f));
    f2 s01 = bc2(0.0f), s23 = bc2(0.0f);
#pragma unroll 2
    for (int c = sl ? sl : L; c < nc - 1; c += L) {
      const float4 v = reinterpret_cast<const float4*>(q)[c];
      s01 = add2(s01, pk2(__saturatef(__fadd_rn(v.x, k1)), __saturatef(__fadd_rn(v.y, k1))));
      s23 = add2(s23, pk2(__saturatef(__fadd_rn(v.z, k1)), __saturatef(__fadd_rn(v.w, k1))));
    }
    float a0, a1, b0, b1;
    up2(s01, a0, a1);
    up2(s23, b0, b1);
    m = (int)((a0 + a1) + (b0 + b1));
    auto edge = [&](int c) {
      const uint4 v = q[c];
      const unsigned u[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) m += (c * 4 + j >= h && c * 4 + j < h + N && u[j] >= tb) ? 1 : 0;
    };
    if (sl == 0) edge(0);
    if (nc > 1 && sl == (nc - 1) % L) edge(nc - 1);
  } else {
    const int tt = (int)t;
    auto ge2 = [&](unsigned w, int j) { return (int)((w >> (16 * (j & 1))) & 0xffffu) >= tt ? 1 : 0; };
#pragma unroll 2
    for (int c = sl; c < nc; c += L) {
      const uint4 v = q[c];
      const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) m += ge2(w[j >> 1], j);
    }
    if (sl == 0) {
      const uint4 v = q[0];
      const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 7; ++j) m -= j < h ? ge2(w[j >> 1], j) : 0;
    }
    if (sl == (nc - 1) % L) {
      const uint4 v = q[nc - 1];
      const unsigned w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 1; j < 8; ++j) m -= j >= 8 - tail ? ge2(w[j >> 1], j) : 0;
    }
  }
  return m;
}

template <int L, typename PX, bool QUAD, bool SMALL = QUAD>
__global__ void __launch_bounds__(32 * init_warps<SMALL>(), init_minb<SMALL>()) init_kernel(const PX* __restrict__ images, int W, int H,
                                                              int64_t count, int P, double smin, double smax,
                                                              float* __restrict__ inits, float* __restrict__ amps) {
  constexpr int G = 32 / L;
  constexpr int kInitWarps = init_warps<SMALL>();  // (shadows the default for this instantiation)
  extern __shared__ __align__(16) unsigned char init_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane / L, sl = lane % L;  // spot of the warp's G, lane within the spot
  const int N = W * H;
  const int be = init_buf_elems<PX>(G, N);
  // 16-byte guard in front of the staging buffers: the tame walk reads a row's left neighbour at a
  // constant -1 offset (and drops it at the grid edge), so the first spot of warp 0 reads inside smem
  PX* buf = reinterpret_cast<PX*>(init_smem + 16) + (size_t)warp * 2 * be;
  const float invW = 1.0f / (float)W;
  const int64_t ntask = (count + G - 1) / G;
  const int64_t stride = (int64_t)gridDim.x * kInitWarps;
  const uintptr_t lo = (uintptr_t)images, hi = (uintptr_t)(images + count * (int64_t)N);
  // the warp's two staging mbarriers (after the sigma table)
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      init_smem + ((16 + (size_t)kInitWarps * 2 * be * sizeof(PX) + (size_t)(N + 1) * sizeof(float) + 7) & ~(size_t)7)) +
      2 * warp;
  // stage task t (spots t*G .. t*G+G-1) into buffer b; returns the first spot's element offset
  auto stage = [&](int64_t t, int b) -> int {
    const PX* src = images + t * G * (int64_t)N;
    const uintptr_t a0 = (uintptr_t)src & ~(uintptr_t)15;
    uintptr_t e0 = ((uintptr_t)(src + G * (int64_t)N) + 15) & ~(uintptr_t)15;
    if (e0 > ((hi + 15) & ~(uintptr_t)15)) e0 = (hi + 15) & ~(uintptr_t)15;
    const int nck = (int)((e0 - a0) >> 4);
    PX* dst = buf + b * be;
#if SF_INIT_TMA
    if (a0 >= lo && e0 <= hi) {  // the whole window inside the caller's array: one bulk copy
      if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // after the warp's reads of dst
        mbar_arrive_tx(&bars[b], (uint32_t)(e0 - a0));
        bulk_to_smem(dst, reinterpret_cast<const void*>(a0), (uint32_t)(e0 - a0), &bars[b]);
      }
      return (int)(((uintptr_t)src & 15) / sizeof(PX));
    }
    for (int c = lane; c < nck; c += 32) {  // the window pokes out of the caller's array
      const uintptr_t cs = a0 + 16 * (uintptr_t)c;
#pragma unroll
      for (int w = 0; w < 16 / (int)sizeof(PX); ++w)
        if (cs + sizeof(PX) * w >= lo && cs + sizeof(PX) * (w + 1) <= hi)
          reinterpret_cast<PX*>(dst)[(16 / sizeof(PX)) * c + w] = *reinterpret_cast<const PX*>(cs + sizeof(PX) * w);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars[b]);
    return (int)(((uintptr_t)src & 15) / sizeof(PX));
#else
    if (a0 >= lo && e0 <= hi) {  // the whole window inside the caller's array: 16-byte copies only
      const char* s0 = reinterpret_cast<const char*>(a0);
      float* d0 = reinterpret_cast<float*>(dst);
#pragma unroll 4
      for (int c = lane; c < nck; c += 32) cp_async16(d0 + 4 * c, s0 + 16 * c);
      return (int)(((uintptr_t)src & 15) / sizeof(PX));
    }
    for (int c = lane; c < nck; c += 32) {
      const uintptr_t cs = a0 + 16 * (uintptr_t)c;
      float* d = reinterpret_cast<float*>(dst) + 4 * c;
      if (cs >= lo && cs + 16 <= hi) {
        cp_async16(d, reinterpret_cast<const void*>(cs));
      } else {  // the window pokes out of the caller's array: in-bounds elements only
#pragma unroll
        for (int w = 0; w < 16 / (int)sizeof(PX); ++w)
          if (cs + sizeof(PX) * w >= lo && cs + sizeof(PX) * (w + 1) <= hi)
            reinterpret_cast<PX*>(d)[w] = *reinterpret_cast<const PX*>(cs + sizeof(PX) * w);
      }
    }
    return (int)(((uintptr_t)src & 15) / sizeof(PX));
#endif
  };
  // sigma(M) for every possible M, once per CTA (init_sigma: the same f64 ops, so the same floats)
  float* sig_tab = reinterpret_cast<float*>(init_smem + 16 + (size_t)kInitWarps * 2 * be * sizeof(PX));
  for (int m = threadIdx.x; m <= N; m += blockDim.x) sig_tab[m] = init_sigma(m, smin, smax);
#if SF_INIT_TMA
  if (lane == 0) {
    mbar_init(&bars[0]);
    mbar_init(&bars[1]);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
#endif
  __syncthreads();
  // every 2D grid (W <= 2L): at most two columns per lane, geometry hoisted out of the spot loop
  const bool narrow = W <= 2 * L;
  const bool two = narrow && W > L;  // two full-height columns per lane, walked in lockstep
  const TameCol tc0 = narrow ? tame_col<L>(W, H, sl, 0) : TameCol{};
  TameCol tcs[2] = {tc0, narrow ? tame_col<L>(W, H, sl, 1) : TameCol{}};
  const bool live[2] = {tc0.active, tcs[1].active};
  if (!tcs[1].active) tcs[1] = tc0;  // a lane without a second column repeats its first (same values)
  const TameCol one[1] = {tc0};
#if !SF_INIT_CCOUNT
  const bool live1[1] = {true};
#endif
  int64_t t = (int64_t)blockIdx.x * kInitWarps + warp;
  int off0 = 0, off1 = 0;  // window offsets of the two staging buffers (registers, no local array)
  if (t < ntask) off0 = stage(t, 0);
#if !SF_INIT_TMA
  cp_async_commit();
#endif
#pragma unroll 1
  for (int i = 0; t < ntask; t += stride, ++i) {
    const int b = i & 1;
    if (t + stride < ntask) {
      const int o = stage(t + stride, b ^ 1);
      if (b) off0 = o;
      else off1 = o;
    }
#if SF_INIT_TMA
    mbar_wait(&bars[b], (uint32_t)(i >> 1) & 1u);  // this task's window has landed (use i >> 1 of buffer b)
#else
    cp_async_commit();
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // this task's copies have landed
#endif
    __syncwarp();
    const int64_t spot = t * G + sub;
    const bool valid = spot < count;
    const PX* sp = buf + b * be + (b ? off1 : off0) + sub * N;
    InitScan a;
    scan_reset(a);
    bool tame = true;
    if constexpr (QUAD) {  // 4 (L - 1) < W <= 4 L: four adjacent columns per lane
      if (valid && 4 * sl < W) walk_quad_f32(reinterpret_cast<const float*>(sp), W, H, 4 * sl, a, tame);
    } else if (narrow) {  // speculative tame walk that checks tameness as it goes
      if (valid && tc0.active) {
        if (two)
#if SF_INIT_PAIR
        {
          if constexpr (sizeof(PX) == 4)
            walk_pair_f32(reinterpret_cast<const float*>(sp), W, H, tcs, live[1], a, tame);
          else
            walk_pair<PX>(sp, W, H, tcs, live[1], a, tame);
        }
#else
          walk_tame<2, PX>(sp, W, H, tcs, a, tame);
#endif
        else
          walk_tame<1, PX>(sp, W, H, one, a, tame);
      }
    } else if (valid) {
      for (int j = sl; j < N; j += L) {
        const float v = (float)sp[j];
        tame = tame && __float_as_uint(v) <= 0x49800000u && __fsub_rn(__fadd_rn(v, 8388608.0f), 8388608.0f) == v;
      }
    }
    int tm = tame ? 1 : 0;  // AND over the spot's lanes (every lane shuffles: no short-circuit)
#pragma unroll
    for (int o = 1; o < L; o <<= 1) tm &= __shfl_xor_sync(kFull, tm, o);
    tame = tm != 0;
    if (valid) {
      if (!tame) {  // the general f64 scan (rare: non-integer or large pixel values)
        scan_reset(a);
        init_scan(sp, W, H, N, invW, sl, L, a);
      } else if (!narrow && !QUAD) {
        init_scan_tame<L, PX>(sp, W, H, sl, a);
      }
    }
    scan_reduce<L>(a);
    int idx;
    float alpha, beta;
    double thr;
    init_finish(a, idx, alpha, beta, thr);
    int m = 0;
    if (valid) {
#if SF_INIT_CCOUNT
      m = tame ? count_contig<L, PX>(sp, N, thr, sl) : init_count(sp, N, thr, sl, L);
#else
      if (tame && narrow)
        m = !tc0.active ? 0 : (two ? count_columns<2, PX>(sp, W, tcs, live, thr) : count_columns<1, PX>(sp, W, one, live1, thr));
      else
        m = tame ? init_count_tame(sp, N, thr, sl, L) : init_count(sp, N, thr, sl, L);
#endif
    }
#pragma unroll
    for (int o = 1; o < L; o <<= 1) m += __shfl_xor_sync(kFull, m, o);
    if (valid) {
      const float sg = sig_tab[m];
      // (x, y, sigma[, sigma]); P = 5 (explicit-5, internal): (x, y, sigma, alpha, beta), the fifth
      // entry by lane 0 when the spot has only 4 lanes
      const int y = (int)(((float)idx + 0.5f) * invW);  // idx / W exactly (see init_smoothed)
      if (sl < P)
        inits[spot * P + sl] = sl == 0 ? (float)(idx - y * W)
                                       : (sl == 1 ? (float)y : (sl == 2 || P == 4 ? sg : (sl == 3 ? alpha : beta)));
      if constexpr (L < 5)
        if (P == 5 && sl == 0) inits[spot * P + 4] = beta;
      if (amps != nullptr && sl < 2) amps[2 * spot + sl] = sl == 0 ? alpha : beta;
    }
    __syncwarp();  // buffer b is restaged two tasks later
  }
#if !SF_INIT_TMA
  cp_async_wait_all();
#endif
}

template <int L, typename PX, bool QUAD = false, bool SMALL = QUAD>
cudaError_t launch_init_l(const PX* images, int W, int H, int64_t count, int P, double smin, double smax,
                          float* inits, float* amps, cudaStream_t stream) {
  constexpr int G = 32 / L;
  constexpr int kInitWarps = init_warps<SMALL>();
  // staging buffers (<= 66 KB) + the sigma(M) table
  const size_t smem = ((16 + (size_t)kInitWarps * 2 * init_buf_elems<PX>(G, W * H) * sizeof(PX) +
                       (size_t)(W * H + 1) * sizeof(float) + 7) & ~(size_t)7) +
                     (size_t)kInitWarps * 2 * sizeof(uint64_t);
  auto kern = init_kernel<L, PX, QUAD, SMALL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0, per_sm = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kInitWarps, smem)) != cudaSuccess)
    return e;
  int64_t blocks = (int64_t)(per_sm > 0 ? per_sm : 1) * sms;
  const int64_t need = ((count + G - 1) / G + kInitWarps - 1) / kInitWarps;
  if (blocks > need) blocks = need;
  kern<<<(unsigned)blocks, 32 * kInitWarps, smem, stream>>>(images, W, H, count, P, smin, smax, inits, amps);
  return cudaGetLastError();
}
}  // namespace

template <typename PX>
cudaError_t launch_init_px(const PX* images, int W, int H, int64_t count, int P, double sigma_min, double sigma_max,
                           float* inits, float* amps, cudaStream_t stream) {
  if (count <= 0) return cudaSuccess;
  const int N = W * H;
  // L lanes per spot, G = 32 / L spots per warp: the fewest lanes that leave each lane at most two
  // columns (W <= 2L) with G * N <= 1024 pixels per warp buffer; more spots per warp share the
  // per-spot reductions and bookkeeping
#ifndef SF_INIT_QUAD8_EVEN
#define SF_INIT_QUAD8_EVEN 1  // widths 17..32: the quad walk for even N too (2-way bank conflicts at most, still faster)
#endif
  if constexpr (sizeof(PX) == 4 && SF_INIT_QUAD) {  // f32 pixels only (walk_quad_f32)
    // widths 9..16: odd N only -- the 8 spots of a warp then start an odd number of words apart, which
    // spreads their lanes' shared loads over the banks (an even N such as 16x16 lines them up: 8-way)
    if ((N & 1) && W > 8 && W <= 16 && N <= 256)
      return launch_init_l<4, PX, true>(images, W, H, count, P, sigma_min, sigma_max, inits, amps, stream);
    if ((N & 1 || SF_INIT_QUAD8_EVEN) && W > 16 && W <= 32 && N <= 512)
      return launch_init_l<8, PX, true>(images, W, H, count, P, sigma_min, sigma_max, inits, amps, stream);
  }
#ifndef SF_INIT_SMALLPAIR
#define SF_INIT_SMALLPAIR 0
#endif
  if (W <= 16 && N <= 256)
    return launch_init_l<8, PX, false, SF_INIT_SMALLPAIR>(images, W, H, count, P, sigma_min, sigma_max, inits, amps, stream);
  if (W <= 32 && N <= 512)
    return launch_init_l<16, PX, false, SF_INIT_SMALLPAIR>(images, W, H, count, P, sigma_min, sigma_max, inits, amps, stream);
#ifndef SF_INIT_BIGPAIR
#define SF_INIT_BIGPAIR 1
#endif
  // 16 < W <= 32 with N up to 1024 (32x32): adjacent pairs on 16 lanes, 2 spots per warp, in small CTAs
  // (3 warps) so that the 8 KB staging windows still leave 12 warps per SM
  if (SF_INIT_BIGPAIR && W > 16 && W <= 32 && N <= 1024)
    return launch_init_l<16, PX, false, true>(images, W, H, count, P, sigma_min, sigma_max, inits, amps, stream);
  return launch_init_l<32, PX>(images, W, H, count, P, sigma_min, sigma_max, inits, amps, stream);
}

cudaError_t launch_estimate_initial(const float* images, int W, int H, int64_t count, int P, double sigma_min,
                                    double sigma_max, float* inits, float* amps, cudaStream_t stream) {
  return launch_init_px<float>(images, W, H, count, P, sigma_min, sigma_max, inits, amps, stream);
}

cudaError_t launch_estimate_initial_u16(const uint16_t* images, int W, int H, int64_t count, int P,
                                        double sigma_min, double sigma_max, float* inits, float* amps,
                                        cudaStream_t stream) {
  return launch_init_px<uint16_t>(images, W, H, count, P, sigma_min, sigma_max, inits, amps, stream);
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

// Exhaustive check of the initializer's integer-path division: tame_div(s, c) == __fdiv_rn(s, c)
// for every integer s in [0, 9 * 2^20] and c in {1, 2, 3, 4, 6, 9}; counts mismatches.
__global__ void tame_div_kernel(unsigned long long* mismatches) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = 9LL * 1048576 + 1;
  if (t >= 6 * n) return;
  const int cs[6] = {1, 2, 3, 4, 6, 9};
  const float c = (float)cs[t / n];
  const float s = (float)(t % n);
  if (__float_as_uint(tame_div(s, c, __frcp_rn(c))) != __float_as_uint(__fdiv_rn(s, c))) atomicAdd(mismatches, 1ull);
}

cudaError_t launch_tame_div(unsigned long long* mismatches, cudaStream_t stream) {
  const int64_t n = 6 * (9LL * 1048576 + 1);
  tame_div_kernel<<<(unsigned)((n + 255) / 256), 256, 0, stream>>>(mismatches);
  return cudaGetLastError();
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
