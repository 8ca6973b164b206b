// sf_inst.cu -- one template-instantiation unit per (SF_P, SF_SLOTS); the
// build compiles this file once per pair (paper_2106_02045_b200/build.py) so
// the fully unrolled kernels compile in parallel.
//
// (CH, TL) = (chain pixels, tail pixels) per lane.  Exact instantiations for
// the benchmark and common square shapes -- 11x11 -> S1 (15,1), 15x15 -> S2
// (14,1), 21x21 -> S4 (14,1), 32x32 -> S8 (16,0) -- plus generic fallbacks with
// TL = 7 so that every N <= 1024 has a kernel (extra pixel slots are masked:
// they cost issue slots, never correctness).  The dispatcher picks the
// cheapest (CH + TL) instantiation with CH >= need and TL >= need.
#include "sf_launch.h"

#ifndef SF_P
#error "compile with -DSF_P=3|4 -DSF_SLOTS=1|2|4|8|16"
#endif

// clang-format off
#if SF_SLOTS == 1
#define SF_SHAPES(X) X(8,0) X(10,1) X(15,1) X(4,4) X(12,4) X(2,7) X(6,7) X(10,7) X(16,7)
#elif SF_SLOTS == 2
#define SF_SHAPES(X) X(14,1) X(16,0) X(9,0) X(11,1) X(12,4) X(12,7) X(16,7)
#elif SF_SLOTS == 4
#define SF_SHAPES(X) X(14,1) X(12,1) X(13,0) X(9,1) X(10,4) X(15,4) X(12,7) X(16,7)
#elif SF_SLOTS == 8
#define SF_SHAPES(X) X(16,0) X(16,1) X(15,1) X(14,1) X(13,0) X(12,1) X(10,1) X(9,0) X(11,4) X(14,4) X(12,7) X(16,7)
#elif SF_SLOTS == 16
#define SF_SHAPES(X) X(16,7)
#endif
// clang-format on

#define SF_CAT5(a, b, c, d, e) a##b##c##d##e
#define SF_UNIT_NAME(kind, P, S) SF_CAT5(kind, _P, P, _S, S)

namespace sf {

namespace {
template <int CH, int TL>
cudaError_t go_fit(const LaunchFit& a) {
  auto kern = fit_kernel<SF_P, CH, TL, SF_SLOTS>;
  constexpr int tpb = threads_per_block<SF_SLOTS>();
  constexpr int groups_per_block = SF_SLOTS >= 8 ? 1 : (tpb / 32) * (32 / (8 * SF_SLOTS));
  constexpr size_t smem = sizeof(Smem<SF_P, CH, TL, SF_SLOTS>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, tpb, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)per_sm * a.sm_count;
  const int64_t need = (a.count + groups_per_block - 1) / groups_per_block;
  if (blocks > need) blocks = need;
  if (blocks < 1) return cudaSuccess;
  kern<<<(unsigned)blocks, tpb, smem, a.stream>>>(a.images, a.inits, a.count, a.geom, a.cfg, a.out);
  return cudaGetLastError();
}

template <int CH, int TL>
cudaError_t go_eval(const LaunchEval& a) {
  auto kern = eval_kernel<SF_P, CH, TL, SF_SLOTS>;
  constexpr int tpb = threads_per_block<SF_SLOTS>();
  constexpr int groups_per_block = SF_SLOTS >= 8 ? 1 : (tpb / 32) * (32 / (8 * SF_SLOTS));
  constexpr size_t smem = sizeof(Smem<SF_P, CH, TL, SF_SLOTS>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t blocks = (a.count + groups_per_block - 1) / groups_per_block;
  if (blocks < 1) return cudaSuccess;
  kern<<<(unsigned)blocks, tpb, smem, a.stream>>>(a.images, a.params, a.count, a.geom, a.out);
  return cudaGetLastError();
}

struct Pick {
  int ch = -1, tl = -1;
};

Pick pick(int ch_need, int tl_need) {
  Pick best;
  int cost = 1 << 30;
#define SF_CONSIDER(C, T)                                             \
  if ((C) >= ch_need && (T) >= tl_need && (C) + (T) < cost) {          \
    cost = (C) + (T);                                                 \
    best.ch = (C);                                                    \
    best.tl = (T);                                                    \
  }
  SF_SHAPES(SF_CONSIDER)
#undef SF_CONSIDER
  return best;
}
}  // namespace

int SF_UNIT_NAME(launch_fit, SF_P, SF_SLOTS)(int ch_need, int tl_need, const LaunchFit& a, cudaError_t* err) {
  const Pick p = pick(ch_need, tl_need);
#define SF_GO(C, T)                 \
  if (p.ch == (C) && p.tl == (T)) { \
    *err = go_fit<C, T>(a);         \
    return (C) * 16 + (T);          \
  }
  SF_SHAPES(SF_GO)
#undef SF_GO
  return -1;
}

int SF_UNIT_NAME(launch_eval, SF_P, SF_SLOTS)(int ch_need, int tl_need, const LaunchEval& a, cudaError_t* err) {
  const Pick p = pick(ch_need, tl_need);
#define SF_GO(C, T)                 \
  if (p.ch == (C) && p.tl == (T)) { \
    *err = go_eval<C, T>(a);        \
    return (C) * 16 + (T);          \
  }
  SF_SHAPES(SF_GO)
#undef SF_GO
  return -1;
}

}  // namespace sf
