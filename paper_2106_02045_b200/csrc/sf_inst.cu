// sf_inst.cu -- one template-instantiation unit per (SF_P, SF_SLOTS); the
// build compiles this file once per pair (paper_2106_02045_b200/build.py) so
// the heavy, fully unrolled kernels compile in parallel.
//
// PPL (pixels per chain lane) instantiations per slot count are chosen so the
// benchmark shapes hit an exact fit: 11x11 -> (1, 16), 15x15 -> (2, 15),
// 21x21 -> (4, 15), 32x32 -> (8, 16); every other N <= 1024 uses the smallest
// PPL >= its need (predicated-off pixels cost issue slots, not correctness).
#include "sf_launch.h"

#ifndef SF_P
#error "compile with -DSF_P=3|4 -DSF_SLOTS=1|2|4|8|16"
#endif

#if SF_SLOTS == 1
#define SF_PPL_LIST(X) X(2) X(4) X(8) X(11) X(16) X(22)
#elif SF_SLOTS == 2
#define SF_PPL_LIST(X) X(9) X(12) X(15) X(16) X(22)
#elif SF_SLOTS == 4
#define SF_PPL_LIST(X) X(10) X(13) X(15) X(19) X(22)
#elif SF_SLOTS == 8
#define SF_PPL_LIST(X) X(9) X(11) X(13) X(15) X(16) X(18) X(22)
#elif SF_SLOTS == 16
#define SF_PPL_LIST(X) X(16)
#endif

#define SF_CAT3(a, b, c, d, e) a##b##c##d##e
#define SF_UNIT_NAME(kind, P, S) SF_CAT3(kind, _P, P, _S, S)

namespace sf {

namespace {
template <int PPL>
cudaError_t go_fit(const LaunchFit& a) {
  auto kern = fit_kernel<SF_P, PPL, SF_SLOTS>;
  constexpr int tpb = threads_per_block<SF_SLOTS>();
  constexpr int groups_per_block = SF_SLOTS >= 8 ? 1 : (tpb / 32) * (32 / (8 * SF_SLOTS));
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, tpb, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)per_sm * a.sm_count;
  const int64_t need = (a.count + groups_per_block - 1) / groups_per_block;
  if (blocks > need) blocks = need;
  if (blocks < 1) return cudaSuccess;
  kern<<<(unsigned)blocks, tpb, 0, a.stream>>>(a.images, a.inits, a.count, a.geom, a.cfg, a.out);
  return cudaGetLastError();
}

template <int PPL>
cudaError_t go_eval(const LaunchEval& a) {
  constexpr int tpb = threads_per_block<SF_SLOTS>();
  constexpr int groups_per_block = SF_SLOTS >= 8 ? 1 : (tpb / 32) * (32 / (8 * SF_SLOTS));
  const int64_t blocks = (a.count + groups_per_block - 1) / groups_per_block;
  if (blocks < 1) return cudaSuccess;
  eval_kernel<SF_P, PPL, SF_SLOTS><<<(unsigned)blocks, tpb, 0, a.stream>>>(a.images, a.params, a.count, a.geom, a.out);
  return cudaGetLastError();
}
}  // namespace

int SF_UNIT_NAME(launch_fit, SF_P, SF_SLOTS)(int ppl_needed, const LaunchFit& a, cudaError_t* err) {
#define SF_TRY(X)                  \
  if (ppl_needed <= X) {           \
    *err = go_fit<X>(a);           \
    return X;                      \
  }
  SF_PPL_LIST(SF_TRY)
#undef SF_TRY
  return -1;
}

int SF_UNIT_NAME(launch_eval, SF_P, SF_SLOTS)(int ppl_needed, const LaunchEval& a, cudaError_t* err) {
#define SF_TRY(X)                  \
  if (ppl_needed <= X) {           \
    *err = go_eval<X>(a);          \
    return X;                      \
  }
  SF_PPL_LIST(SF_TRY)
#undef SF_TRY
  return -1;
}

}  // namespace sf
