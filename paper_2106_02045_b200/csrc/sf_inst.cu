// sf_inst.cu -- one template-instantiation unit per (SF_P, SF_SLOTS); the
// build compiles this file once per pair (paper_2106_02045_b200/build.py).
// Chain / tail pixel counts are uniform runtime loop bounds (Geom::ch, tl), so
// one kernel per (P, SLOTS) serves every grid with that pairwise-tree depth.
#include "sf_launch.h"
#if (SF_P == 3 || SF_P == 4) && (SF_SLOTS == 2 || SF_SLOTS == 4 || SF_SLOTS == 8)
#define SF_HAS_FIT2L 1
#include <cstdlib>

#include "sf_fit2l.cuh"
#endif

#ifndef SF_P
#error "compile with -DSF_P=3|4 -DSF_SLOTS=1|2|4|8|16"
#endif

#include <mutex>
#include <vector>

#define SF_CAT5(a, b, c, d, e) a##b##c##d##e
#define SF_UNIT_NAME(kind, P, S) SF_CAT5(kind, _P, P, _S, S)

namespace sf {

// Launch setup done once per (kernel, device, shared-memory size) instead of on every launch --
// small batches are latency-bound, and these are driver calls: the dynamic shared-memory attribute
// (raised to the largest size seen for the kernel on the device, so it always covers smem) and the
// occupancy query (query = false skips it).
static cudaError_t prepare_kernel(const void* kern, int tpb, size_t smem, int* per_sm, bool query,
                                  bool max_carveout = false) {
  struct Attr {
    const void* kern;
    int dev;
    size_t max_smem;
  };
  struct Occ {
    const void* kern;
    int dev;
    size_t smem;
    int per_sm;
  };
  static std::mutex mu;
  static std::vector<Attr> attrs;
  static std::vector<Occ> occs;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  Attr* at = nullptr;
  for (Attr& x : attrs)
    if (x.kern == kern && x.dev == dev) at = &x;
  if (at == nullptr || at->max_smem < smem) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    if (max_carveout) {  // all of L1 as shared memory (the two-leaf kernel's 4 x 54 KB); the general
                         // kernel keeps the driver's choice (its explicit-5 spills want L1)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
      if (e != cudaSuccess) return e;
    }
    if (at == nullptr)
      attrs.push_back(Attr{kern, dev, smem});
    else
      at->max_smem = smem;
  }
  *per_sm = 1;
  if (!query) return cudaSuccess;
  for (const Occ& x : occs)
    if (x.kern == kern && x.dev == dev && x.smem == smem) {
      *per_sm = x.per_sm;
      return cudaSuccess;
    }
  int n = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, tpb, smem);
  if (e != cudaSuccess) return e;
  occs.push_back(Occ{kern, dev, smem, n});
  *per_sm = n;
  return cudaSuccess;
}

#ifdef SF_HAS_FIT2L
// Spots of 2, 4 or 8 leaves with given inits (float or 16-bit pixels; symmetric or elliptical): the
// two-leaves-per-lane kernel with its profile cache in Tensor Memory (sf_fit2l.cuh), when its
// shared memory leaves room for its CTAs per SM (4 for P = 3, 3 for P = 4).  SPOTFIT_FIT2L=0 selects
// the general kernel.
template <typename PX>
static int launch_fit2l(const LaunchFit& a, const PX* images, cudaError_t* err) {
  auto kern = a.geom.full ? fit_kernel2l<SF_SLOTS, SF_P, true, PX> : fit_kernel2l<SF_SLOTS, SF_P, false, PX>;
  const size_t smem = l2::Smem<SF_SLOTS, SF_P>::bytes(a.geom.ch, a.geom.tl, a.geom.N);
  int unused = 0;
  *err = prepare_kernel((const void*)kern, l2::TPB, smem, &unused, false, true);
  if (*err != cudaSuccess) return 0;
  // TMEM: 512 columns per SM.  The occupancy API reports 1 CTA per SM for this kernel (it uses
  // tcgen05); registers (launch bound), shared memory (use_fit2l) and TMEM (128 columns) all allow
  // minb2l CTAs.
  const int per_sm = minb2l<SF_P>();
  constexpr int GPB = l2::groups_per_cta<SF_SLOTS>();
  int64_t blocks = (int64_t)per_sm * a.sm_count;
  const int64_t need = (a.count + GPB - 1) / GPB;
  if (blocks > need) blocks = need;
  if (blocks < 1) return 0;
  kern<<<(unsigned)blocks, l2::TPB, smem, a.stream>>>(images, a.inits, a.count, a.geom, a.cfg, a.out);
  *err = cudaGetLastError();
  return (int)blocks;
}

#ifndef SF_FIT2L_WAVES
#define SF_FIT2L_WAVES 1
#endif
static bool use_fit2l(const LaunchFit& a) {
  // SPOTFIT_FIT2L: 0 = never, 1 (default) = from one full wave upward, 2 = always (validation)
  static const int mode = [] {
    const char* e = std::getenv("SPOTFIT_FIT2L");
    return e ? (int)std::strtol(e, nullptr, 10) : 1;
  }();
  const bool on = mode > 0;
  // A batch smaller than one full wave of the kernel (every group of every CTA busy) finishes faster
  // on the general kernel, whose spots walk both leaves in parallel lanes (lower latency per spot):
  // the two-leaf kernel pays off when spots queue up.
  const int64_t wave = (int64_t)a.sm_count * minb2l<SF_P>() * l2::groups_per_cta<SF_SLOTS>() * SF_FIT2L_WAVES;
  return on && a.inits != nullptr && (a.count >= wave || mode >= 2) && a.geom.ch <= 2 * l2::kMaxPairs &&
         l2::Smem<SF_SLOTS, SF_P>::bytes(a.geom.ch, a.geom.tl, a.geom.N) + 1024 <= (size_t)228 * 1024 / minb2l<SF_P>();
}
#endif

template <typename PX>
static int launch_fit_px(const LaunchFit& a, const PX* images, cudaError_t* err) {
#ifdef SF_HAS_FIT2L
  if (use_fit2l(a)) return launch_fit2l<PX>(a, images, err);
#endif
  const bool fused = a.inits == nullptr;
  auto kern = a.geom.full ? (fused ? fit_kernel<SF_P, SF_SLOTS, true, PX, true> : fit_kernel<SF_P, SF_SLOTS, true, PX, false>)
                          : (fused ? fit_kernel<SF_P, SF_SLOTS, false, PX, true> : fit_kernel<SF_P, SF_SLOTS, false, PX, false>);
  constexpr int tpb = threads_per_block<SF_SLOTS>();
  constexpr int groups_per_block = SF_SLOTS >= 8 ? 1 : (tpb / 32) * (32 / (8 * SF_SLOTS));
  const size_t smem = Smem<SF_P, SF_SLOTS>::bytes(a.geom.ch, a.geom.tl, a.geom.N);
  int per_sm = 0;
  *err = prepare_kernel((const void*)kern, tpb, smem, &per_sm, true);
  if (*err != cudaSuccess) return 0;
  if (per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)per_sm * a.sm_count;
  const int64_t need = (a.count + groups_per_block - 1) / groups_per_block;
  if (blocks > need) blocks = need;
  if (blocks < 1) return 0;
  kern<<<(unsigned)blocks, tpb, smem, a.stream>>>(images, a.inits, a.count, a.geom, a.cfg, a.out);
  *err = cudaGetLastError();
  return (int)blocks;
}

int SF_UNIT_NAME(launch_fit, SF_P, SF_SLOTS)(const LaunchFit& a, cudaError_t* err) {
  return a.images16 ? launch_fit_px<uint16_t>(a, a.images16, err) : launch_fit_px<float>(a, a.images, err);
}

#if SF_P != 5  // model-level evaluation exists for the implicit models only
int SF_UNIT_NAME(launch_eval, SF_P, SF_SLOTS)(const LaunchEval& a, cudaError_t* err) {
  auto kern = a.geom.full ? eval_kernel<SF_P, SF_SLOTS, true> : eval_kernel<SF_P, SF_SLOTS, false>;
  constexpr int tpb = threads_per_block<SF_SLOTS>();
  constexpr int groups_per_block = SF_SLOTS >= 8 ? 1 : (tpb / 32) * (32 / (8 * SF_SLOTS));
  const size_t smem = Smem<SF_P, SF_SLOTS>::bytes(a.geom.ch, a.geom.tl, a.geom.N);
  *err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (*err != cudaSuccess) return 0;
  const int64_t blocks = (a.count + groups_per_block - 1) / groups_per_block;
  if (blocks < 1) return 0;
  kern<<<(unsigned)blocks, tpb, smem, a.stream>>>(a.images, a.params, a.count, a.geom, a.out);
  *err = cudaGetLastError();
  return (int)blocks;
}
#endif

}  // namespace sf
