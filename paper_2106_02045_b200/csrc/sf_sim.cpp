// sf_sim.cpp -- host simulator over the shared generator in
// sf_sim_core.h; compiled with -ffp-contract=off.  Host threads take
// contiguous index ranges; output is independent of the thread count.
#include <algorithm>
#include <thread>
#include <vector>

#include "sf_sim_core.h"

namespace {

void sim_one(const sf_sim_config& c, int W, int H, int64_t index, float* img, float* truth) {
  const sfsim::SpotTruth t = sfsim::spot_truth(c, W, H, index);
  const int N = W * H;
  double z[4];
  for (int i = 0; i < N; ++i) {
    if ((i & 3) == 0) sfsim::pixel_normals(c, index, i, z);
    img[i] = sfsim::pixel_value(c, t, W, i, z[i & 3]);
  }
  if (truth) sfsim::write_truth(c, t, truth);
}

}  // namespace

extern "C" int sf_simulate_host(const sf_sim_config* cfg, int32_t width, int32_t height, int64_t first_index,
                                int64_t count, float* images, float* truth, int32_t threads) {
  if (!cfg || width < 1 || height < 1 || (int64_t)width * height > 1024 || count < 0) return -1;
  if (cfg->model != 3 && cfg->model != 4) return -1;
  if (count == 0) return 0;
  const int N = width * height, T = cfg->model + 2;
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = (int)std::min<int64_t>(nt, std::max<int64_t>(1, count / 64));
  auto work = [&](int t) {
    const int64_t lo = count * t / nt, hi = count * (t + 1) / nt;
    for (int64_t s = lo; s < hi; ++s)
      sim_one(*cfg, width, height, first_index + s, images + s * N, truth ? truth + s * T : nullptr);
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  return 0;
}
