// sf_sim.cpp -- synthetic spot generator (protocol
// PAPER.md:206-208), host side.  Counter-based Philox4x32-10 keyed by the
// 64-bit seed with the spot index in the counter, so every
// index regenerates alone and parallel generation is order-independent.
// Compiled with -ffp-contract=off so tests/test_simulator.py can restate it
// in Python bit-for-bit.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "spotfit.h"

namespace {

inline void mulhilo(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
  const uint64_t p = (uint64_t)a * (uint64_t)b;
  hi = (uint32_t)(p >> 32);
  lo = (uint32_t)p;
}

void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo(0xD2511F53u, c[0], hi0, lo0);
    mulhilo(0xCD9E8D57u, c[2], hi1, lo1);
    const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}

constexpr uint32_t kTag = 0x53504F54u;  // "SPOT"
constexpr double kTwoPi = 6.283185307179586;

inline void block_uniforms(uint64_t seed, int64_t index, uint32_t blk, double u[4]) {
  uint32_t c[4] = {(uint32_t)index, (uint32_t)((uint64_t)index >> 32), blk, kTag};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  for (int i = 0; i < 4; ++i) u[i] = ((double)c[i] + 0.5) * 2.3283064365386963e-10;  // (x + 0.5) 2^-32
}

inline void box_muller(double u1, double u2, double& z1, double& z2) {
  const double r = std::sqrt(-2.0 * std::log(u1));
  const double t = kTwoPi * u2;
  z1 = r * std::cos(t);
  z2 = r * std::sin(t);
}

void sim_one(const sf_sim_config& c, int W, int H, int64_t index, float* img, float* truth) {
  double u[4], z[4];
  block_uniforms(c.seed, index, 0u, u);
  box_muller(u[0], u[1], z[0], z[1]);
  const double spx = c.spread > 0 ? c.spread : W / 20.0;
  const double spy = c.spread > 0 ? c.spread : H / 20.0;
  const double cx = (W - 1) / 2.0 + z[0] * spx;
  const double cy = (H - 1) / 2.0 + z[1] * spy;
  const double sx = c.sigma_lo + (c.sigma_hi - c.sigma_lo) * u[2];
  const double sy = c.model == 4 ? c.sigma_lo + (c.sigma_hi - c.sigma_lo) * u[3] : sx;
  const double alpha = c.n_signal / (kTwoPi * sx * sy);
  const double beta = c.n_background / (double)(W * H);
  const int N = W * H;
  for (int i = 0; i < N; ++i) {
    if ((i & 3) == 0) {
      block_uniforms(c.seed, index, 1u + (uint32_t)(i >> 2), u);
      box_muller(u[0], u[1], z[0], z[1]);
      box_muller(u[2], u[3], z[2], z[3]);
    }
    const double dx = (i % W) - cx, dy = (i / W) - cy;
    const double lam = alpha * std::exp(-(dx * dx / (2.0 * sx * sx) + dy * dy / (2.0 * sy * sy))) + beta;
    double v = c.noise ? lam + z[i & 3] * std::sqrt(lam) : lam;
    if (c.rounding) v = std::round(v);  // half away from zero
    if (c.noise) v = std::max(0.0, v);
    img[i] = (float)v;
  }
  if (truth) {
    int k = 0;
    truth[k++] = (float)cx;
    truth[k++] = (float)cy;
    truth[k++] = (float)sx;
    if (c.model == 4) truth[k++] = (float)sy;
    truth[k++] = (float)alpha;
    truth[k++] = (float)beta;
  }
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
