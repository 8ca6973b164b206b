// sf_sim_core.h -- the synthetic-spot generator shared by the host
// (sf_sim.cpp) and device (sf_sim.cu) simulators (SPEC.md:316-368,
// PAPER.md:206-208).  Counter-based Philox4x32-10 keyed by the 64-bit seed,
// counter = (index lo, index hi, block, "SPOT"), so any spot regenerates alone
// and generation order / thread count never matters.
//
// Draws per spot: block 0 -> Box-Muller(u0, u1) = centre offsets, u2 = sigma
// (u3 = sigma_y for the elliptical model); block 1 + i/4 -> two Box-Muller
// pairs = the noise normals of pixels 4k..4k+3.
#pragma once
#include <cmath>
#include <cstdint>

#include "spotfit.h"

#ifdef __CUDACC__
#define SF_HD __host__ __device__ __forceinline__
#else
#define SF_HD inline
#endif

namespace sfsim {

SF_HD void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
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

SF_HD void block_uniforms(uint64_t seed, int64_t index, uint32_t blk, double u[4]) {
  uint32_t c[4] = {(uint32_t)index, (uint32_t)((uint64_t)index >> 32), blk, kTag};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  for (int i = 0; i < 4; ++i) u[i] = ((double)c[i] + 0.5) * 2.3283064365386963e-10;  // (x + 0.5) 2^-32
}

SF_HD void box_muller(double u1, double u2, double& z1, double& z2) {
  const double r = sqrt(-2.0 * log(u1));
  const double t = kTwoPi * u2;
  z1 = r * cos(t);
  z2 = r * sin(t);
}

struct SpotTruth {
  double cx, cy, sx, sy, alpha, beta;
};

SF_HD SpotTruth spot_truth(const sf_sim_config& c, int W, int H, int64_t index) {
  double u[4], z0, z1;
  block_uniforms(c.seed, index, 0u, u);
  box_muller(u[0], u[1], z0, z1);
  const double spx = c.spread > 0 ? c.spread : W / 20.0;
  const double spy = c.spread > 0 ? c.spread : H / 20.0;
  SpotTruth t;
  t.cx = (W - 1) / 2.0 + z0 * spx;
  t.cy = (H - 1) / 2.0 + z1 * spy;
  t.sx = c.sigma_lo + (c.sigma_hi - c.sigma_lo) * u[2];
  t.sy = c.model == 4 ? c.sigma_lo + (c.sigma_hi - c.sigma_lo) * u[3] : t.sx;
  t.alpha = c.n_signal / (kTwoPi * t.sx * t.sy);
  t.beta = c.n_background / (double)(W * H);
  return t;
}

// pixel i of spot `index` given its truth and the 4 noise normals of block 1 + i/4
SF_HD float pixel_value(const sf_sim_config& c, const SpotTruth& t, int W, int i, double z) {
  const double dx = (i % W) - t.cx, dy = (i / W) - t.cy;
  const double lam = t.alpha * exp(-(dx * dx / (2.0 * t.sx * t.sx) + dy * dy / (2.0 * t.sy * t.sy))) + t.beta;
  double v = c.noise ? lam + z * sqrt(lam) : lam;
  if (c.rounding) v = round(v);  // half away from zero
  if (c.noise) v = v <= 0.0 ? 0.0 : v;  // clamp at +0 (also maps round()'s -0.0 to +0.0)
  return (float)v;
}

SF_HD void pixel_normals(const sf_sim_config& c, int64_t index, int i, double z[4]) {
  double u[4];
  block_uniforms(c.seed, index, 1u + (uint32_t)(i >> 2), u);
  box_muller(u[0], u[1], z[0], z[1]);
  box_muller(u[2], u[3], z[2], z[3]);
}

SF_HD void write_truth(const sf_sim_config& c, const SpotTruth& t, float* truth) {
  int k = 0;
  truth[k++] = (float)t.cx;
  truth[k++] = (float)t.cy;
  truth[k++] = (float)t.sx;
  if (c.model == 4) truth[k++] = (float)t.sy;
  truth[k++] = (float)t.alpha;
  truth[k++] = (float)t.beta;
}

}  // namespace sfsim
