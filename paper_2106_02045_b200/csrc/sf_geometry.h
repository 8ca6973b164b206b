// sf_geometry.h -- host-side lane geometry: numpy's pairwise-sum tree for an
// N-pixel spot mapped onto chain lanes.  Pure C++, no CUDA.
#pragma once
#include <algorithm>
#include <cstring>
#include <vector>

#include "sf_device.cuh"

namespace sf {

struct Leaf {
  int start, m, slot;
};

inline int pw_depth(int n) {
  if (n <= 128) return 0;
  int n2 = n / 2;
  n2 -= n2 % 8;
  return 1 + std::max(pw_depth(n2), pw_depth(n - n2));
}

// numpy pairwise recursion (n2 = n/2 - (n/2)%8, leaves <= 128); each leaf goes
// to the leftmost slot of its subtree in the complete tree of depth pw_depth.
inline void pw_place(int n, int start, int slot, int span, std::vector<Leaf>& out) {
  if (n <= 128) {
    out.push_back({start, n, slot});
    return;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  pw_place(n2, start, slot, span / 2, out);
  pw_place(n - n2, start + n2, slot + span / 2, span / 2, out);
}

// Fills g; returns the pixels-per-lane requirement and, through ch_need /
// tl_need, the largest chain and tail pixel counts of any lane.  N in [1, 1024].
inline int build_geom(int W, int H, int P, Geom& g, int* ch_need = nullptr, int* tl_need = nullptr) {
  std::memset(&g, 0, sizeof(g));
  g.W = W;
  g.H = H;
  g.N = W * H;
  g.P = P;
  const int D = pw_depth(g.N);
  g.slots = 1 << D;
  g.lanes = 8 * g.slots;
  std::vector<Leaf> leaves;
  pw_place(g.N, 0, 0, g.slots, leaves);
  int ppl = 1, chn = 0, tln = 0;
  for (const Leaf& L : leaves) {
    const int nc = L.m >= 8 ? L.m / 8 : 0;
    const int nt = L.m >= 8 ? L.m % 8 : L.m;
    for (int k = 0; k < 8; ++k) {
      const int lane = L.slot * 8 + k;
      g.nc[lane] = (int16_t)nc;
      g.nt[lane] = (int16_t)nt;
      g.base[lane] = (int16_t)(L.start + k);
      g.tbase[lane] = (int16_t)(L.start + 8 * nc);
    }
    ppl = std::max(ppl, nc + nt);
    chn = std::max(chn, nc);
    tln = std::max(tln, nt);
  }
  g.ch = chn;
  g.tl = tln;
  g.full = 1;
  for (int l = 0; l < g.lanes; ++l) g.full = g.full && g.nc[l] == chn;
  g.nz2 = 0x8000000080000000ull;
  if (ch_need) *ch_need = chn;
  if (tl_need) *tl_need = tln;
  return ppl;
}

}  // namespace sf
