// sf_fit2l.cuh -- the two-leaves-per-lane fit kernel for symmetric spots of 129..1024 pixels (2, 4
// or 8 leaves: SL), with the per-pixel profile cache in Tensor Memory.  The text below describes the
// two-leaf case (the 15x15 headline); with SL leaves a spot takes 4 SL lanes (one octet of lanes per
// pair of leaves), and the octets' pair sums are combined in numpy's slot-tree order by shuffles.
//
// The general kernel (sf_fit_kernel.cuh) gives each chain of the tree its own lane, so a two-leaf
// spot takes 16 lanes and a warp fits two spots; every warp-level step that is not a pixel loop
// (the amplitude and coefficient-gradient divisions, the LM decision, the damped f64 solve, the
// refill bookkeeping) then serves two spots.  Here a lane owns chain k of BOTH leaves (virtual
// lanes k and 8 + k of the same geometry), so a spot takes 8 lanes and a warp fits four: the
// pixel work per spot is unchanged, the per-warp scalar work is shared by twice the spots.  The
// lane walks its two chains one after the other with the same accumulators, parking leaf 0's
// chain sums in shared memory; the reduction then combines each leaf in numpy's order, adds its
// tail, and adds the two leaves (the depth-1 slot tree) -- the same operations in the same order
// as reduce_group, so every sum is bit-identical.
//
// Twice the spots per warp need twice the per-pixel cache per warp: f and its three partials of
// every chain pixel pair (32 B per pair and lane) live in Tensor Memory -- 2 leaves x <= 8 pairs x
// 8 columns = 128 TMEM columns per 128-thread CTA, written with tcgen05.st (pass 1) and read back
// with tcgen05.ld (pass 2) -- so shared memory keeps only the pixel values, coordinates, staging
// windows and reduction scratch, and four CTAs (16 warps, 64 spots) fit an SM as before.
#pragma once
#include "sf_fit_kernel.cuh"

#ifndef SF_2L_U1
#define SF_2L_U1 1  // pass-1 pair loop unroll (A/B knob)
#endif
#ifndef SF_2L_U2
#define SF_2L_U2 1  // pass-2 pair loop unroll (A/B knob)
#endif
#define SF_STR_(x) #x
#define SF_UNROLL(n) _Pragma(SF_STR_(unroll n))

namespace sf {
namespace l2 {

constexpr int TPB = 128;   // 4 warps
// SL leaves per spot: 4 SL lanes per group, 8 / SL groups per warp, 32 / SL per CTA
template <int SL>
__host__ __device__ constexpr int lanes_per_group() { return 4 * SL; }
template <int SL>
__host__ __device__ constexpr int groups_per_cta() { return 4 * (8 / SL); }
constexpr int kCols = 128; // TMEM columns per CTA
constexpr int kTS = 34;    // scratch row stride in doubles (32 lanes + a 2-double bank skew)
constexpr int kMaxPairs = 8;
// per model P (3: x, y, sigma; 4: x, y, sigma_x, sigma_y)
template <int P>
__host__ __device__ constexpr int q1_of() { return 3 + 3 * P; }             // pass-1 quantities
template <int P>
__host__ __device__ constexpr int q2_of() { return 1 + P + P * (P + 1) / 2; }  // pass-2 quantities
template <int P>
__host__ __device__ constexpr int qa_of() { return q1_of<P>() > q2_of<P>() ? q1_of<P>() : q2_of<P>(); }
template <int P>
__host__ __device__ constexpr int sysq_of() { return ((P * (P + 1) / 2 + P) + 1) & ~1; }  // saved JtJ + rhs

template <int SL, int P = 3>
struct Smem {
  static constexpr int GPB = groups_per_cta<SL>();
  static constexpr int VL = 8 * SL;              // virtual lanes (coordinate table width)
  static constexpr bool kGen = SL >= 8;          // coordinates generated in registers (no table)
  static constexpr int kQA = qa_of<P>();         // parked rows: one leaf's chain sums
  static constexpr int kSysQ = sysq_of<P>();
  double* sys;   // [GPB][kSysQ]
  double* kc;    // [2]: ddiv_rcp(lam_down), ddiv_rcp(N - 5)
  double* park;  // [4 warps][kQA][kTS]: one leaf's chain sums
  double* res;   // [4 warps][2][4 octets][kQA]: leaf-0 sums, then the pair sums
  float* tbuf;   // [4 warps][4 octets][kQA]: tail terms of one tail slot
  float2* g;     // [2][np][TPB]: pixel values of chain slot pairs (0 where not owned)
  float2* f3;    // [2][np][TPB]: P = 4: df/dsigma_y of the pair (the other 8 floats are in TMEM)
  float4* xy;    // [np][VL]: pair coordinates (x_A, x_B, y_A, y_B) per virtual lane (not when kGen)
  float4* sfq;   // [2][ns][TPB]: solo slots (odd last chain slot, tails): f, df/dp0, df/dp1, df/dp2
  float* sf3;    // [2][ns][TPB]: P = 4: solo df/dp3
  float* sg;     // [2][ns][TPB]: solo pixel values
  float2* sxy;   // [ns][VL]: solo coordinates (not when kGen)
  float* stage;  // [GPB][sw]: next-spot staging windows
  int np, ns, sw;

  static __host__ __device__ int stage_floats(int N) { return (N + 6) & ~3; }
  static __host__ __device__ size_t bytes(int ch, int tl, int N) {
    const int np = ch / 2, ns = (ch & 1) + tl;
    return (size_t)GPB * kSysQ * 8 + 16 + (size_t)4 * kQA * kTS * 8 + (size_t)4 * 2 * 4 * kQA * 8 +
           (size_t)4 * 4 * kQA * 4 + (size_t)2 * np * TPB * 8 + (P == 4 ? (size_t)2 * np * TPB * 8 : 0) +
           (kGen ? 0 : (size_t)np * VL * 16) + (size_t)2 * ns * TPB * 16 + (P == 4 ? (size_t)2 * ns * TPB * 4 : 0) +
           (size_t)2 * ns * TPB * 4 + (kGen ? 0 : (size_t)ns * VL * 8) + (size_t)GPB * stage_floats(N) * 4 + 64;
  }
  __device__ __forceinline__ void bind(unsigned char* raw, int ch, int tl, int N) {
    np = ch / 2;
    ns = (ch & 1) + tl;
    sw = stage_floats(N);
    unsigned char* p = raw;
    sys = reinterpret_cast<double*>(p);
    p += (size_t)GPB * kSysQ * 8;
    kc = reinterpret_cast<double*>(p);
    p += 16;
    park = reinterpret_cast<double*>(p);
    p += (size_t)4 * kQA * kTS * 8;
    res = reinterpret_cast<double*>(p);
    p += (size_t)4 * 2 * 4 * kQA * 8;
    tbuf = reinterpret_cast<float*>(p);
    p += (size_t)4 * 4 * kQA * 4;
    g = reinterpret_cast<float2*>(p);
    p += (size_t)2 * np * TPB * 8;
    f3 = reinterpret_cast<float2*>(p);
    p += P == 4 ? (size_t)2 * np * TPB * 8 : 0;
    xy = reinterpret_cast<float4*>(p);
    p += kGen ? 0 : (size_t)np * VL * 16;
    sfq = reinterpret_cast<float4*>(p);
    p += (size_t)2 * ns * TPB * 16;
    sf3 = reinterpret_cast<float*>(p);
    p += P == 4 ? (size_t)2 * ns * TPB * 4 : 0;
    sg = reinterpret_cast<float*>(p);
    p += (size_t)2 * ns * TPB * 4;
    sxy = reinterpret_cast<float2*>(p);
    p += kGen ? 0 : (size_t)ns * VL * 8;
    stage = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p) + 15) & ~(uintptr_t)15);
  }
};

// ---- Tensor Memory: per-thread rows of the warp's lane quarter
__device__ __forceinline__ void tm_st8(uint32_t taddr, f2 a, f2 b, f2 c, f2 d) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
               "r"((uint32_t)a.v), "r"((uint32_t)(a.v >> 32)), "r"((uint32_t)b.v), "r"((uint32_t)(b.v >> 32)),
               "r"((uint32_t)c.v), "r"((uint32_t)(c.v >> 32)), "r"((uint32_t)d.v), "r"((uint32_t)(d.v >> 32))
               : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, f2& a, f2& b, f2& c, f2& d) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  a.v = (unsigned long long)r[0] | ((unsigned long long)r[1] << 32);
  b.v = (unsigned long long)r[2] | ((unsigned long long)r[3] << 32);
  c.v = (unsigned long long)r[4] | ((unsigned long long)r[5] << 32);
  d.v = (unsigned long long)r[6] | ((unsigned long long)r[7] << 32);
}
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// One thread's view: lane in group, its two virtual lanes' ownership and pixel bases.
struct Lane {
  int gl, gw, gib;  // lane in group, group in warp, group in CTA
  int vl0;          // virtual lane of leaf 0 (leaf 1: vl0 + 8): 16 * octet + chain
  float basef[2], tbasef[2], Wf, invW;  // coordinate generation (SL >= 8)
  uint32_t own[2];  // per virtual lane: bit j chain slot j < ch, bit ch + t tail t
  int base[2], tbase[2];
  int ch, tl;
  int tlv[2];       // tail pixels of each leaf (a leaf without tail skips its zero tail terms)
  uint32_t tw;      // TMEM address of this warp's lane quarter, column 0
};

// ---------------------------------------------------------------------------------- pass loops
// Coordinates of chain slot pair i (slots 2i, 2i+1): the table entry xyp, or generated in registers
// when SL >= 8 (sf_device.cuh:pair_xy: y = floor((idx + 0.5) / W) by the RNE magic number).
template <int SL, int P>
__device__ __forceinline__ void pair_xy2l(const float4* xyp, const Lane& L, int v, int i, f2 nz, f2& cx, f2& cy) {
  if constexpr (Smem<SL, P>::kGen) {
    const float iA = __fmaf_rn(16.0f, (float)i, v ? L.basef[1] : L.basef[0]);
    const f2 idx = pk2(iA, __fadd_rn(iA, 8.0f));
    const f2 t = mul2(add2(idx, bc2(0.5f)), bc2(L.invW), nz);
    cy = sub2(add2(sub2(t, bc2(0.5f)), bc2(12582912.0f)), bc2(12582912.0f));
    cx = fma2(bc2(-L.Wf), cy, idx);
  } else {
    const float4 c = *xyp;
    cx = pk2(c.x, c.y);
    cy = pk2(c.z, c.w);
  }
}
// Coordinates of solo slot j (j >= ch & ~1: the odd last chain slot or tail j - ch) of virtual lane vl.
template <int SL, int P>
__device__ __forceinline__ float2 solo_xy2l(const Smem<SL, P>& S, const Lane& L, int v, int vl, int j) {
  if constexpr (Smem<SL, P>::kGen) {
    const float idx = j < L.ch ? __fmaf_rn(8.0f, (float)j, v ? L.basef[1] : L.basef[0])
                               : __fadd_rn(v ? L.tbasef[1] : L.tbasef[0], (float)(j - L.ch));
    const float t = __fmul_rn(__fadd_rn(idx, 0.5f), L.invW);
    const float y = __fsub_rn(__fadd_rn(__fsub_rn(t, 0.5f), 12582912.0f), 12582912.0f);
    return make_float2(__fmaf_rn(-L.Wf, y, idx), y);
  } else {
    return S.sxy[(j - (L.ch & ~1)) * Smem<SL, P>::VL + vl];
  }
}

// solo slot cache (the odd last chain slot and the tails stay in shared memory)
template <int SL, int P>
__device__ __forceinline__ void store_solo(Smem<SL, P>& S, int r, float f, const float (&fg)[P]) {
  S.sfq[r * TPB + threadIdx.x] = make_float4(f, fg[0], fg[1], fg[2]);
  if constexpr (P == 4) S.sf3[r * TPB + threadIdx.x] = fg[3];
}
template <int SL, int P>
__device__ __forceinline__ void load_solo(const Smem<SL, P>& S, int r, float& f, float (&fg)[P]) {
  const float4 q = S.sfq[r * TPB + threadIdx.x];
  f = q.x;
  fg[0] = q.y;
  fg[1] = q.z;
  fg[2] = q.w;
  if constexpr (P == 4) fg[3] = S.sf3[r * TPB + threadIdx.x];
}

// Pass-1 chain loop of virtual lane v (leaf v): pair loop (profiles to TMEM; P = 4 keeps df/dp3 in
// shared memory), odd last slot.
template <int SL, int P, bool FULL, bool GT>
__device__ __forceinline__ void chain1_2l(Smem<SL, P>& S, const Lane& L, int v, const float (&pe)[P], float ix, float iy,
                                          unsigned long long nz2, double (&a1)[q1_of<P>()]) {
  constexpr int Q1 = q1_of<P>();
  const f2 nz{nz2};
  const f2 x0 = bc2(pe[0]), y0 = bc2(pe[1]), ix2 = bc2(ix), iy2 = bc2(iy);
  const int tid = threadIdx.x, vl = L.vl0 + 8 * v;
  const uint32_t own = v ? L.own[1] : L.own[0];
#pragma unroll
  for (int q = 0; q < Q1; ++q) a1[q] = 0.0;
  const float2* gp = S.g + v * S.np * TPB + tid;  // pair i: gp[TPB i]
  float2* f3p = S.f3 + v * S.np * TPB + tid;      // P = 4
  const float4* xyp = S.xy + vl;                  // pair i: xyp[VL i] (coordinate table)
  uint32_t tc = L.tw + (uint32_t)(v * S.np * 8);  // pair i: column tc + 8 i
  SF_UNROLL(SF_2L_U1)
  for (int i = 0; i < S.np; ++i, gp += TPB, f3p += TPB, tc += 8, xyp += Smem<SL, P>::VL) {
    f2 cx, cy, f, fg[P], t[Q1];
    pair_xy2l<SL, P>(xyp, L, v, i, nz, cx, cy);
    pixel_profile2<P, FULL>(cx, cy, x0, y0, ix2, iy2, nz, owns(own, 2 * i), owns(own, 2 * i + 1), f, fg);
    tm_st8(tc, f, fg[0], fg[1], fg[2]);
    if constexpr (P == 4) {
      float a, b;
      up2(fg[3], a, b);
      *f3p = make_float2(a, b);
    }
    const float2 g = *gp;
    pass1_terms2<P>(f, fg, pk2(g.x, g.y), nz, t);
    acc_pair2<Q1, P, 1, GT>(a1, t);
  }
  if (L.ch & 1) {  // odd chain length: last chain slot, scalar, cached in shared memory
    float f, fg[P], t[Q1];
    pixel_profile<P>(solo_xy2l<SL, P>(S, L, v, vl, L.ch - 1), pe, ix, iy, owns(own, L.ch - 1), f, fg);
    store_solo<SL, P>(S, v * S.ns, f, fg);
    pass1_terms<P>(f, fg, S.sg[(v * S.ns) * TPB + tid], t);
    acc1<Q1, P, 1>(a1, t, GT);
  }
  unscale<Q1, P, 1>(a1, GT);
}

// Pass-2 chain loop of virtual lane v (profiles from TMEM).
template <int SL, int P, bool FULL, bool T2>
__device__ __forceinline__ void chain2_2l(Smem<SL, P>& S, const Lane& L, int v, float a32, float b32,
                                          const float (&da)[P], const float (&db)[P], unsigned long long nz2,
                                          double (&a2)[q2_of<P>()]) {
  constexpr int Q2 = q2_of<P>();
  const f2 nz{nz2};
  const f2 a2p = bc2(a32), b2p = bc2(b32);
  f2 da2[P], db2[P];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    da2[k] = bc2(da[k]);
    db2[k] = bc2(db[k]);
  }
  const int tid = threadIdx.x;
  const uint32_t own = v ? L.own[1] : L.own[0];
#pragma unroll
  for (int q = 0; q < Q2; ++q) a2[q] = 0.0;
  const float2* gp = S.g + v * S.np * TPB + tid;
  const float2* f3p = S.f3 + v * S.np * TPB + tid;
  uint32_t tc = L.tw + (uint32_t)(v * S.np * 8);
  SF_UNROLL(SF_2L_U2)
  for (int i = 0; i < S.np; ++i, gp += TPB, f3p += TPB, tc += 8) {
    f2 f, fg[P], t[Q2];
    tm_ld8(tc, f, fg[0], fg[1], fg[2]);
    if constexpr (P == 4) {
      const float2 c = *f3p;
      fg[3] = pk2(c.x, c.y);
    }
    const float2 g = *gp;
    pass2_terms2<P, FULL>(f, fg, pk2(g.x, g.y), owns(own, 2 * i), owns(own, 2 * i + 1), a2p, b2p, da2, db2, nz, t);
    acc_pair2<Q2, P, 2, T2>(a2, t);
  }
  if (L.ch & 1) {
    float f, fg[P], t[Q2];
    load_solo<SL, P>(S, v * S.ns, f, fg);
    pass2_terms<P>(f, fg, S.sg[(v * S.ns) * TPB + tid], owns(own, L.ch - 1), a32, b32, da, db, t);
    acc1<Q2, P, 2>(a2, t, T2);
  }
  unscale<Q2, P, 2>(a2, T2);
}

// One leaf's sums of Q quantities in numpy's order (reduce_group's leaf step): the octet's 8 chain
// sums of quantity q combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the leaf's tail terms
// serially (tail(t, terms) fills the Q terms of tail slot t; they pass through the warp's tail
// buffer so that a lane reads only the terms of its quantities).  Lane l8 of an octet does
// quantities l8 and l8 + 8.  Leaf 0 (v = 0) leaves its sums in res; leaf 1 adds them (the octet's
// pair of leaves in the slot tree) and broadcasts into a[] of every lane of the octet; with one
// pair per group (SL = 2) numpy's outer 0.0 + is applied here, otherwise after the octets' tree.
// All 32 lanes of the warp call it.
template <int SL, int QA, int Q, class Tail>
__device__ __forceinline__ void combine_leaf(double (&a)[Q], double* pk, double* res, float* tb, int v, int tl,
                                             Tail&& tail) {
  const int lane = threadIdx.x & 31, l8 = lane & 7, g0 = lane & ~7, wo = lane >> 3;
#pragma unroll
  for (int q = 0; q < Q; ++q) pk[q * kTS + lane] = a[q];
  double sc[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (r == 1 && Q <= 8) break;
    const int q = l8 + 8 * r < Q ? l8 + 8 * r : Q - 1;
    __syncwarp();
    const double2* rp = reinterpret_cast<const double2*>(pk + q * kTS + g0);
    const double2 r01 = rp[0], r23 = rp[1], r45 = rp[2], r67 = rp[3];
    sc[r] = __dadd_rn(__dadd_rn(__dadd_rn(r01.x, r01.y), __dadd_rn(r23.x, r23.y)),
                      __dadd_rn(__dadd_rn(r45.x, r45.y), __dadd_rn(r67.x, r67.y)));
  }
#pragma unroll 1
  for (int t = 0; t < tl; ++t) {  // leaf tail, serial (numpy's pairwise remainder loop)
    float tt[Q];
    tail(t, tt);
    if (l8 == 0) {
#pragma unroll
      for (int q = 0; q < Q; ++q) tb[wo * QA + q] = tt[q];
    }
    __syncwarp();
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (r == 1 && Q <= 8) break;
      const int q = l8 + 8 * r < Q ? l8 + 8 * r : Q - 1;
      sc[r] = __dadd_rn(sc[r], (double)tb[wo * QA + q]);
    }
    __syncwarp();
  }
  double* r0 = res + wo * QA;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (r == 1 && Q <= 8) break;
    const int q = l8 + 8 * r;
    if (q < Q) {
      if (v == 0)
        r0[q] = sc[r];
      else if (SL == 2)  // the whole tree: leaf 0 + leaf 1, then numpy's outer 0.0 +
        r0[4 * QA + q] = __dadd_rn(0.0, __dadd_rn(r0[q], sc[r]));
      else  // this octet's pair of leaves; the slot tree continues across octets below
        r0[4 * QA + q] = __dadd_rn(r0[q], sc[r]);
    }
  }
  __syncwarp();
  if (v != 0) {
    if constexpr (Q % 2 == 0) {
      const double2* r2 = reinterpret_cast<const double2*>(r0 + 4 * QA);
#pragma unroll
      for (int k = 0; k < Q / 2; ++k) {
        const double2 t = r2[k];
        a[2 * k] = t.x;
        a[2 * k + 1] = t.y;
      }
    } else {
#pragma unroll
      for (int q = 0; q < Q; ++q) a[q] = r0[4 * QA + q];
    }
    if constexpr (SL >= 4) {  // slot tree over the group's octets (xor 8, then 16), then 0.0 +
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        a[q] = __dadd_rn(a[q], shfl_xor_d(a[q], 8));
        if constexpr (SL >= 8) a[q] = __dadd_rn(a[q], shfl_xor_d(a[q], 16));
        a[q] = __dadd_rn(0.0, a[q]);
      }
    }
    __syncwarp();
  }
}

// One fused evaluation (sf_device.cuh:evaluate, two leaves per lane).
template <int SL, int P, bool FULL>
__device__ __forceinline__ void evaluate2l(Smem<SL, P>& S, const Lane& L, double G, double n, const float (&pe)[P],
                                           bool gt, bool lane_g40, bool care, unsigned long long nz2, Eval<P>& E) {
  constexpr int Q1 = q1_of<P>(), Q2 = q2_of<P>(), QA = Smem<SL, P>::kQA, T = P * (P + 1) / 2;
  const int tid = threadIdx.x;
  double* pk = S.park + (size_t)(tid >> 5) * QA * kTS;
  const float ix = __frcp_rn(pe[2]);
  const float iy = (P == 4) ? __frcp_rn(pe[P - 1]) : ix;
  const int so0 = L.ch & 1;

  // ---- pass 1, leaf 0 then leaf 1 (profiles cached in TMEM), each leaf combined as it finishes
  double* res = S.res + (size_t)(tid >> 5) * 2 * 4 * QA;
  float* tbuf = S.tbuf + (size_t)(tid >> 5) * 4 * QA;
  double a1[Q1];
#pragma unroll 1
  for (int v = 0; v < 2; ++v) {
    if (gt)
      chain1_2l<SL, P, FULL, true>(S, L, v, pe, ix, iy, nz2, a1);
    else
      chain1_2l<SL, P, FULL, false>(S, L, v, pe, ix, iy, nz2, a1);
    const uint32_t own = v ? L.own[1] : L.own[0];
    const int tlv = v ? L.tlv[1] : L.tlv[0];  // (+0.0 terms of unowned tail slots leave the sums unchanged)
#pragma unroll 1
    for (int t = 0; t < tlv; ++t) {  // tail profiles (added after the 8-way combine)
      float f, fg[P];
      pixel_profile<P>(solo_xy2l<SL, P>(S, L, v, L.vl0 + 8 * v, L.ch + t), pe, ix, iy, owns(own, L.ch + t), f, fg);
      store_solo<SL, P>(S, v * S.ns + so0 + t, f, fg);
    }
    combine_leaf<SL, QA, Q1>(a1, pk, res, tbuf, v, tlv, [&](int t, float (&tt)[Q1]) {
      const int r = v * S.ns + so0 + t;
      float f, fg[P];
      load_solo<SL, P>(S, r, f, fg);
      pass1_terms<P>(f, fg, S.sg[r * TPB + tid], tt);
    });
  }

  // ---- alpha_beta (model.py:222-234) and coefficient gradients (270-288) on the group's lanes
  const double F = a1[0], FF = a1[1], FG = a1[2];
  const double denom = n * FF - F * F;
  E.singular = denom <= 1e-12 * n * FF;
  const int tb = (tid & 31) & ~(lanes_per_group<SL>() - 1);  // the group's lanes share the divisions
  const int k = (tid & 31) - tb;
  const double rden = ddiv_rcp(denom);
  {
    const double num = k == 1 ? G * FF - F * FG : n * FG - F * G;
    const float qf = (float)ddiv_with(num, denom, rden);
    E.alpha = __shfl_sync(kFull, qf, tb);
    E.beta = __shfl_sync(kFull, qf, tb + 1);
  }
  const float a32 = E.alpha, b32 = E.beta;
  float da[P], db[P];
  {
    const int kk = k < 2 * P ? k : 0;
    const int j = kk < P ? kk : kk - P;
    double dF = a1[3], S_ = a1[3 + P], dFG = a1[3 + 2 * P];
#pragma unroll
    for (int i = 1; i < P; ++i) {
      if (j == i) {
        dF = a1[3 + i];
        S_ = a1[3 + P + i];
        dFG = a1[3 + 2 * P + i];
      }
    }
    const double dFF = 2.0 * S_;
    const double gamma = n * dFF - 2.0 * F * dF;
    const double num = kk < P ? n * dFG - G * dF - (double)a32 * gamma : G * dFF - FG * dF - F * dFG - (double)b32 * gamma;
    const float qf = (float)ddiv_with(num, denom, rden);
#pragma unroll
    for (int i = 0; i < P; ++i) {
      da[i] = __shfl_sync(kFull, qf, tb + i);
      db[i] = __shfl_sync(kFull, qf, tb + P + i);
    }
  }

  // ---- pass 2 (sf_device.cuh:evaluate's tame vote and loops), leaf 0 then leaf 1
  bool ok = lane_g40 && fabsf(a32) <= 0x1p40f && fabsf(b32) <= 0x1p40f;
#pragma unroll
  for (int i = 0; i < P; ++i) ok = ok && fabsf(da[i]) <= 0x1p40f && fabsf(db[i]) <= 0x1p40f;
  const bool t2 = __all_sync(kFull, ok || !care);
  tm_wait_st();  // pass 1's TMEM stores have landed before pass 2 reads them
  double a2[Q2];
#pragma unroll 1
  for (int v = 0; v < 2; ++v) {
    if (t2)
      chain2_2l<SL, P, FULL, true>(S, L, v, a32, b32, da, db, nz2, a2);
    else
      chain2_2l<SL, P, FULL, false>(S, L, v, a32, b32, da, db, nz2, a2);
    const uint32_t own = v ? L.own[1] : L.own[0];
    const int tlv = v ? L.tlv[1] : L.tlv[0];
    combine_leaf<SL, QA, Q2>(a2, pk, res, tbuf, v, tlv, [&](int t, float (&tt)[Q2]) {
      const int r = v * S.ns + so0 + t;
      float f, fg[P];
      load_solo<SL, P>(S, r, f, fg);
      pass2_terms<P>(f, fg, S.sg[r * TPB + tid], owns(own, L.ch + t), a32, b32, da, db, tt);
    });
  }
  E.chi = (float)a2[0];
#pragma unroll
  for (int i = 0; i < P; ++i) E.rhs[i] = a2[1 + i];
#pragma unroll
  for (int m = 0; m < T; ++m) E.jtj[m] = a2[1 + P + m];
}

// Scatter the staged spot into both virtual lanes' pixel slots and sum G in numpy order
// (sf_device.cuh:load_spot); tameness flags as load_spot.
template <int SL, int P, bool FULL, typename PX>
__device__ __forceinline__ double load_spot2l(Smem<SL, P>& S, const Lane& L, const PX* st, bool load, bool& gt,
                                              bool& g40) {
  const int tid = threadIdx.x;
  unsigned mx = 0u;
  double sum0 = 0.0, sum1 = 0.0;
#pragma unroll 1
  for (int v = 0; v < 2; ++v) {
    double a[1] = {0.0};
    const uint32_t own = v ? L.own[1] : L.own[0];
    const int base = v ? L.base[1] : L.base[0], tbase = v ? L.tbase[1] : L.tbase[0];
    auto take = [&](int j, int idx) {
      const bool o = (FULL && j < L.ch) ? true : owns(own, j);
      const float g = (load && o) ? (float)st[idx] : 0.0f;  // u16 counts widen exactly
      mx = max(mx, __float_as_uint(g));
      a[0] = __dadd_rn(a[0], (double)g);
      return g;
    };
#pragma unroll 2
    for (int i = 0; i < S.np; ++i) {
      const float gA = take(2 * i, base + 16 * i);
      const float gB = take(2 * i + 1, base + 16 * i + 8);
      if (load) S.g[(v * S.np + i) * TPB + tid] = make_float2(gA, gB);
    }
    if (L.ch & 1) {
      const float g = take(L.ch - 1, base + 8 * (L.ch - 1));
      if (load) S.sg[(v * S.ns) * TPB + tid] = g;
    }
    leaf_combine<1>(a);  // xor 1, 2, 4: the 8 lanes of the octet
#pragma unroll 1
    for (int t = 0; t < L.tl; ++t) {
      const float g = take(L.ch + t, tbase + t);
      if (load) S.sg[(v * S.ns + (L.ch & 1) + t) * TPB + tid] = g;
    }
    if (v)
      sum1 = a[0];
    else
      sum0 = a[0];
  }
  gt = mx < 0x71800000u;
  g40 = mx < 0x53800000u;
  double g = __dadd_rn(sum0, sum1);  // this octet's pair of leaves, then the slot tree over octets
  if constexpr (SL >= 4) g = __dadd_rn(g, shfl_xor_d(g, 8));
  if constexpr (SL >= 8) g = __dadd_rn(g, shfl_xor_d(g, 16));
  return __dadd_rn(0.0, g);
}

// The group's lanes stream the 16-B aligned window around the next spot (stage_spot; PX = float or
// 16-bit counts).
template <int SL, int P, typename PX>
__device__ __forceinline__ int stage2l(const Smem<SL, P>& S, int gib, int gl, const PX* src, uintptr_t lo,
                                       uintptr_t hi, int N) {
  constexpr int LG = lanes_per_group<SL>();
  const uintptr_t a0 = (uintptr_t)src & ~(uintptr_t)15;
  const uintptr_t e0 = ((uintptr_t)(src + N) + 15) & ~(uintptr_t)15;
  const int nck = (int)((e0 - a0) >> 4);
  float* dst = S.stage + gib * S.sw;
  if (a0 >= lo && e0 <= hi) {
    for (int c = gl; c < nck; c += LG) cp_async16(dst + 4 * c, reinterpret_cast<const void*>(a0 + 16 * (uintptr_t)c));
  } else {
    for (int c = gl; c < nck; c += LG) {
      const uintptr_t cs = a0 + 16 * (uintptr_t)c;
      if (cs >= lo && cs + 16 <= hi) {
        cp_async16(dst + 4 * c, reinterpret_cast<const void*>(cs));
      } else if constexpr (sizeof(PX) == 4) {
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (cs + 4 * w >= lo && cs + 4 * w + 4 <= hi) cp_async4(dst + 4 * c + w, reinterpret_cast<const float*>(cs + 4 * w));
      } else {  // 2-byte pixels: plain loads (visible to the group after the refill's __syncwarp)
        PX* d = reinterpret_cast<PX*>(dst + 4 * c);
#pragma unroll
        for (int w = 0; w < 16 / (int)sizeof(PX); ++w)
          if (cs + sizeof(PX) * w >= lo && cs + sizeof(PX) * (w + 1) <= hi)
            d[w] = *reinterpret_cast<const PX*>(cs + sizeof(PX) * w);
      }
    }
  }
  return (int)(((uintptr_t)src & 15) / sizeof(PX));
}

}  // namespace l2

// launch bound: 4 CTAs per SM (128 registers) for P = 3; 3 for the elliptical model
template <int P>
#ifndef SF_MINB2L_P3
#define SF_MINB2L_P3 4
#endif
__host__ __device__ constexpr int minb2l() { return P == 3 ? SF_MINB2L_P3 : 3; }

// The kernel: fit_kernel's loop (refill -> fused evaluation -> LM step) for spots of SL leaves with
// given inits; PX: float pixels or 16-bit counts (staged as u16, widened exactly in load_spot2l).
template <int SL, int P, bool FULL, typename PX = float>
__global__ void __launch_bounds__(l2::TPB, minb2l<P>())
    fit_kernel2l(const PX* __restrict__ images, const float* __restrict__ inits, int64_t count, const Geom geom,
                 const Cfg cfg, FitOut out) {
  using namespace l2;
  constexpr int LG = lanes_per_group<SL>(), GPW = 32 / LG, VL = l2::Smem<SL, P>::VL;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t tmem_base;
  l2::Smem<SL, P> S;
  S.bind(smem_raw, geom.ch, geom.tl, geom.N);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // TMEM: 128 columns for the CTA (4 CTAs per SM use all 512)
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&tmem_base)),
                 "n"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");

  // lane -> group (LG lanes), octet of the group (a pair of leaves), chain k of both leaves
  l2::Lane L;
  L.gl = lane & (LG - 1);
  L.gw = lane / LG;
  L.gib = warp * GPW + L.gw;
  L.vl0 = 16 * (L.gl >> 3) + (lane & 7);
  L.ch = geom.ch;
  L.tl = geom.tl;
  // tail loop bound per leaf slot, uniform over the warp's octets (their leaves' largest tail)
#pragma unroll
  for (int v = 0; v < 2; ++v) {
    int m = 0;
    for (int o = 0; o < SL / 2; ++o) m = max(m, (int)geom.nt[16 * o + 8 * v]);
    L.tlv[v] = m;
  }
  L.tw = tmem_base + ((uint32_t)(warp * 32) << 16);
  L.Wf = (float)geom.W;
  L.invW = 1.0f / (float)geom.W;
#pragma unroll
  for (int v = 0; v < 2; ++v) {
    const int vl = L.vl0 + 8 * v;
    const int nc = geom.nc[vl], nt = geom.nt[vl];
    L.base[v] = geom.base[vl];
    L.tbase[v] = geom.tbase[vl];
    L.basef[v] = (float)geom.base[vl];
    L.tbasef[v] = (float)geom.tbase[vl];
    uint32_t own = 0u;
    for (int j = 0; j < L.ch + L.tl; ++j) {
      const bool o = j < L.ch ? j < nc : (j - L.ch) < nt;
      own |= (o ? 1u : 0u) << j;
    }
    L.own[v] = own;
  }
  // coordinate tables: thread vl < VL writes its virtual lane's pairs and solo slots
  if (!l2::Smem<SL, P>::kGen && tid < VL) {
    const int vl = tid, nc = geom.nc[vl], nt = geom.nt[vl], base = geom.base[vl], tbase = geom.tbase[vl];
    auto xy = [&](int j) {
      const bool o = j < L.ch ? j < nc : (j - L.ch) < nt;
      const int pp = !o ? 0 : (j < L.ch ? base + 8 * j : tbase + (j - L.ch));
      return make_float2((float)(pp % geom.W), (float)(pp / geom.W));
    };
    for (int i = 0; i < S.np; ++i) {
      const float2 a = xy(2 * i), b = xy(2 * i + 1);
      S.xy[i * VL + vl] = make_float4(a.x, b.x, a.y, b.y);
    }
    for (int s = 0; s < S.ns; ++s) S.sxy[s * VL + vl] = xy((L.ch & ~1) + s);
  }
  if (tid == 0) {
    S.kc[0] = ddiv_rcp(cfg.lam_down);
    S.kc[1] = ddiv_rcp((double)(geom.N - 5));
  }
  for (int i = 0; i < 2 * S.np; ++i) S.g[i * TPB + tid] = make_float2(0.0f, 0.0f);
  for (int r = 0; r < 2 * S.ns; ++r) S.sg[r * TPB + tid] = 0.0f;
  __syncthreads();

  const bool leader = L.gl == 0;
  const int N = geom.N;
  const double n = (double)N;
  double G = 0.0;
  LMState<P> s;
  s.sys = S.sys + L.gib * l2::Smem<SL, P>::kSysQ;
  s.gmask = LG == 32 ? kFull : ((1u << LG) - 1u) << (lane & ~(LG - 1));
  s.sys_writer = L.gl == 0;
  int64_t spot = -1;
  bool need = true, exhausted = false;
  bool lane_gt = true, lane_g40 = true, warp_gt = true;
  unsigned n_g = 0, n_t = 0, n_e = 0;
  float nxt[P];
  int nsh = 0;
  const uintptr_t lo = (uintptr_t)images, hi = (uintptr_t)(images + count * (int64_t)N);
  unsigned long long* wk = g_work[out.work_slot];
  auto claim = [&](bool want) -> int64_t {
    unsigned long long v = 0ull;
    if (want && L.gl == 0) v = atomicAdd(wk, 1ull);
    return (int64_t)__shfl_sync(kFull, v, lane & ~(LG - 1));
  };
  auto prefetch = [&](int64_t sp) {
    if (sp < count) {
      nsh = stage2l<SL, P, PX>(S, L.gib, L.gl, images + sp * (int64_t)N, lo, hi, N);
#pragma unroll
      for (int k = 0; k < P; ++k) nxt[k] = __ldg(inits + sp * P + k);
    }
    cp_async_commit();
  };
  int64_t nspot = claim(true);
  prefetch(nspot);

#pragma unroll 1
  for (;;) {
    bool skip = false;
    if (__any_sync(kFull, need)) {
      if (need) {
        spot = nspot;
        exhausted = spot >= count;
      }
      const bool load = need && !exhausted;
      if (load) cp_async_wait_all();
      __syncwarp(kFull);
      const PX* win = reinterpret_cast<const PX*>(S.stage + L.gib * S.sw) + nsh;
      bool sgt, sg40;
      const double gsum = load_spot2l<SL, P, FULL, PX>(S, L, win, load, sgt, sg40);
      bool bad = false;
      if (load) {
        float init[P];
        double v[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
          init[k] = nxt[k];
          bad = bad || !isfinite(init[k]);
          v[k] = (double)init[k];
        }
        limit_params<P>(cfg, v, s.p);
        s.lam = cfg.lam0;
        s.it = 0;
        s.fl = 0u;
#pragma unroll
        for (int k = 0; k < P; ++k) s.best[k] = init[k];
      }
      __syncwarp(kFull);  // the staging window has been read: refill it
      const int64_t nxt_spot = claim(load);
      if (load) {
        nspot = nxt_spot;
        prefetch(nspot);
      }
      const bool gbad = bad || !isfinite(gsum);
      if (load) {
        lane_gt = sgt;
        lane_g40 = sg40;
      }
      warp_gt = __all_sync(kFull, lane_gt || exhausted);
      if (load) {
        G = gsum;
        if (gbad) {
          write_result<P>(out, spot, leader, s.best, true, 0.f, 0.f, 0.f, N, SF_STOP_NOT_CONVERGED | SF_FLAG_INVALID, 0,
                          S.kc[1]);
          need = true;
          skip = true;
        } else {
          need = false;
        }
      } else if (need) {
        need = false;
      }
    }
    if (__all_sync(kFull, exhausted)) break;
    Eval<P> E;
    evaluate2l<SL, P, FULL>(S, L, G, n, s.p, warp_gt, lane_g40, !exhausted && !skip, geom.nz2, E);
    if (!exhausted && !skip) {
      n_e += 1;
      if (lm_step<P>(s, E, cfg, out, spot, leader, N, n_g, n_t, S.kc)) need = true;
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(wk + 1, 1ull) == (unsigned long long)gridDim.x - 1ull) {
      wk[0] = 0ull;
      wk[1] = 0ull;
    }
  }
  if (out.evals != nullptr && leader) {
    atomicAdd(out.evals + 0, (unsigned long long)n_g);
    atomicAdd(out.evals + 1, (unsigned long long)n_t);
    atomicAdd(out.evals + 2, (unsigned long long)n_e);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "n"(kCols));
}

}  // namespace sf
