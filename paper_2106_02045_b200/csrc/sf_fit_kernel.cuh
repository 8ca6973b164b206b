// sf_fit_kernel.cuh -- the fused, device-resident LM fit kernel (sm_100a).
//
// One "group" of 8*SLOTS chain lanes fits one spot at a time; groups are
// persistent and claim their next spot from a launch-wide counter (g_work), so
// a group that stops early loads its next spot while its warp-mates keep
// iterating, and the launch ends with every group busy.  Each loop trip is:
// [refill groups that finished] -> one fused evaluation
// (sf_device.cuh:evaluate) -> the LM state machine of SURVEY App. A
// (PAPER.md:126-180), divergent across groups but cheap.  No host round trip
// happens inside a fit.
#pragma once
#include "sf_device.cuh"
#include "sf_init_core.cuh"

namespace sf {

struct FitOut {
  float* params;
  float* alpha;
  float* beta;
  float* nchi2;
  uint8_t* status;
  uint8_t* iters;
  unsigned long long* evals;  // [3]: reference G-evals, reference T-evals, fused kernel evals (or null)
  int work_slot;              // g_work slot of this launch (sf_capi.cu:acquire_work_slot)
};

// Dynamic spot claiming.  Persistent groups take their next spot from a launch-
// wide counter instead of a static stride, so groups whose spots converge fast
// take more of them and the launch ends with every group busy until the last few
// spots (a static stride left ~10% of warp slots idle at the tail: v9 profile,
// warps_active 14.4 of 16).  g_work[slot] = {next spot, CTAs finished}; the last
// CTA of a launch resets its slot, so a slot is zero whenever no launch holds it.
// Slots [0, kStreamSlots) serve ordinary launches: the host (sf_capi.cu:WorkPool)
// hands a slot out only after the event recorded behind its previous launch has
// completed, so two launches never share a counter.  Slots [kStreamSlots,
// kWorkSlots) are owned for good by launches captured into CUDA graphs (replays
// of one graph exec are serialised by CUDA); when they run out the capture fails
// with an error instead of sharing.
constexpr int kStreamSlots = 256;
constexpr int kGraphSlots = 256;
constexpr int kWorkSlots = kStreamSlots + kGraphSlots;
static __device__ unsigned long long g_work[kWorkSlots][2];

// Per-spot LM state, replicated in every lane of the group.  The normal system
// at `best` (needed again only for lambda retries) lives in the group's shared
// slot `sys`: every lane holds the identical system, one lane per (group, warp)
// stores it (sys_writer) and __syncwarp(gmask) publishes it to the group's other
// lanes (compute-sanitizer racecheck clean: profiles/r01_compute_sanitizer.txt).
template <int P>
struct LMState {
  float p[P];     // parameters under evaluation (G point or trial point)
  float best[P];  // PAPER.md:144 "best := current"
  double lam;
  double* sys;    // [T + P]: JtJ (upper packed) then rhs at best (group's copy for this warp)
  unsigned gmask;  // the group's lanes in this warp; lane gl == 0 of them (sys_writer) stores sys
  bool sys_writer;
  float chib, ab, bb;  // chi^2, alpha, beta at best
  int it;
  unsigned fl;  // kTrial | kFirst | kSmall (one register, no byte packing)
  static constexpr unsigned kTrial = 1u, kFirst = 2u, kSmall = 4u;
  __device__ __forceinline__ bool trial() const { return fl & kTrial; }
  __device__ __forceinline__ bool first() const { return fl & kFirst; }
  __device__ __forceinline__ bool small() const { return fl & kSmall; }
};

template <int P>
__device__ __forceinline__ void write_result(const FitOut& o, int64_t spot, bool leader, const float (&p)[P],
                                             bool singular, float chi, float a, float b, int n_pix, int status,
                                             int it, double rcp_n5) {
  if (!leader) return;
#pragma unroll
  for (int k = 0; k < P; ++k) o.params[spot * P + k] = p[k];
  if (singular) {
    o.alpha[spot] = __int_as_float(0x7fc00000);
    o.beta[spot] = __int_as_float(0x7fc00000);
    o.nchi2[spot] = __int_as_float(0x7fc00000);
  } else {
    o.alpha[spot] = a;
    o.beta[spot] = b;
    // normalized_chi: chi^2/(N-5) in f64, quantised to f32
    o.nchi2[spot] = n_pix > 5 ? (float)ddiv_with((double)chi, (double)(n_pix - 5), rcp_n5) : chi;
  }
  o.status[spot] = (uint8_t)status;
  o.iters[spot] = (uint8_t)it;
}

// Post-trial decision of PAPER.md:153-174 (oracle/lm.py:fit_single) for a trial
// chi^2 `chit` (+inf for StepFailed, NaN for a singular / non-finite trial):
// returns kRetry (retry the step with the raised lambda), kAccept (the trial is
// the next iteration's point), or StopReason | flags >= 0 (MaxError is 0; with
// *at_best: restore best).
constexpr int kRetry = -1, kAccept = -2;
template <int P>
__device__ __forceinline__ int post_trial(LMState<P>& s, const Cfg& c, float chit, bool small, bool* at_best,
                                          double rcp_down) {
  if (s.first()) {
    s.fl &= ~LMState<P>::kFirst;
    if (s.chib > chit) s.lam = ddiv_with(s.lam, c.lam_down, rcp_down);  // == s.lam / c.lam_down
  }
  if (!small && s.chib < chit && s.lam < c.lam_max) {
    s.lam = s.lam * c.lam_up;
    return kRetry;
  }
  if (isnan(chit) || (s.chib < chit && s.lam >= c.lam_max)) {
    *at_best = true;
    return SF_STOP_NOT_CONVERGED;
  }
  if (s.chib < chit) {
    *at_best = true;
    return SF_STOP_MIN_DELTA | SF_FLAG_NOIMP;
  }
  if ((double)chit < c.max_error) return SF_STOP_MAX_ERROR;
  if ((double)s.chib * c.one_minus_min_delta < (double)chit) return SF_STOP_MIN_DELTA;
  if (small) return SF_STOP_MIN_STEP;
  if (s.it >= c.max_it) return SF_STOP_MAX_ITERATIONS;
  return kAccept;
}

// Consume one evaluation; returns true when the spot's fit has finished (result written).
// Mirrors oracle/lm.py:fit_single, with the accepted trial's
// evaluation reused as the next iteration's G-eval ([A6]).  Straight-line
// decision first, then ONE solve site: every group of the warp that needs a
// step reaches the (f64-division-bound) damped solve in the same pass, so the
// warp executes it once per trip instead of once per divergent path.
template <int P>
__device__ __forceinline__ bool lm_step(LMState<P>& s, const Eval<P>& E, const Cfg& c, const FitOut& o,
                                        int64_t spot, bool leader, int n_pix, unsigned& n_g, unsigned& n_t,
                                        const double* kc) {
  constexpr int T = P * (P + 1) / 2;
  int status = -1;       // StopReason | flags once the fit has finished
  bool at_best = false;  // result is the saved best point (restore) rather than E's point
  bool g_eval = !s.trial();
  if (s.trial()) {
    const float chit = E.singular ? __int_as_float(0x7fc00000) : E.chi;
    const int d = post_trial<P>(s, c, chit, s.small(), &at_best, kc[0]);
    if (d == kAccept) {
      s.fl &= ~LMState<P>::kTrial;  // accepted, budget left: E is exactly the next iteration's G-eval at s.p
      g_eval = true;
    } else if (d >= 0) {
      status = d;
    }
  }
  if (g_eval) {
    s.it += 1;
    n_g += 1;
    if (E.singular || !isfinite(E.chi)) {
      status = SF_STOP_NOT_CONVERGED;
    } else if ((double)E.chi < c.max_error) {
      status = SF_STOP_MAX_ERROR;
    } else {
      s.chib = E.chi;
      s.ab = E.alpha;
      s.bb = E.beta;
#pragma unroll
      for (int k = 0; k < P; ++k) s.best[k] = s.p[k];
      // every lane holds the identical system: one lane per (group, warp) stores it
      if (s.sys_writer) {
#pragma unroll
        for (int k = 0; k < P; ++k) s.sys[T + k] = E.rhs[k];
#pragma unroll
        for (int m = 0; m < T; ++m) s.sys[m] = E.jtj[m];
      }
      __syncwarp(s.gmask);
      s.fl |= LMState<P>::kFirst;
    }
  }
  // PAPER.md:147-151 and the retry body 159-164
#pragma unroll 1
  while (status < 0) {
    double jtj[T], rhs[P], delta[P];
#pragma unroll
    for (int m = 0; m < T; ++m) jtj[m] = s.sys[m];
#pragma unroll
    for (int k = 0; k < P; ++k) rhs[k] = s.sys[T + k];
    bool solved;
    if constexpr (P == 5) {
      solved = solve_pivot5(jtj, rhs, s.lam, delta);
    } else {
      solved = solve_step<P>(jtj, rhs, s.lam, delta);
#ifdef SF_ABL_SOLVE2
      {  // ablation: a second solve at a perturbed lambda (marginal cost of the damped solve)
        double d2[P];
        const bool ok2 = solve_step<P>(jtj, rhs, s.lam + c.zero * s.lam, d2);
#pragma unroll
        for (int k = 0; k < P; ++k) delta[k] = __fma_rn(d2[k], c.zero, delta[k]);
        solved = solved && (ok2 || c.zero == 0.0);
      }
#endif
    }
    if (solved) {
      double v[P];
      bool small = true;
#pragma unroll
      for (int k = 0; k < P; ++k) {
        v[k] = (double)s.best[k] + delta[k];
        // min_step * max(|best|, 1) (oracle/lm.py): the max of two f32 values is exact in f32
        const double thr = c.min_step * (double)fmaxf(fabsf(s.best[k]), 1.0f);
        small = small && (fabs(delta[k]) < thr);
      }
      limit_params<P>(c, v, s.p);
      s.fl = (s.fl & ~LMState<P>::kSmall) | LMState<P>::kTrial | (small ? LMState<P>::kSmall : 0u);
      n_t += 1;
      return false;  // evaluate the trial point next
    }
    // StepFailed: chi'^2 = +inf, not small -> retry with a raised lambda or stop
    const int d = post_trial<P>(s, c, __int_as_float(0x7f800000), false, &at_best, kc[0]);
    if (d >= 0) status = d;  // (never kAccept: +inf is not below chi_best)
  }
  float rp[P];
#pragma unroll
  for (int k = 0; k < P; ++k) rp[k] = at_best ? s.best[k] : s.p[k];
  write_result<P>(o, spot, leader, rp, !at_best && E.singular, at_best ? s.chib : E.chi, at_best ? s.ab : E.alpha,
                  at_best ? s.bb : E.beta, n_pix, status, s.it, kc[1]);
  return true;
}

// Fused initializer (inits == NULL): estimate_initial of the spot
// in the group's staging window, computed during the refill, so the pixels cross
// HBM (and, for host batches, PCIe) once.  Same arithmetic as the standalone
// initializer (sf_init_core.cuh); tame: every pixel of the spot is an integer in
// [0, 2^20] (load_spot), which takes the exact integer column walk.  When exactly
// one group of a multi-group warp refills -- the common case -- the whole warp
// scans its spot (the other groups' lanes would idle through the refill anyway),
// else each refilling group scans its own.  Every lane of the warp (CTA when
// SLOTS >= 8) calls it; lanes with !load only take part in the reductions.
// Result: (x, y, sigma[, sigma]) -- explicit-5: (x, y, sigma, alpha, beta) as
// batch_engine._auto_inits builds it.
template <int P, int SLOTS, typename PX>
__device__ __forceinline__ void fused_init(const PX* st, bool load, bool tame, const Geom& geom, const Cfg& cfg,
                                           float invW, int gl, float (&init)[P]) {
  constexpr int LANES = 8 * SLOTS;
  constexpr int LW = LANES < 32 ? LANES : 32;
  const int N = geom.N, W = geom.W, H = geom.H;
  int m = 0;
  int idx;
  float alpha, beta;
  double thr;
  bool done = false;
  if constexpr (LANES < 32) {
    const unsigned lm = __ballot_sync(kFull, load);
    if (__popc(lm) == LANES) {  // warp-uniform: one group refills, all 32 lanes scan its window
      const int src = __ffs(lm) - 1, lane = threadIdx.x & 31;
      const PX* wst = reinterpret_cast<const PX*>(__shfl_sync(kFull, reinterpret_cast<unsigned long long>(st), src));
      const bool wtame = __shfl_sync(kFull, tame ? 1 : 0, src) != 0;
      InitScan a;
      scan_reset(a);
      if (wtame)
        init_scan_tame<32, PX>(wst, W, H, lane, a);
      else
        init_scan(wst, W, H, N, invW, lane, 32, a);
      scan_reduce<32>(a);
      init_finish(a, idx, alpha, beta, thr);
      m = wtame ? init_count_tame(wst, N, thr, lane, 32) : init_count(wst, N, thr, lane, 32);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) m += __shfl_xor_sync(kFull, m, o);
      done = true;
    }
  }
  if (!done) {
    InitScan a;
    scan_reset(a);
    if (load) {  // tame is group-uniform (it may differ between the groups of a warp): no shuffles inside
      if (tame)
        init_scan_tame<LANES, PX>(st, W, H, gl, a);
      else
        init_scan(st, W, H, N, invW, gl, LANES, a);
    }
    scan_reduce<LW>(a);
    if constexpr (SLOTS >= 8) {  // the group is the CTA: merge the warps' partials through shared memory
      constexpr int WARPS = LANES / 32;
      __shared__ InitScan part[WARPS];
      __shared__ int msum[WARPS];
      const int warp = threadIdx.x >> 5;
      if ((threadIdx.x & 31) == 0) part[warp] = a;
      __syncthreads();
#pragma unroll
      for (int w = 0; w < WARPS; ++w) scan_merge(a, part[w].key, part[w].lo, part[w].nan);
      init_finish(a, idx, alpha, beta, thr);
      if (load) m = tame ? init_count_tame(st, N, thr, gl, LANES) : init_count(st, N, thr, gl, LANES);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) m += __shfl_xor_sync(kFull, m, o);
      if ((threadIdx.x & 31) == 0) msum[warp] = m;
      __syncthreads();
      m = 0;
#pragma unroll
      for (int w = 0; w < WARPS; ++w) m += msum[w];
      __syncthreads();  // part / msum are rewritten by the next refill
    } else {
      init_finish(a, idx, alpha, beta, thr);
      if (load) m = tame ? init_count_tame(st, N, thr, gl, LANES) : init_count(st, N, thr, gl, LANES);
#pragma unroll
      for (int o = 1; o < LW; o <<= 1) m += __shfl_xor_sync(kFull, m, o);
    }
  }
  const float sg = init_sigma(m, cfg.lo[2], cfg.hi[2]);
  const int iy = (int)(((float)idx + 0.5f) * invW);  // idx / W exactly (sf_init_core.cuh:init_smoothed)
  init[0] = (float)(idx - iy * W);
  init[1] = (float)iy;
  init[2] = sg;
  if constexpr (P == 4) init[3] = sg;
  if constexpr (P == 5) {
    init[3] = alpha;
    init[4] = beta;
  }
}

// Lane identity and pixel ownership, shared by the fit and eval kernels.
template <int P, int SLOTS>
struct LaneSetup {
  int gl;         // lane within the group
  int64_t gid;    // group id
  int64_t ngroups;
  uint32_t own;   // owned-pixel mask, bit j (chain j < ch, tail ch + t)
  int base, tbase, ch, tl;
  LaneGeo lg;

  // group index within the CTA
  __device__ __forceinline__ int gib() const {
    return SLOTS >= 8 ? 0 : (threadIdx.x >> 5) * (32 / (8 * SLOTS)) + (threadIdx.x & 31) / (8 * SLOTS);
  }
  // pixel index of slot j (chain: base + 8 j, tail: tbase + j - ch), or -1 if not owned
  __device__ __forceinline__ int off(int j) const {
    return owns(own, j) ? (j < ch ? base + 8 * j : tbase + (j - ch)) : -1;
  }

  __device__ __forceinline__ void init(Smem<P, SLOTS>& S, const Geom& geom, double cfg_lam_down = 1.0) {
    constexpr int LANES = 8 * SLOTS;
    const int lane = threadIdx.x & 31;
    if constexpr (SLOTS >= 8) {
      gl = threadIdx.x;
      gid = blockIdx.x;
      ngroups = gridDim.x;
    } else {
      constexpr int GPW = 32 / LANES;
      gl = lane % LANES;
      gid = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * GPW + lane / LANES;
      ngroups = (int64_t)gridDim.x * (blockDim.x >> 5) * GPW;
    }
    ch = geom.ch;
    tl = geom.tl;
    const int nc = geom.nc[gl], nt = geom.nt[gl];
    base = geom.base[gl];
    tbase = geom.tbase[gl];
    own = 0u;
    for (int j = 0; j < ch + tl; ++j) {
      const bool o = j < ch ? j < nc : (j - ch) < nt;
      own |= (o ? 1u : 0u) << j;
    }
    lg.gl = gl;
    lg.basef = (float)base;
    lg.tbasef = (float)tbase;
    lg.Wf = (float)geom.W;
    lg.invW = 1.0f / (float)geom.W;
    lg.nz2 = geom.nz2;
    // coordinate table (single-warp groups), written by the lanes of the CTA's first group:
    // pair rows hold (x_A, x_B, y_A, y_B) of chain slots (2i, 2i+1), solo rows (x, y)
    if (SLOTS < 8 && threadIdx.x < LANES) {
      auto xy = [&](int j) {
        const int o = off(j);
        const int pp = o < 0 ? 0 : o;
        return make_float2((float)(pp % geom.W), (float)(pp / geom.W));
      };
      for (int i = 0; i < ch / 2; ++i) {
        const float2 a = xy(2 * i), b = xy(2 * i + 1);
        S.pr[i].xy[SLOTS >= 8 ? 0 : gl] = make_float4(a.x, b.x, a.y, b.y);
      }
      for (int j = ch & ~1; j < ch + tl; ++j) S.so[j - (ch & ~1)].xy[SLOTS >= 8 ? 0 : gl] = xy(j);
    }
    // CTA constants: reciprocal stages of the fixed divisors lambda_down and N - 5
    if (threadIdx.x == 0) {
      S.kc[0] = ddiv_rcp(cfg_lam_down);
      S.kc[1] = ddiv_rcp((double)(geom.N - 5));
    }
    // pixel values start at 0 (load_spot rewrites a group's slots on every refill)
    for (int i = 0; i < ch / 2; ++i) S.pr[i].g[threadIdx.x] = make_float2(0.0f, 0.0f);
    for (int r = 0; r < (ch & 1) + tl; ++r) S.so[r].g[threadIdx.x] = 0.0f;
    __syncthreads();
  }
};

// PX: pixel type of `images` -- float, or uint16_t camera counts (sf_fit_batch_u16), staged as
// u16 and widened exactly in load_spot, so the host pipeline needs no separate widening kernel.
// FUSED: inits == NULL, the refill estimates them (fused_init); a separate instantiation, so the
// kernel that is given inits carries none of the initializer's code or registers.
template <int P, int SLOTS, bool FULL, typename PX = float, bool FUSED = false>
__global__ void __launch_bounds__(threads_per_block<SLOTS>(),
                                  P == 5 ? (SLOTS >= 8 ? 1 : SF_MINB_P5)
                                         : (SLOTS == 8 ? 2 * SF_MINB_P3 : (SLOTS == 16 ? SF_MINB_P3
                                                                                     : (P == 3 ? SF_MINB_P3 : SF_MINB_P4))))
    fit_kernel(const PX* __restrict__ images, const float* __restrict__ inits, int64_t count, const Geom geom,
               const Cfg cfg, FitOut out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<P, SLOTS> S;
  S.bind(smem_raw, geom.ch, geom.tl, geom.N);
  LaneSetup<P, SLOTS> L;
  L.init(S, geom, cfg.lam_down);
  const bool leader = L.gl == 0;
  const int N = geom.N;
  const double n = (double)N;

  double G = 0.0;
  LMState<P> s;
  s.sys = S.sys + (SLOTS >= 8 ? (int)(threadIdx.x >> 5) : L.gib()) * Smem<P, SLOTS>::kSysQ;
  {
    constexpr int LW = 8 * SLOTS < 32 ? 8 * SLOTS : 32;
    s.gmask = LW == 32 ? kFull : ((1u << LW) - 1u) << ((threadIdx.x & 31) & ~(LW - 1));
    s.sys_writer = ((threadIdx.x & 31) & (LW - 1)) == 0;
  }
  int64_t spot = L.gid - L.ngroups;
  bool need = true, exhausted = false;
  bool lane_gt = true, lane_g40 = true, warp_gt = true;  // spot tameness (load_spot)
  unsigned n_g = 0, n_t = 0, n_e = 0;

  // Next-spot prefetch: the group streams the next spot into its staging window
  // (stage_spot) while the current spot iterates, the init into registers; a
  // refill waits for the copies, scatters the window into the lanes' pixel
  // slots (load_spot), then starts the following spot's copy.
  float nxt[P];
  constexpr bool fused = FUSED;  // fused initializer: inits estimated from the staged spot
  int nsh = 0;  // float offset of the staged spot inside its window
  const int gib = L.gib();
  const uintptr_t lo = (uintptr_t)images, hi = (uintptr_t)(images + count * (int64_t)N);
  auto prefetch = [&](int64_t sp) {
    if (sp < count) {
      nsh = stage_spot<P, SLOTS, PX>(S, gib, L.gl, images + sp * (int64_t)N, lo, hi, N);
      if constexpr (!fused) {
#pragma unroll
        for (int k = 0; k < P; ++k) nxt[k] = __ldg(inits + sp * P + k);
      }
    }
    cp_async_commit();
  };
  unsigned long long* wk = g_work[out.work_slot];
  __shared__ unsigned long long claim_bc;  // multi-warp groups: the claimed index, CTA-wide
  // next spot for the group (want: group-uniform); every lane of the warp (CTA) calls it
  auto claim = [&](bool want) -> int64_t {
    if constexpr (SLOTS >= 8) {
      if (threadIdx.x == 0 && want) claim_bc = atomicAdd(wk, 1ull);
      __syncthreads();
      const unsigned long long v = claim_bc;
      __syncthreads();
      return (int64_t)v;
    } else {
      unsigned long long v = 0ull;
      if (want && L.gl == 0) v = atomicAdd(wk, 1ull);
      return (int64_t)__shfl_sync(kFull, v, (threadIdx.x & 31) & ~(8 * SLOTS - 1));
    }
  };
  int64_t nspot = claim(true);  // claimed and staged
  prefetch(nspot);

#pragma unroll 1
  for (;;) {
    // Every warp-collective below (votes, shuffles inside load_spot and
    // evaluate) is reached by all 32 lanes on every trip: groups only diverge
    // in the LM bookkeeping after the evaluation.
    bool skip = false;  // group refilled with an InvalidInput spot: no LM step this trip
    if (__any_sync(kFull, need)) {
      // ---- refill: next spot for every group whose fit finished
      if (need) {
        spot = nspot;
        exhausted = spot >= count;
      }
      const bool load = need && !exhausted;
      if (load) cp_async_wait_all();  // this lane's copies of `spot` have landed
      group_sync<SLOTS>();             // ... and every other lane's
      const PX* win = reinterpret_cast<const PX*>(S.stage + gib * S.sw) + nsh;
      // G = sum g (model.py:223); it is non-finite iff some pixel is (a sum of <= 1024 finite
      // f32 values cannot overflow f64), so it doubles as the InvalidInput pixel check
      bool sgt, sg40, sint = true;
      const double gsum = load_spot<P, SLOTS, FULL, PX>(S, win, load, L.own, L.base, L.tbase, L.ch, L.tl, sgt, sg40,
                                                        fused ? &sint : nullptr);
      bool bad = false;
      if constexpr (fused) fused_init<P, SLOTS, PX>(win, load, group_all<SLOTS>(sint), geom, cfg, L.lg.invW, L.gl, nxt);
      if (load) {
        float init[P];
        double v[P];
#pragma unroll
        for (int k = 0; k < P; ++k) {
          init[k] = nxt[k];
          bad = bad || !isfinite(init[k]);
          v[k] = (double)init[k];
        }
        limit_params<P>(cfg, v, s.p);  // SPEC.md:211 "sigma within bounds after limit"
        s.lam = cfg.lam0;
        s.it = 0;
        s.fl = 0u;
        // the raw init is the InvalidInput result (oracle/lm.py:fit_single) whether the init or a
        // pixel is non-finite; `best` is free until the first G-eval overwrites it
#pragma unroll
        for (int k = 0; k < P; ++k) s.best[k] = init[k];
      }
      group_sync<SLOTS>();  // the staging window has been read: refill it
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
          need = true;  // fetch the next spot on the next trip
          skip = true;
        } else {
          need = false;
        }
      } else if (need) {
        need = false;  // exhausted
      }
    }
    if (__all_sync(kFull, exhausted)) break;

    Eval<P> E;
    if constexpr (P == 5) {
      evaluate_explicit5<SLOTS, FULL>(S, L.lg, L.own, L.ch, L.tl, s.p, lane_g40, !exhausted && !skip, E);
    } else {
      evaluate<P, SLOTS, FULL>(S, L.lg, L.own, L.ch, L.tl, G, n, s.p, warp_gt, lane_g40, !exhausted && !skip, E,
                               nullptr, cfg.zero);
    }
    if (!exhausted && !skip) {
      n_e += 1;
      if (lm_step<P>(s, E, cfg, out, spot, leader, N, n_g, n_t, S.kc)) need = true;
    }
  }
  // release the claim counter: the last CTA to finish resets the slot
  __syncthreads();
  if (threadIdx.x == 0) {
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
}

// Model-level evaluation (sf_eval_batch_device): one group per spot, no LM.
template <int P, int SLOTS, bool FULL>
__global__ void __launch_bounds__(threads_per_block<SLOTS>())
    eval_kernel(const float* __restrict__ images, const float* __restrict__ params, int64_t count, const Geom geom,
                sf_eval_record* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<P, SLOTS> S;
  S.bind(smem_raw, geom.ch, geom.tl, geom.N);
  LaneSetup<P, SLOTS> L;
  L.init(S, geom);
  const int N = geom.N;
  const bool valid = L.gid < count;
  const int64_t spot = valid ? L.gid : 0;
  const int gib = L.gib();
  int sh = 0;
  if (valid)
    sh = stage_spot<P, SLOTS>(S, gib, L.gl, images + spot * (int64_t)N, (uintptr_t)images,
                              (uintptr_t)(images + count * (int64_t)N), N);
  cp_async_commit();
  cp_async_wait_all();
  group_sync<SLOTS>();
  float pe[P];
#pragma unroll
  for (int k = 0; k < P; ++k) pe[k] = valid ? __ldg(params + spot * P + k) : 1.0f;
  bool gt, g40;
  const double G = load_spot<P, SLOTS>(S, S.stage + gib * S.sw + sh, valid, L.own, L.base, L.tbase, L.ch, L.tl, gt, g40);
  Eval<P> E;
  EvalExtras<P> X;
  evaluate<P, SLOTS, FULL, true>(S, L.lg, L.own, L.ch, L.tl, G, (double)N, pe, __all_sync(kFull, gt), g40, true, E, &X);
  if (valid && L.gl == 0) {
    sf_eval_record r;
    r.singular = E.singular ? 1 : 0;
    r.alpha = E.alpha;
    r.beta = E.beta;
    r.chi = E.chi;
    r.F = X.F;
    r.G = G;
    r.FF = X.FF;
    r.FG = X.FG;
    r.denom = X.denom;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int kk = k < P ? k : 0;
      const bool in = k < P;
      r.dF[k] = in ? X.dF[kk] : 0.0;
      r.dFF[k] = in ? X.dFF[kk] : 0.0;
      r.dFG[k] = in ? X.dFG[kk] : 0.0;
      r.gamma[k] = in ? X.gamma[kk] : 0.0;
      r.dalpha[k] = in ? X.dalpha[kk] : 0.0;
      r.dbeta[k] = in ? X.dbeta[kk] : 0.0;
      r.rhs[k] = in ? E.rhs[kk] : 0.0;
    }
    constexpr int T = P * (P + 1) / 2;
#pragma unroll
    for (int m = 0; m < 10; ++m) r.jtj[m] = m < T ? E.jtj[m < T ? m : 0] : 0.0;
    out[spot] = r;
  }
}

}  // namespace sf
