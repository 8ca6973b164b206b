// sf_capi.cu -- the C-ABI (include/spotfit.h): argument checking, lane
// geometry, kernel dispatch, and the host-side batch scheduler (chunked
// H2D -> kernel -> D2H over round-robin streams, one host thread per device,
// contiguous shards, no collectives -- SURVEY 8e).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "sf_geometry.h"
#include "sf_launch.h"

namespace {

thread_local std::string g_err;

int fail(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return -1;
}

#define SF_CUDA(call)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return fail("%s failed: %s", #call, cudaGetErrorString(e_));       \
  } while (0)

int check_grid(int W, int H) {
  if (W < 1 || H < 1) return fail("degenerate grid %dx%d", W, H);                   // model.py:53-54
  if ((int64_t)W * H > 1024) return fail("grid %dx%d exceeds 1024 pixels", W, H);  // model.py:55-58
  return 0;
}

int make_cfg(const sf_config* c, int W, int H, sf::Cfg& k) {
  if (c == nullptr) return fail("cfg is NULL");
  if (c->model != SF_MODEL_SYMMETRIC && c->model != SF_MODEL_ELLIPTICAL && c->model != SF_MODEL_EXPLICIT5)
    return fail("model must be 3, 4 or 5");
  if (c->max_iterations < 1 || c->max_iterations > 255) return fail("max_iterations must be in [1, 255]");
  if (!(c->min_delta > 0) || !(c->min_step > 0)) return fail("min_delta and min_step must be > 0");
  if (!(c->max_error >= 0)) return fail("max_error must be >= 0");
  if (!(c->lambda_init > 0) || !(c->lambda_init < c->lambda_max)) return fail("need 0 < lambda_init < lambda_max");
  // > 1 guarantees the retry loop terminates (lambda reaches lambda_max)
  if (!(c->lambda_up > 1) || !(c->lambda_down > 1)) return fail("lambda factors must be > 1");
  if (!(c->sigma_min > 0) || !(c->sigma_max > c->sigma_min)) return fail("need 0 < sigma_min < sigma_max");
  if (!(c->margin_x >= 0) || !(c->margin_y >= 0)) return fail("margins must be >= 0");
  k.max_it = c->max_iterations;
  k.max_error = c->max_error;
  k.min_delta = c->min_delta;
  k.one_minus_min_delta = 1.0 - c->min_delta;
  k.zero = 0.0;
  k.min_step = c->min_step;
  k.lam0 = c->lambda_init;
  k.lam_up = c->lambda_up;
  k.lam_down = c->lambda_down;
  k.lam_max = c->lambda_max;
  k.lo[0] = -c->margin_x;
  k.hi[0] = (double)(W - 1) + c->margin_x;
  k.lo[1] = -c->margin_y;
  k.hi[1] = (double)(H - 1) + c->margin_y;
  k.lo[2] = k.lo[3] = c->sigma_min;
  k.hi[2] = k.hi[3] = c->sigma_max;
  k.lo[4] = -INFINITY;  // explicit-5 beta (free); alpha uses [3] only in the explicit limit (free too)
  k.hi[4] = INFINITY;
  return 0;
}

constexpr int kMaxP = 5;  // widest parameter vector (explicit-5) -- staging layout

int sm_count_of_current() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 1;
}


// Work-claim counter slots (sf_fit_kernel.cuh:g_work), per device.  An ordinary
// launch takes a stream slot whose previous launch has completed (the event
// recorded behind it has fired); with all kStreamSlots launches still in flight
// the caller waits for the oldest.  A launch being captured into a CUDA graph
// takes a graph slot for good (the graph may replay at any time); when those run
// out the call fails.  Two launches therefore never share a counter, which would
// split one launch's spots between two grids and leave some unfitted.
struct WorkPool {
  std::mutex mu;
  bool init = false;
  cudaEvent_t ev[sf::kStreamSlots] = {};
  bool armed[sf::kStreamSlots] = {};
  unsigned next = 0;
  int next_graph = 0;
  int dev = 0;
};
std::mutex g_pool_mu;
std::vector<std::unique_ptr<WorkPool>> g_pool;

WorkPool* pool_for(int dev) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if ((int)g_pool.size() <= dev) g_pool.resize(dev + 1);
  if (!g_pool[dev]) {
    g_pool[dev].reset(new WorkPool());
    g_pool[dev]->dev = dev;
  }
  return g_pool[dev].get();
}

// Launches the fit through `launch(slot)` with a private claim counter, under the pool lock.
template <class Launch>
int with_work_slot(cudaStream_t st, Launch&& launch) {
  int dev = 0;
  SF_CUDA(cudaGetDevice(&dev));
  WorkPool* w = pool_for(dev);
  std::lock_guard<std::mutex> lk(w->mu);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  SF_CUDA(cudaStreamIsCapturing(st, &cs));
  if (cs == cudaStreamCaptureStatusActive) {
    if (w->next_graph >= sf::kGraphSlots)
      return fail("device %d: %d fit launches were already captured into CUDA graphs; each keeps a private "
                  "work-claim counter and none is left", dev, sf::kGraphSlots);
    return launch(sf::kStreamSlots + w->next_graph++);
  }
  if (cs != cudaStreamCaptureStatusNone) return fail("stream capture was invalidated");
  if (!w->init) {
    for (auto& e : w->ev) SF_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    w->init = true;
  }
  int slot = -1;
  for (int t = 0; t < sf::kStreamSlots && slot < 0; ++t) {
    const int k = (int)(w->next++ % (unsigned)sf::kStreamSlots);
    if (!w->armed[k]) {
      slot = k;
      break;
    }
    const cudaError_t q = cudaEventQuery(w->ev[k]);
    if (q == cudaSuccess) {
      slot = k;
    } else if (q == cudaErrorNotReady) {
      (void)cudaGetLastError();  // not an error: the slot's launch is still running
    } else {
      return fail("cudaEventQuery failed: %s", cudaGetErrorString(q));
    }
  }
  if (slot < 0) {  // every slot busy: wait for the next one in round-robin order
    slot = (int)(w->next++ % (unsigned)sf::kStreamSlots);
    SF_CUDA(cudaEventSynchronize(w->ev[slot]));
  }
  if (launch(slot) != 0) return -1;
  SF_CUDA(cudaEventRecord(w->ev[slot], st));
  w->armed[slot] = true;
  return 0;
}

int dispatch_fit(int P, const sf::LaunchFit& a_in) {
  return with_work_slot(a_in.stream, [&](int work_slot) -> int {
    sf::LaunchFit a = a_in;
    a.out.work_slot = work_slot;
    cudaError_t err = cudaSuccess;
    int used = -1;
    const int slots = a.geom.slots, ch = a.geom.ch, tl = a.geom.tl;
#define SF_CASE(PP, S) \
  if (P == PP && slots == S) used = sf::launch_fit_P##PP##_S##S(a, &err);
    SF_CASE(3, 1) SF_CASE(3, 2) SF_CASE(3, 4) SF_CASE(3, 8) SF_CASE(3, 16)
    SF_CASE(4, 1) SF_CASE(4, 2) SF_CASE(4, 4) SF_CASE(4, 8) SF_CASE(4, 16)
    SF_CASE(5, 1) SF_CASE(5, 2) SF_CASE(5, 4) SF_CASE(5, 8) SF_CASE(5, 16)
#undef SF_CASE
    if (used < 0) return fail("no kernel instantiation for P=%d slots=%d chain=%d tail=%d", P, slots, ch, tl);
    if (err != cudaSuccess) return fail("fit kernel launch failed: %s", cudaGetErrorString(err));
    return 0;
  });
}

int dispatch_eval(int P, const sf::LaunchEval& a) {
  cudaError_t err = cudaSuccess;
  int used = -1;
  const int slots = a.geom.slots, ch = a.geom.ch, tl = a.geom.tl;
#define SF_CASE(PP, S) \
  if (P == PP && slots == S) used = sf::launch_eval_P##PP##_S##S(a, &err);
  SF_CASE(3, 1) SF_CASE(3, 2) SF_CASE(3, 4) SF_CASE(3, 8) SF_CASE(3, 16)
  SF_CASE(4, 1) SF_CASE(4, 2) SF_CASE(4, 4) SF_CASE(4, 8) SF_CASE(4, 16)
#undef SF_CASE
  if (used < 0) return fail("no kernel instantiation for P=%d slots=%d chain=%d tail=%d", P, slots, ch, tl);
  if (err != cudaSuccess) return fail("eval kernel launch failed: %s", cudaGetErrorString(err));
  return 0;
}

// ---------------------------------------------------------------------------
// Per-device context: streams, device chunk buffers, pinned staging, events.
// ---------------------------------------------------------------------------
#ifndef SF_STREAMS
#define SF_STREAMS 4  // chunk slots (stream + staging) per device: profiles/r02_ab_narrow_pinned.txt
#endif
constexpr int kStreams = SF_STREAMS;

struct Slot {
  cudaStream_t stream = nullptr;
  cudaEvent_t ev[4] = {};  // start, h2d done, kernel done, d2h done
  float* d_img = nullptr;
  uint16_t* d_img16 = nullptr;  // 16-bit chunk (sf_fit_batch_u16), read as u16 by the fit kernel
  float* d_init = nullptr;
  float* d_par = nullptr;
  float* d_a = nullptr;
  float* d_b = nullptr;
  float* d_c = nullptr;
  uint8_t* d_st = nullptr;
  uint8_t* d_it = nullptr;
  float* h_in = nullptr;   // pinned staging (pageable callers): images then inits
  uint16_t* h_in16 = nullptr;  // pinned u16 staging: integer-valued f32 chunks narrowed for the PCIe leg
  float* h_out = nullptr;  // pinned staging: params, alpha, beta, nchi2, status, iters
  size_t cap_spots = 0, cap_npix = 0;
  bool pending = false;  // staged results of a finished chunk waiting to be copied out
  int64_t p_lo = 0, p_n = 0;
};

struct DevCtx {
  std::mutex mu;
  bool init = false;
  int sms = 1;
  Slot slot[kStreams];
  unsigned long long* d_evals = nullptr;
  unsigned long long* h_evals = nullptr;  // pinned: the evaluation counters read back with the results
  cudaEvent_t evals_zeroed = nullptr;     // the counter reset, which every slot stream waits for
};

std::mutex g_ctx_mu;
std::vector<std::unique_ptr<DevCtx>> g_ctx;

DevCtx* ctx_for(int dev) {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if ((int)g_ctx.size() <= dev) g_ctx.resize(dev + 1);
  if (!g_ctx[dev]) g_ctx[dev].reset(new DevCtx());
  return g_ctx[dev].get();
}

void free_slot_buffers(Slot& s) {
  cudaFree(s.d_img); cudaFree(s.d_img16); cudaFree(s.d_init); cudaFree(s.d_par); cudaFree(s.d_a); cudaFree(s.d_b); cudaFree(s.d_c);
  cudaFree(s.d_st); cudaFree(s.d_it);
  cudaFreeHost(s.h_in); cudaFreeHost(s.h_out); cudaFreeHost(s.h_in16);
  s.d_img = s.d_init = s.d_par = s.d_a = s.d_b = s.d_c = nullptr;
  s.d_img16 = nullptr;
  s.d_st = s.d_it = nullptr;
  s.h_in = s.h_out = nullptr;
  s.h_in16 = nullptr;
  s.cap_spots = 0;
}

int ensure_ctx(DevCtx& c, int dev, size_t spots, int npix, int P, bool staging, bool narrow) {
  if (!c.init) {
    SF_CUDA(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev));
    for (auto& s : c.slot) {
      SF_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
      for (auto& e : s.ev) SF_CUDA(cudaEventCreate(&e));
    }
    SF_CUDA(cudaMalloc(&c.d_evals, 3 * sizeof(unsigned long long)));
    SF_CUDA(cudaHostAlloc(&c.h_evals, 3 * sizeof(unsigned long long), cudaHostAllocPortable));
    SF_CUDA(cudaEventCreateWithFlags(&c.evals_zeroed, cudaEventDisableTiming));
    c.init = true;
  }
  for (auto& s : c.slot) {
    const bool grow = s.cap_spots < spots || s.cap_npix < (size_t)npix || (staging && s.h_in == nullptr) ||
                      (narrow && s.h_in16 == nullptr);
    if (!grow) continue;
    free_slot_buffers(s);
    SF_CUDA(cudaMalloc(&s.d_img, spots * npix * sizeof(float)));
    SF_CUDA(cudaMalloc(&s.d_img16, spots * npix * sizeof(uint16_t)));
    SF_CUDA(cudaMalloc(&s.d_init, spots * kMaxP * sizeof(float)));
    SF_CUDA(cudaMalloc(&s.d_par, spots * kMaxP * sizeof(float)));
    SF_CUDA(cudaMalloc(&s.d_a, spots * sizeof(float)));
    SF_CUDA(cudaMalloc(&s.d_b, spots * sizeof(float)));
    SF_CUDA(cudaMalloc(&s.d_c, spots * sizeof(float)));
    SF_CUDA(cudaMalloc(&s.d_st, spots));
    SF_CUDA(cudaMalloc(&s.d_it, spots));
    if (staging) {  // h_in: images | inits[kMaxP];  h_out: params[kMaxP] | alpha | beta | nchi2 | status, iters
      SF_CUDA(cudaHostAlloc(&s.h_in, spots * (npix + kMaxP) * sizeof(float), cudaHostAllocPortable));
      SF_CUDA(cudaHostAlloc(&s.h_out, spots * (kMaxP + 3 + 1) * sizeof(float), cudaHostAllocPortable));
    }
    if (narrow) SF_CUDA(cudaHostAlloc(&s.h_in16, spots * npix * sizeof(uint16_t), cudaHostAllocPortable));
    s.cap_spots = spots;
    s.cap_npix = npix;
  }
  (void)P;
  return 0;
}

bool is_device_ptr(const void* p, int* dev) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    if (dev) *dev = a.device;
    return true;
  }
  return false;
}

bool is_pinned_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Device that owns a device (or managed) allocation, -1 for host memory.
int owning_device(const void* p) {
  int d = -1;
  return (p != nullptr && is_device_ptr(p, &d)) ? d : -1;
}

// Makes `dev` current for the scope and restores the caller's device afterwards.
struct DeviceGuard {
  int prev = -1;
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  cudaError_t set(int dev) {
    int cur = 0;
    cudaError_t e = cudaGetDevice(&cur);
    if (e != cudaSuccess || cur == dev) return e;
    e = cudaSetDevice(dev);
    if (e == cudaSuccess) prev = cur;
    return e;
  }
};

struct HostJob {
  const float* images;
  const uint16_t* images16;  // non-null: 16-bit input, widened to f32 on the device
  const float* inits;
  int W, H, P;
  int64_t lo, hi;
  const sf_config* cfg;
  float *par, *alpha, *beta, *nchi2;
  uint8_t *status, *iters;
  bool pinned_in, pinned_out;
  int copy_threads = 1;  // host threads for staging pageable input (par_memcpy)
  // results
  unsigned long long evals[3] = {0, 0, 0};
  double h2d_ms = 0, kernel_ms = 0, d2h_ms = 0;
  int chunks = 0;
  int chunks_u16 = 0;
  uint64_t h2d_bytes = 0;
  int rc = 0;
  std::string err;
};

// Pageable host input is staged into pinned buffers by the CPU.  One thread copies ~10 GB/s, far
// below PCIe (~53 GB/s), so large chunks are copied by copy_threads threads (the host's cores split
// over the devices of the call; SPOTFIT_COPY_THREADS overrides): sf::par_copy.
void par_memcpy(void* dst, const void* src, size_t bytes, int threads) { sf::par_copy(dst, src, bytes, threads); }

void copy_out_staged(Slot& s, HostJob& j) {
  if (!s.pending) return;
  const int P = j.P;
  const int64_t n = s.p_n, lo = s.p_lo;
  const float* o = s.h_out;
  const size_t cap = s.cap_spots;
  std::memcpy(j.par + lo * P, o, n * P * sizeof(float));
  std::memcpy(j.alpha + lo, o + cap * kMaxP, n * sizeof(float));
  std::memcpy(j.beta + lo, o + cap * (kMaxP + 1), n * sizeof(float));
  std::memcpy(j.nchi2 + lo, o + cap * (kMaxP + 2), n * sizeof(float));
  const uint8_t* b = reinterpret_cast<const uint8_t*>(o + cap * (kMaxP + 3));
  std::memcpy(j.status + lo, b, n);
  std::memcpy(j.iters + lo, b + cap, n);
  s.pending = false;
}

int run_shard(int dev, HostJob& j) {
  DeviceGuard guard;  // the caller's current device is restored on return
  SF_CUDA(guard.set(dev));
  DevCtx* c = ctx_for(dev);
  std::lock_guard<std::mutex> lk(c->mu);
  const int N = j.W * j.H, P = j.P;
  const int64_t total = j.hi - j.lo;
  if (total <= 0) return 0;
  sf::Geom geom;
  sf::build_geom(j.W, j.H, P, geom);
  sf::Cfg kc;
  if (make_cfg(j.cfg, j.W, j.H, kc) != 0) return -1;
  // Chunk schedule.  The host path is bound by the H2D copy engine (PCIe Gen5 x16: 53 GB/s at
  // 100 MB copies, 55.5 GB/s at 900 MB; tools/h2d_bw.py), so copies are large (<= 256 MB), and
  // the tail halves down to kMinChunk so that the kernel + D2H of the last chunk, which run
  // after the final H2D, are short.  Four streams overlap H2D(k+1) with kernel(k).
  const size_t px_bytes_in = j.images16 ? sizeof(uint16_t) : sizeof(float);
  // smallest chunk: total / 8 within [2048, 16384] spots, so that mid-size batches (1e4..1e5 spots)
  // still pipeline copy and fit over a few chunks (tools/call_overhead.py: 3e4 pageable spots
  // 1.81 -> 1.43 ms) while large ones keep 16384-spot tails
  const int64_t kMinChunk = std::min<int64_t>(16384, std::max<int64_t>(2048, total / 8));
  // chunk caps (MB of input per H2D), measured with tools/e2e_sweep.py on a B200 (PCIe Gen5 x16):
  // f32 input is copy-bound and flat above ~64 MB (96 MB best); u16 input is kernel-bound and
  // wants short chunks so that the first kernel starts early.  SPOTFIT_CHUNK_MB[16] override.
  auto env_mb = [](const char* name, int64_t dflt) {
    const char* e = std::getenv(name);
    const long v = e ? std::strtol(e, nullptr, 10) : 0;
    return (int64_t)(v > 0 ? v : dflt);
  };
  static const int64_t mb32 = env_mb("SPOTFIT_CHUNK_MB", 96), mb16 = env_mb("SPOTFIT_CHUNK_MB16", 24);
  const int64_t chunk_mb = j.images16 ? mb16 : mb32;
  const int64_t cap = std::max<int64_t>(kMinChunk, (chunk_mb << 20) / (int64_t)(px_bytes_in * N));
  const int64_t big = std::min<int64_t>(cap, std::max<int64_t>(kMinChunk, (total + 3) / 4));
  std::vector<std::pair<int64_t, int64_t>> chunks;  // (offset, spots)
  for (int64_t lo = 0; lo < total;) {
    const int64_t rem = total - lo;
    int64_t n = rem > 2 * big ? big : (rem <= 2 * kMinChunk ? rem : std::max<int64_t>(kMinChunk, rem / 2));
    chunks.emplace_back(lo, n);
    lo += n;
  }
  int64_t chunk = 0;
  for (const auto& ch : chunks) chunk = std::max(chunk, ch.second);
  const bool staging = !(j.pinned_in && j.pinned_out);
  // f32 chunks whose pixels are all integers in [0, 65535] cross PCIe as u16 (sf_host_narrow.cpp):
  // the host narrows them into pinned staging with streaming stores, half the bytes cross PCIe and
  // the fit kernel widens them back exactly.  Pageable input has to be staged by the CPU anyway;
  // for pinned input a share of the chunks is narrowed (below).  The first chunk that does not narrow
  // ends narrowing for the rest of the call (the pass gives up at its first bad value), so
  // non-integer data costs one partial pass.  SPOTFIT_NARROW=0 disables, =1 narrows pageable input only.
  static const int narrow_env = [] {
    const char* e = std::getenv("SPOTFIT_NARROW");
    return e ? (int)std::strtol(e, nullptr, 10) : 2;
  }();
  const bool narrow = narrow_env > 0 && !j.images16 && j.images != nullptr && (!j.pinned_in || narrow_env > 1);
  bool narrow_live = narrow;  // cleared by the first chunk that does not narrow (or narrows too slowly)
  bool probed = false;        // pinned input: the first narrowed chunk's probe has run
  // Pinned input: three chunks in four are narrowed (SPOTFIT_NARROW_PINNED percent, default 75; never
  // the first).  The others go as f32 straight from the caller's buffer, so the copy engine moves
  // them while the host narrows the next ones: the host's narrowing rate and PCIe add up
  // (profiles/r02_ab_narrow_pinned.txt: 7.7e7 15x15 fits/s vs 6.7-7.1e7 narrowing all, 5.9e7 none).
  static const int pinned_pct = [] {
    const char* e = std::getenv("SPOTFIT_NARROW_PINNED");
    const long v = e ? std::strtol(e, nullptr, 10) : 75;
    return (int)(v < 0 ? 0 : (v > 100 ? 100 : v));
  }();
  auto share = [&](size_t ci) {
    return !j.pinned_in || pinned_pct >= 100 ||
           (int64_t)(ci + 1) * pinned_pct / 100 > (int64_t)ci * pinned_pct / 100;
  };
  if (ensure_ctx(*c, dev, (size_t)chunk, N, P, staging, narrow) != 0) return -1;
  // reset the evaluation counters; the other slot streams wait on the device, not the host
  SF_CUDA(cudaMemsetAsync(c->d_evals, 0, 3 * sizeof(unsigned long long), c->slot[0].stream));
  SF_CUDA(cudaEventRecord(c->evals_zeroed, c->slot[0].stream));
  for (int k = 1; k < kStreams; ++k) SF_CUDA(cudaStreamWaitEvent(c->slot[k].stream, c->evals_zeroed, 0));
  // SPOTFIT_TRACE=1: per-chunk device timeline on stderr (diagnostic; tools/e2e_sweep.py)
  static const bool trace = std::getenv("SPOTFIT_TRACE") != nullptr;
  std::vector<cudaEvent_t> tev;
  auto mark = [&](cudaStream_t st) -> cudaError_t {
    if (!trace) return cudaSuccess;
    cudaEvent_t e;
    const cudaError_t r = cudaEventCreate(&e);
    if (r != cudaSuccess) return r;
    tev.push_back(e);
    return cudaEventRecord(e, st);
  };
  for (size_t ci = 0; ci < chunks.size(); ++ci) {
    Slot& s = c->slot[ci % kStreams];
    const int64_t lo = j.lo + chunks[ci].first;
    const int64_t n = chunks[ci].second;
    const bool nar = narrow_live && share(ci);
    if (staging || nar) {  // the slot's previous chunk must be finished before its staging is reused
      SF_CUDA(cudaEventSynchronize(s.ev[3]));
      if (staging) copy_out_staged(s, j);
    }
    SF_CUDA(cudaEventRecord(s.ev[0], s.stream));
    SF_CUDA(mark(s.stream));
    // this chunk as u16: 16-bit input, or f32 input whose pixels all narrow exactly
    // Pinned input is narrowed only while the host keeps up: narrowing that runs slower than the f32
    // bytes would cross PCIe (~50 GB/s, with 1.5x slack for the thread start-up) ends it for the call
    // -- e.g. several processes or devices sharing the host's cores and memory bandwidth.  The call's
    // first narrowed chunk is probed on its first half, so a slow host gives up after a partial pass
    // and sends the chunk as f32.
    auto narrow_part = [&](int64_t a, int64_t m, bool guard) -> int {  // 1 narrowed, 0 not integer, -1 too slow
      const auto t0 = std::chrono::steady_clock::now();
      if (!sf::par_narrow_u16(s.h_in16 + a * N, j.images + (lo + a) * N, (size_t)(m * N), j.copy_threads)) return 0;
      const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      return guard && t > 1.5 * (double)m * N * sizeof(float) / 50e9 ? -1 : 1;
    };
    bool u16 = j.images16 != nullptr;
    if (nar) {
      int r = 1;
      if (j.pinned_in && !probed) {
        probed = true;
        const int64_t m = std::max<int64_t>(1, n / 2);
        const int r0 = narrow_part(0, m, true);
        if (r0 == 1 && m < n) r = narrow_part(m, n - m, true);
        u16 = r0 == 1 && r != 0;  // a slow probe leaves the rest un-narrowed: the chunk goes as f32
        if (r0 != 1 || r != 1) narrow_live = false;
      } else {
        r = narrow_part(0, n, j.pinned_in);
        u16 = r != 0;  // narrowed (a slow pass still counts for this chunk, not for the next ones)
        if (r != 1) narrow_live = false;
      }
    }
    const size_t px_bytes = u16 ? sizeof(uint16_t) : sizeof(float);
    const void* src_img = j.images16 ? (const void*)(j.images16 + lo * N)
                                     : (u16 ? (const void*)s.h_in16 : (const void*)(j.images + lo * N));
    const float* src_init = j.inits ? j.inits + lo * P : nullptr;  // NULL: the fit kernel estimates them
    if (!j.pinned_in) {
      if (!(u16 && !j.images16)) {  // a narrowed chunk is already in pinned memory
        par_memcpy(s.h_in, src_img, n * N * px_bytes, j.copy_threads);
        src_img = s.h_in;
      }
      if (src_init) {
        std::memcpy(s.h_in + s.cap_spots * N, src_init, n * P * sizeof(float));
        src_init = s.h_in + s.cap_spots * N;
      }
    }
    // inits first, then pixels: the fit needs nothing else, so it can start (and fill the previous
    // fit's tail) as soon as the copy engine is done.  (A widening kernel between the two copies
    // made the init copy wait behind the next chunks' pixel copies: tools/e2e_trace.py.)
    if (src_init)
      SF_CUDA(cudaMemcpyAsync(s.d_init, src_init, n * P * sizeof(float), cudaMemcpyHostToDevice, s.stream));
    j.h2d_bytes += (uint64_t)n * N * px_bytes + (src_init ? (uint64_t)n * P * sizeof(float) : 0);
    j.chunks_u16 += u16 ? 1 : 0;
    if (u16) {
      SF_CUDA(cudaMemcpyAsync(s.d_img16, src_img, n * N * px_bytes, cudaMemcpyHostToDevice, s.stream));
      SF_CUDA(mark(s.stream));
    } else {
      SF_CUDA(cudaMemcpyAsync(s.d_img, src_img, n * N * px_bytes, cudaMemcpyHostToDevice, s.stream));
      SF_CUDA(mark(s.stream));
    }
    SF_CUDA(cudaEventRecord(s.ev[1], s.stream));
    SF_CUDA(mark(s.stream));
    sf::LaunchFit a;
    a.images = s.d_img;
    a.images16 = u16 ? s.d_img16 : nullptr;  // staged as u16 by the fit kernel itself
    a.inits = s.d_init;
    if (!j.inits) {  // no inits: estimate them on the device from the chunk just copied
      if (n <= sf::kFusedInitMaxSpots) {
        a.inits = nullptr;  // the fit kernel's fused initializer
      } else {
        // P = 5: (x, y, sigma, alpha, beta), as batch_engine._auto_inits builds it
        const cudaError_t e = u16 ? sf::launch_estimate_initial_u16(s.d_img16, j.W, j.H, n, P, kc.lo[2],
                                                                           kc.hi[2], s.d_init, nullptr, s.stream)
                                         : sf::launch_estimate_initial(s.d_img, j.W, j.H, n, P, kc.lo[2], kc.hi[2],
                                                                       s.d_init, nullptr, s.stream);
        if (e != cudaSuccess) return fail("initializer launch failed: %s", cudaGetErrorString(e));
      }
    }
    a.count = n;
    a.geom = geom;
    a.cfg = kc;
    a.out = sf::FitOut{s.d_par, s.d_a, s.d_b, s.d_c, s.d_st, s.d_it, c->d_evals};
    a.stream = s.stream;
    a.sm_count = c->sms;
    if (dispatch_fit(P, a) != 0) return -1;
    SF_CUDA(cudaEventRecord(s.ev[2], s.stream));
    SF_CUDA(mark(s.stream));
    if (j.pinned_out) {
      SF_CUDA(cudaMemcpyAsync(j.par + lo * P, s.d_par, n * P * sizeof(float), cudaMemcpyDeviceToHost, s.stream));
      SF_CUDA(cudaMemcpyAsync(j.alpha + lo, s.d_a, n * sizeof(float), cudaMemcpyDeviceToHost, s.stream));
      SF_CUDA(cudaMemcpyAsync(j.beta + lo, s.d_b, n * sizeof(float), cudaMemcpyDeviceToHost, s.stream));
      SF_CUDA(cudaMemcpyAsync(j.nchi2 + lo, s.d_c, n * sizeof(float), cudaMemcpyDeviceToHost, s.stream));
      SF_CUDA(cudaMemcpyAsync(j.status + lo, s.d_st, n, cudaMemcpyDeviceToHost, s.stream));
      SF_CUDA(cudaMemcpyAsync(j.iters + lo, s.d_it, n, cudaMemcpyDeviceToHost, s.stream));
    } else {
      float* o = s.h_out;
      const size_t cap = s.cap_spots;
      uint8_t* b = reinterpret_cast<uint8_t*>(o + cap * (kMaxP + 3));
      SF_CUDA(cudaMemcpyAsync(o, s.d_par, n * P * sizeof(float), cudaMemcpyDeviceToHost, s.stream));
      SF_CUDA(cudaMemcpyAsync(o + cap * kMaxP, s.d_a, n * sizeof(float), cudaMemcpyDeviceToHost, s.stream));
      SF_CUDA(cudaMemcpyAsync(o + cap * (kMaxP + 1), s.d_b, n * sizeof(float), cudaMemcpyDeviceToHost, s.stream));
      SF_CUDA(cudaMemcpyAsync(o + cap * (kMaxP + 2), s.d_c, n * sizeof(float), cudaMemcpyDeviceToHost, s.stream));
      SF_CUDA(cudaMemcpyAsync(b, s.d_st, n, cudaMemcpyDeviceToHost, s.stream));
      SF_CUDA(cudaMemcpyAsync(b + cap, s.d_it, n, cudaMemcpyDeviceToHost, s.stream));
      s.pending = true;
      s.p_lo = lo;
      s.p_n = n;
    }
    SF_CUDA(cudaEventRecord(s.ev[3], s.stream));
    SF_CUDA(mark(s.stream));
    ++j.chunks;
  }
  // the counters follow every chunk's fit: slot 0 waits for the other slots' last events, then
  // copies them back with its own results (no separate blocking copy afterwards)
  for (int k = 1; k < kStreams; ++k) SF_CUDA(cudaStreamWaitEvent(c->slot[0].stream, c->slot[k].ev[3], 0));
  SF_CUDA(cudaMemcpyAsync(c->h_evals, c->d_evals, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          c->slot[0].stream));
  for (auto& s : c->slot) {
    SF_CUDA(cudaStreamSynchronize(s.stream));
    if (staging) copy_out_staged(s, j);
  }
  if (trace && !tev.empty()) {  // per chunk: start, H2D images, H2D inits (+widen), fit, D2H (ms from chunk 0)
    for (size_t i = 0; i < tev.size(); ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[0], tev[i]);
      std::fprintf(stderr, "%s%.3f%s", i % 5 == 0 ? "TRACE " : "", ms, i % 5 == 4 ? "\n" : " ");
    }
    for (auto e : tev) cudaEventDestroy(e);
  }
  for (int k = 0; k < 3; ++k) j.evals[k] = c->h_evals[k];
  return 0;
}

}  // namespace

extern "C" {

int sf_version(void) { return SF_ABI_VERSION; }

int sf_simulate_device(const sf_sim_config* cfg, int32_t width, int32_t height, int64_t first_index, int64_t count,
                       float* d_images, float* d_truth, void* stream) {
  if (!cfg) return fail("cfg is NULL");
  if (check_grid(width, height) != 0) return -1;
  if (cfg->model != 3 && cfg->model != 4) return fail("model must be 3 or 4");
  if (count < 0) return fail("negative count");
  cudaError_t e = sf::launch_simulate(*cfg, width, height, first_index, count, d_images, d_truth,
                                      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail("simulator launch failed: %s", cudaGetErrorString(e));
  return 0;
}

int sf_debug_npexp_device(const float* d_x, float* d_y, int64_t n, int32_t variant, void* stream) {
  if (n < 0 || variant < 0 || variant > 2) return fail("bad arguments");
  cudaError_t e = sf::launch_npexp(d_x, d_y, n, variant, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail("npexp launch failed: %s", cudaGetErrorString(e));
  return 0;
}

int sf_debug_ddiv_device(const double* d_a, const double* d_b, double* d_out, int64_t n, void* stream) {
  if (n < 0) return fail("bad arguments");
  cudaError_t e = sf::launch_ddiv(d_a, d_b, d_out, n, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail("ddiv launch failed: %s", cudaGetErrorString(e));
  return 0;
}

int sf_debug_tame_div_device(uint64_t* d_mismatches, void* stream) {
  if (!d_mismatches) return fail("NULL buffer");
  cudaError_t e = sf::launch_tame_div(reinterpret_cast<unsigned long long*>(d_mismatches),
                                      static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail("tame_div launch failed: %s", cudaGetErrorString(e));
  return 0;
}

int sf_lane_geometry(int32_t width, int32_t height, int32_t* slots, int32_t* ppl, int16_t* nc, int16_t* nt,
                     int16_t* base, int16_t* tbase) {
  if (check_grid(width, height) != 0) return -1;
  sf::Geom g;
  const int need = sf::build_geom(width, height, 3, g);
  if (slots) *slots = g.slots;
  if (ppl) *ppl = need;
  for (int l = 0; l < g.lanes; ++l) {
    if (nc) nc[l] = g.nc[l];
    if (nt) nt[l] = g.nt[l];
    if (base) base[l] = g.base[l];
    if (tbase) tbase[l] = g.tbase[l];
  }
  return 0;
}

int sf_shard_range(int64_t count, int32_t shard, int32_t n_shards, int64_t* lo, int64_t* hi) {
  if (count < 0 || n_shards < 1 || shard < 0 || shard >= n_shards || !lo || !hi) return fail("bad shard arguments");
  // contiguous, order-preserving, sizes differ by at most one; exact in 128-bit
  *lo = (int64_t)((__int128)count * shard / n_shards);
  *hi = (int64_t)((__int128)count * (shard + 1) / n_shards);
  return 0;
}

const char* sf_last_error(void) { return g_err.c_str(); }

int sf_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

void* sf_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes ? bytes : 1, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    fail("cudaHostAlloc(%zu) failed", bytes);
    return nullptr;
  }
  return p;
}

void sf_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

static int fit_device_impl(const float* d_images, const uint16_t* d_images16, int32_t width, int32_t height,
                           int64_t count, const float* d_inits, const sf_config* cfg, float* d_params, float* d_alpha,
                           float* d_beta, float* d_nchi2, uint8_t* d_status, uint8_t* d_iters, uint64_t* d_evals,
                           void* stream) {
  if (check_grid(width, height) != 0) return -1;
  if (count < 0) return fail("negative count");
  sf::Cfg kc;
  if (make_cfg(cfg, width, height, kc) != 0) return -1;
  if (count == 0) return 0;
  if ((!d_images && !d_images16) || !d_params || !d_alpha || !d_beta || !d_nchi2 || !d_status || !d_iters)
    return fail("NULL buffer");  // d_inits may be NULL: the fit kernel estimates them (fused initializer)
  // launch on the device that owns the pixels (the current device for device-mapped host memory)
  DeviceGuard guard;
  const int owner = owning_device(d_images ? (const void*)d_images : (const void*)d_images16);
  if (owner >= 0) SF_CUDA(guard.set(owner));
  sf::Geom geom;
  sf::build_geom(width, height, cfg->model, geom);
  sf::LaunchFit a;
  a.images = d_images;
  a.images16 = d_images16;
  a.inits = d_inits;
  a.count = count;
  a.geom = geom;
  a.cfg = kc;
  a.out = sf::FitOut{d_params, d_alpha, d_beta, d_nchi2, d_status, d_iters,
                     reinterpret_cast<unsigned long long*>(d_evals)};
  a.stream = static_cast<cudaStream_t>(stream);
  a.sm_count = sm_count_of_current();
  float* tmp = nullptr;
  if (!d_inits && count > sf::kFusedInitMaxSpots) {
    // large batch without inits: the standalone initializer into a stream-ordered scratch buffer
    // in front of the fit (the fused initializer is the small-batch / latency path)
    const int P = cfg->model;
    SF_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&tmp), (size_t)count * P * sizeof(float), a.stream));
    const cudaError_t e = d_images16
                              ? sf::launch_estimate_initial_u16(d_images16, width, height, count, P, kc.lo[2],
                                                                kc.hi[2], tmp, nullptr, a.stream)
                              : sf::launch_estimate_initial(d_images, width, height, count, P, kc.lo[2], kc.hi[2],
                                                            tmp, nullptr, a.stream);
    if (e != cudaSuccess) {
      cudaFreeAsync(tmp, a.stream);
      return fail("initializer launch failed: %s", cudaGetErrorString(e));
    }
    a.inits = tmp;
  }
  const int rc = dispatch_fit(cfg->model, a);
  if (tmp) SF_CUDA(cudaFreeAsync(tmp, a.stream));
  return rc;
}

int sf_fit_batch_device(const float* d_images, int32_t width, int32_t height, int64_t count, const float* d_inits,
                        const sf_config* cfg, float* d_params, float* d_alpha, float* d_beta, float* d_nchi2,
                        uint8_t* d_status, uint8_t* d_iters, uint64_t* d_evals, void* stream) {
  return fit_device_impl(d_images, nullptr, width, height, count, d_inits, cfg, d_params, d_alpha, d_beta, d_nchi2,
                         d_status, d_iters, d_evals, stream);
}

int sf_fit_batch_device_u16(const uint16_t* d_images, int32_t width, int32_t height, int64_t count,
                            const float* d_inits, const sf_config* cfg, float* d_params, float* d_alpha,
                            float* d_beta, float* d_nchi2, uint8_t* d_status, uint8_t* d_iters, uint64_t* d_evals,
                            void* stream) {
  if (!d_images && count > 0) return fail("NULL buffer");
  return fit_device_impl(nullptr, d_images, width, height, count, d_inits, cfg, d_params, d_alpha, d_beta, d_nchi2,
                         d_status, d_iters, d_evals, stream);
}

int sf_eval_batch_device(const float* d_images, int32_t width, int32_t height, int64_t count, int32_t model,
                         const float* d_params, sf_eval_record* d_out, void* stream) {
  if (check_grid(width, height) != 0) return -1;
  if (model != 3 && model != 4) return fail("model must be 3 or 4");
  if (count < 0) return fail("negative count");
  if (count == 0) return 0;
  if (!d_images || !d_params || !d_out) return fail("NULL buffer");
  DeviceGuard guard;
  const int owner = owning_device(d_images);
  if (owner >= 0) SF_CUDA(guard.set(owner));
  sf::Geom geom;
  sf::build_geom(width, height, model, geom);
  sf::LaunchEval a;
  a.images = d_images;
  a.params = d_params;
  a.count = count;
  a.geom = geom;
  a.out = d_out;
  a.stream = static_cast<cudaStream_t>(stream);
  return dispatch_eval(model, a);
}

static int model_args(int n, int model, int64_t count) {
  if (n < 1 || n > 1024) return fail("n = %d pixels per spot: need 1..1024 (model.py:55-58)", n);
  if (model != 3 && model != 4) return fail("model must be 3 or 4");
  if (count < 0) return fail("negative count");
  return 0;
}

#define SF_LAUNCHED(call)                                                            \
  do {                                                                               \
    const cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) return fail("%s: %s", #call, cudaGetErrorString(e_));     \
    return 0;                                                                        \
  } while (0)

int sf_model_profile_device(const float* d_params, int32_t width, int32_t height, int64_t count, int32_t model,
                            float* d_f, float* d_fgrad, void* stream) {
  if (check_grid(width, height) != 0 || model_args(width * height, model, count) != 0) return -1;
  if (count > 0 && (!d_params || !d_f)) return fail("NULL buffer");
  DeviceGuard guard;
  const int owner = owning_device(d_params);
  if (owner >= 0) SF_CUDA(guard.set(owner));
  SF_LAUNCHED(sf::launch_model_profile(d_params, width, height, count, model, d_f, d_fgrad,
                                       static_cast<cudaStream_t>(stream)));
}

int sf_model_alpha_beta_device(const float* d_f, const float* d_g, int32_t n, int64_t count, float* d_alpha,
                               float* d_beta, double* d_sums, int32_t* d_singular, void* stream) {
  if (model_args(n, 3, count) != 0) return -1;
  if (count > 0 && (!d_f || !d_g || !d_alpha || !d_beta || !d_sums || !d_singular)) return fail("NULL buffer");
  DeviceGuard guard;
  const int owner = owning_device(d_f);
  if (owner >= 0) SF_CUDA(guard.set(owner));
  SF_LAUNCHED(sf::launch_model_alpha_beta(d_f, d_g, n, count, d_alpha, d_beta, d_sums, d_singular,
                                          static_cast<cudaStream_t>(stream)));
}

int sf_model_chi_squared_device(const float* d_g, const float* d_f, const float* d_alpha, const float* d_beta,
                                int32_t n, int64_t count, float* d_h, float* d_r, float* d_chi, void* stream) {
  if (model_args(n, 3, count) != 0) return -1;
  if (count > 0 && (!d_g || !d_f || !d_alpha || !d_beta || !d_chi)) return fail("NULL buffer");
  DeviceGuard guard;
  const int owner = owning_device(d_f);
  if (owner >= 0) SF_CUDA(guard.set(owner));
  SF_LAUNCHED(sf::launch_model_chi(d_g, d_f, d_alpha, d_beta, n, count, d_h, d_r, d_chi,
                                   static_cast<cudaStream_t>(stream)));
}

int sf_model_gradient_sums_device(const float* d_f, const float* d_fgrad, const float* d_g, const double* d_sums,
                                  int32_t n, int32_t model, int64_t count, double* d_gsums, void* stream) {
  if (model_args(n, model, count) != 0) return -1;
  if (count > 0 && (!d_f || !d_fgrad || !d_g || !d_sums || !d_gsums)) return fail("NULL buffer");
  DeviceGuard guard;
  const int owner = owning_device(d_f);
  if (owner >= 0) SF_CUDA(guard.set(owner));
  SF_LAUNCHED(sf::launch_model_gradient_sums(d_f, d_fgrad, d_g, d_sums, n, model, count, d_gsums,
                                             static_cast<cudaStream_t>(stream)));
}

int sf_model_coefficient_gradients_device(const double* d_sums, const double* d_gsums, const float* d_alpha,
                                          const float* d_beta, int32_t n, int32_t model, int64_t count,
                                          double* d_dalpha, double* d_dbeta, int32_t* d_singular, void* stream) {
  if (model_args(n, model, count) != 0) return -1;
  if (count > 0 && (!d_sums || !d_gsums || !d_alpha || !d_beta || !d_dalpha || !d_dbeta || !d_singular))
    return fail("NULL buffer");
  DeviceGuard guard;
  const int owner = owning_device(d_sums);
  if (owner >= 0) SF_CUDA(guard.set(owner));
  SF_LAUNCHED(sf::launch_model_coefficient_gradients(d_sums, d_gsums, d_alpha, d_beta, n, model, count, d_dalpha,
                                                     d_dbeta, d_singular, static_cast<cudaStream_t>(stream)));
}

int sf_model_chi_gradient_device(const float* d_g, const float* d_f, const float* d_fgrad, const float* d_alpha,
                                 const float* d_beta, const double* d_dalpha, const double* d_dbeta, int32_t n,
                                 int32_t model, int64_t count, double* d_grad, float* d_dmat, void* stream) {
  if (model_args(n, model, count) != 0) return -1;
  if (count > 0 && (!d_g || !d_f || !d_fgrad || !d_alpha || !d_beta || !d_dalpha || !d_dbeta || !d_grad))
    return fail("NULL buffer");
  DeviceGuard guard;
  const int owner = owning_device(d_f);
  if (owner >= 0) SF_CUDA(guard.set(owner));
  SF_LAUNCHED(sf::launch_model_chi_gradient(d_g, d_f, d_fgrad, d_alpha, d_beta, d_dalpha, d_dbeta, n, model, count,
                                            d_grad, d_dmat, static_cast<cudaStream_t>(stream)));
}

int sf_estimate_initial_device(const float* d_images, int32_t width, int32_t height, int64_t count, int32_t model,
                               double sigma_min, double sigma_max, float* d_inits, float* d_amps, void* stream) {
  if (check_grid(width, height) != 0) return -1;
  if (model != 3 && model != 4) return fail("model must be 3 or 4");
  if (count < 0) return fail("negative count");
  if (!(sigma_min > 0) || !(sigma_max > sigma_min)) return fail("need 0 < sigma_min < sigma_max");
  if (count > 0 && (!d_images || !d_inits)) return fail("NULL buffer");
  DeviceGuard guard;
  const int owner = owning_device(d_images);
  if (owner >= 0) SF_CUDA(guard.set(owner));
  cudaError_t e = sf::launch_estimate_initial(d_images, width, height, count, model, sigma_min, sigma_max, d_inits,
                                              d_amps, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail("initializer launch failed: %s", cudaGetErrorString(e));
  return 0;
}

static int fit_batch_impl(const float* images, const uint16_t* images16, int32_t width, int32_t height,
                          int64_t count, const float* inits, const sf_config* cfg, float* out_params,
                          float* out_alpha, float* out_beta, float* out_nchi2, uint8_t* out_status, uint8_t* out_iters,
                          const int32_t* devices, int32_t n_devices, sf_stats* stats);

int sf_fit_batch(const float* images, int32_t width, int32_t height, int64_t count, const float* inits,
                 const sf_config* cfg, float* out_params, float* out_alpha, float* out_beta, float* out_nchi2,
                 uint8_t* out_status, uint8_t* out_iters, const int32_t* devices, int32_t n_devices,
                 sf_stats* stats) {
  return fit_batch_impl(images, nullptr, width, height, count, inits, cfg, out_params, out_alpha, out_beta, out_nchi2,
                        out_status, out_iters, devices, n_devices, stats);
}

int sf_fit_batch_u16(const uint16_t* images, int32_t width, int32_t height, int64_t count, const float* inits,
                     const sf_config* cfg, float* out_params, float* out_alpha, float* out_beta, float* out_nchi2,
                     uint8_t* out_status, uint8_t* out_iters, const int32_t* devices, int32_t n_devices,
                     sf_stats* stats) {
  if (images && is_device_ptr(images, nullptr)) return fail("sf_fit_batch_u16 takes host images");
  return fit_batch_impl(nullptr, images, width, height, count, inits, cfg, out_params, out_alpha, out_beta,
                        out_nchi2, out_status, out_iters, devices, n_devices, stats);
}

}  // extern "C"

static int fit_batch_impl(const float* images, const uint16_t* images16, int32_t width, int32_t height,
                          int64_t count, const float* inits, const sf_config* cfg, float* out_params,
                          float* out_alpha, float* out_beta, float* out_nchi2, uint8_t* out_status, uint8_t* out_iters,
                          const int32_t* devices, int32_t n_devices, sf_stats* stats) {
  const auto t0 = std::chrono::steady_clock::now();
  if (check_grid(width, height) != 0) return -1;
  if (count < 0) return fail("negative count");
  sf::Cfg kc;
  if (make_cfg(cfg, width, height, kc) != 0) return -1;
  if (stats) std::memset(stats, 0, sizeof(*stats));
  if (count == 0) return 0;
  if ((!images && !images16) || !out_params || !out_alpha || !out_beta || !out_nchi2 || !out_status || !out_iters)
    return fail("NULL buffer");  // inits may be NULL: estimated by the fit kernel (fused initializer)
  int ndev_avail = sf_device_count();
  if (ndev_avail < 1) return fail("no CUDA device available (the CUDA engine has no CPU fallback)");
  std::vector<int> devs;
  if (devices && n_devices > 0) {
    for (int i = 0; i < n_devices; ++i) {
      if (devices[i] < 0 || devices[i] >= ndev_avail) return fail("device %d out of range", devices[i]);
      devs.push_back(devices[i]);
    }
  } else {
    devs.push_back(0);
  }
  int dptr_dev = -1;
  const void* outs[] = {inits, out_params, out_alpha, out_beta, out_nchi2, out_status, out_iters};
  const char* names[] = {"inits", "out_params", "out_alpha", "out_beta", "out_nchi2", "out_status", "out_iters"};
  if (images && is_device_ptr(images, &dptr_dev)) {
    // device-resident batch: one device, synchronous call on the library stream; every other
    // array must live on the same device (a host output would be written through a device store)
    if (devs.size() > 1) return fail("device-pointer batches run on the owning device only");
    for (int i = 0; i < 7; ++i) {
      int d = -1;
      if (outs[i] == nullptr) continue;  // NULL inits: fused initializer
      if (!is_device_ptr(outs[i], &d) || d != dptr_dev)
        return fail("mixed arguments: images are device memory of device %d but %s is not", dptr_dev, names[i]);
    }
    DeviceGuard guard;
    SF_CUDA(guard.set(dptr_dev));
    DevCtx* c = ctx_for(dptr_dev);
    std::lock_guard<std::mutex> lk(c->mu);
    if (ensure_ctx(*c, dptr_dev, 1, width * height, cfg->model, false, false) != 0) return -1;
    cudaStream_t st = c->slot[0].stream;
    SF_CUDA(cudaMemsetAsync(c->d_evals, 0, 3 * sizeof(unsigned long long), st));
    SF_CUDA(cudaEventRecord(c->slot[0].ev[1], st));
    if (sf_fit_batch_device(images, width, height, count, inits, cfg, out_params, out_alpha, out_beta, out_nchi2,
                            out_status, out_iters, reinterpret_cast<uint64_t*>(c->d_evals), st) != 0)
      return -1;
    SF_CUDA(cudaEventRecord(c->slot[0].ev[2], st));
    SF_CUDA(cudaStreamSynchronize(st));
    if (stats) {
      unsigned long long ev[3];
      SF_CUDA(cudaMemcpy(ev, c->d_evals, sizeof(ev), cudaMemcpyDeviceToHost));
      float ms = 0;
      cudaEventElapsedTime(&ms, c->slot[0].ev[1], c->slot[0].ev[2]);
      stats->n_gradient_evals = ev[0];
      stats->n_trial_evals = ev[1];
      stats->n_kernel_evals = ev[2];
      stats->kernel_ms = ms;
      stats->n_devices = 1;
      stats->n_chunks = 1;
      stats->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return 0;
  }
  for (int i = 0; i < 7; ++i)  // host images: every array is host memory (staged / DMA'd by the pipeline)
    if (outs[i] != nullptr && is_device_ptr(outs[i], nullptr)) return fail("mixed arguments: images are host memory but %s is device "
                                                     "memory", names[i]);
  const bool pin_in =
      is_pinned_ptr(images ? (const void*)images : (const void*)images16) && (!inits || is_pinned_ptr(inits));
  const bool pin_out = is_pinned_ptr(out_params) && is_pinned_ptr(out_alpha) && is_pinned_ptr(out_beta) &&
                       is_pinned_ptr(out_nchi2) && is_pinned_ptr(out_status) && is_pinned_ptr(out_iters);
  const int nd = (int)devs.size();
  std::vector<HostJob> jobs(nd);
  int copy_threads = (int)std::thread::hardware_concurrency() / nd;
  if (const char* e = std::getenv("SPOTFIT_COPY_THREADS")) copy_threads = (int)std::strtol(e, nullptr, 10);
  copy_threads = std::max(1, std::min(copy_threads, 16));
  for (int d = 0; d < nd; ++d) {
    HostJob& j = jobs[d];
    j.images = images;
    j.images16 = images16;
    j.inits = inits;
    j.W = width;
    j.H = height;
    j.P = cfg->model;
    sf_shard_range(count, d, nd, &j.lo, &j.hi);
    j.cfg = cfg;
    j.par = out_params;
    j.alpha = out_alpha;
    j.beta = out_beta;
    j.nchi2 = out_nchi2;
    j.status = out_status;
    j.iters = out_iters;
    j.pinned_in = pin_in;
    j.pinned_out = pin_out;
    j.copy_threads = copy_threads;
  }
  std::vector<std::thread> th;
  for (int d = 1; d < nd; ++d)
    th.emplace_back([&, d]() {
      jobs[d].rc = run_shard(devs[d], jobs[d]);
      if (jobs[d].rc != 0) jobs[d].err = g_err;
    });
  jobs[0].rc = run_shard(devs[0], jobs[0]);
  if (jobs[0].rc != 0) jobs[0].err = g_err;
  for (auto& t : th) t.join();
  for (int d = 0; d < nd; ++d)
    if (jobs[d].rc != 0) return fail("device %d: %s", devs[d], jobs[d].err.c_str());
  if (stats) {
    for (auto& j : jobs) {
      stats->n_gradient_evals += j.evals[0];
      stats->n_trial_evals += j.evals[1];
      stats->n_kernel_evals += j.evals[2];
      stats->n_chunks += j.chunks;
      stats->n_chunks_u16 += j.chunks_u16;
      stats->h2d_bytes += j.h2d_bytes;
    }
    stats->n_devices = nd;
    stats->total_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return 0;
}
