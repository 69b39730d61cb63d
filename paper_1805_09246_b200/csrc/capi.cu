// capi.cu — host side of the C ABI declared in include/srlg.h.
//
// Handles own u32 stamp arrays on one device plus an O(1) host clock
// (slides / now / floor). Every device operation of a device runs on that
// device's single in-order stream, so all calls see a consistent state and
// the detection scratch can be shared. Host-side double arithmetic uses the
// reference's exact expressions (src/linear_counting.cpp:10-24,
// src/slea.cpp:57-61, 85-95) and is compiled with -ffp-contract=off.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstddef>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "srlg_internal.cuh"

using namespace srlg;
using dev::EngineOp;
using dev::EngineRing;
using dev::InboxHeader;
using dev::InboxRank;
using dev::kInboxMaxCtas;
using dev::kInboxSlots;

namespace {

// ------------------------------------------------------------------ errors

thread_local std::string g_err;

struct Failure {
  int code;
  std::string msg;
};

[[noreturn]] void raise(int code, const std::string& msg) { throw Failure{code, msg}; }

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) raise(SRLG_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SRLG_OK;
  } catch (const Failure& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SRLG_ERR_RESOURCE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SRLG_ERR_RESOURCE;
  }
}

std::atomic<uint64_t> g_launches{0};

// -------------------------------------------------------- device buffers

// Buffers grow geometrically and a replaced buffer is released only at exit:
// cudaFree / cudaFreeHost synchronise the whole device, which would wait on
// the persistent kernels of other execution lanes (a merge group's peers,
// themselves waiting on this lane) — nothing on a lane's call path may
// synchronise the device.
std::mutex g_retired_mu;
std::vector<std::pair<void*, bool>> g_retired;  // {pointer, pinned host}

void retire(void* p, bool host) {
  std::lock_guard<std::mutex> lk(g_retired_mu);
  g_retired.emplace_back(p, host);
}

uint64_t grown(uint64_t have, uint64_t want) {
  return have ? std::max(want, have + have / 2) : want;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  uint64_t n = 0;
  void ensure(uint64_t want) {
    if (want <= n) return;
    want = grown(n, want);
    if (p) retire(p, false);
    p = nullptr;
    n = 0;
    cuda_ok(cudaMalloc(&p, std::max<uint64_t>(want, 1) * sizeof(T)), "cudaMalloc (scratch)");
    // zero-filled before first use (the overlap tables rely on it); rare path.
    // The memset runs on the legacy stream, which the library's non-blocking
    // streams do not synchronise with: wait for it alone.
    cuda_ok(cudaMemset(p, 0, std::max<uint64_t>(want, 1) * sizeof(T)), "cudaMemset (scratch)");
    cuda_ok(cudaStreamSynchronize(cudaStreamLegacy), "cudaStreamSynchronize");
    n = want;
  }
};

template <class T>
struct HostBuf {  // pinned and mapped: kernels write results straight into it
  T* p = nullptr;
  T* dptr = nullptr;
  uint64_t n = 0;
  void ensure(uint64_t want) {
    if (want <= n) return;
    want = grown(n, want);
    if (p) retire(p, true);
    p = dptr = nullptr;
    n = 0;
    cuda_ok(cudaHostAlloc(reinterpret_cast<void**>(&p), std::max<uint64_t>(want, 1) * sizeof(T),
                          cudaHostAllocMapped | cudaHostAllocPortable),
            "cudaHostAlloc");
    std::memset(static_cast<void*>(p), 0, std::max<uint64_t>(want, 1) * sizeof(T));
    cuda_ok(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dptr), p, 0), "mapped pointer");
    n = want;
  }
};

// detection slot: device result + candidates, pinned mirrors, completion event
constexpr uint64_t kCandPrefix = 1024;

struct Slot {
  DevBuf<WinResult> res_d;
  DevBuf<Candidate> cand_d;
  HostBuf<WinResult> res_h;
  HostBuf<Candidate> cand_h;
  cudaEvent_t ev = nullptr;
};

// ------------------------------------------------------ per-device context

constexpr uint64_t kStagePairs = 1ull << 23;  // 64 MB of pairs per staging buffer
constexpr uint64_t kResidentPairs = 1ull << 31;  // pinned input up to 16 GB is copied whole
constexpr uint64_t kChunkPairs = 1ull << 20;     // 8 MB host-input copy chunks (streamed runs)
constexpr int kStageBufs = 2;

// Optional per-launch CUDA-event timing on the compute stream (bench
// instrumentation): kind 0 = packet scan (K1), kind 1 = detection pipeline.
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  struct Span {
    int kind;
    size_t a, b;
  };
  std::vector<Span> spans;
  double ms[3] = {0, 0, 0};  // kind 2 = persistent engine batch
  uint64_t count[3] = {0, 0, 0};
  uint64_t units[3] = {0, 0, 0};

  cudaEvent_t next() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cuda_ok(cudaEventCreate(&e), "event");
      pool.push_back(e);
    }
    return pool[used++];
  }
  size_t begin(cudaStream_t st) {
    const size_t i = used;
    cuda_ok(cudaEventRecord(next(), st), "record");
    return i;
  }
  void end(cudaStream_t st, int kind, size_t a, uint64_t u) {
    const size_t b = used;
    cuda_ok(cudaEventRecord(next(), st), "record");
    spans.push_back(Span{kind, a, b});
    units[kind] += u;
  }
  // after the stream has drained
  void collect() {
    for (const Span& s : spans) {
      float t = 0;
      cuda_ok(cudaEventElapsedTime(&t, pool[s.a], pool[s.b]), "elapsed");
      ms[s.kind] += t;
      count[s.kind]++;
    }
    spans.clear();
    used = 0;
  }
};

struct DeviceCtx {
  int device = 0;
  int n_sms = 148;
  cudaStream_t st = nullptr;  // compute stream (all state access)
  cudaStream_t cp = nullptr;  // host->device copies
  cudaStream_t cp2 = nullptr; // second copy stream (streamed engine input alternates chunks)
  std::recursive_mutex mu;
  // host-input staging (double buffered)
  srlg_pair* stage_d[kStageBufs] = {};
  srlg_pair* stage_h[kStageBufs] = {};
  cudaEvent_t h2d_done[kStageBufs] = {};
  cudaEvent_t scan_done[kStageBufs] = {};
  int next_stage = 0;
  // detection scratch (stream-ordered reuse)
  DevBuf<uint32_t> hot_bits, hot_cols, partials, tuples_a, tuples_b;
  DevBuf<unsigned long long> tables;  // zero-initialised; entries carry a launch generation
  DevBuf<uint32_t> le_bits;           // SLEA inside bitmap of the current detection
  DevBuf<uint32_t> dfs_scratch;       // reconstruction: per-thread walk state (DetectParams)
  DevBuf<uint32_t> left;              // detection: candidates weighed by the publishing CTA
  // pinned host input of a pre-sliced engine run is copied whole into this
  // buffer, chunk by chunk on the copy stream, so the copy engine streams
  // without waiting for staging buffers to drain
  DevBuf<srlg_pair> input_d;
  DevBuf<unsigned> chunk_flags;  // set by the copy stream (cuStreamWriteValue32) per chunk
  std::vector<cudaEvent_t> chunk_ev;
  cudaEvent_t chunk_event(size_t i) {
    while (chunk_ev.size() <= i) {
      cudaEvent_t e;
      cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
      chunk_ev.push_back(e);
    }
    return chunk_ev[i];
  }
  // second and third buffer sets of the per-detection state (engine pipelining)
  // buffer sets 1 .. kMaxSets - 1 of the per-detection state (set 0 is the
  // detection scratch above): engine detection d uses set d % n_sets
  struct SetBufs {
    DevBuf<uint32_t> hot_cols, le_bits, left;
    DevBuf<unsigned long long> tables;
    DetectScratch* scratch = nullptr;
  };
  SetBufs extra[kMaxSets - 1];
  // incremental window tracking of engine launches (srlg_internal.cuh IncDev);
  // rebuilt by the first detection of every launch
  DevBuf<uint32_t> rs_smin, le_smin, live_bits;
  DevBuf<uint8_t> live_hot;
  DevBuf<unsigned long long> live_row;
  DevBuf<unsigned long long> inc_stats;  // diagnostics: srlg_engine_inc_stats
  DevBuf<uint32_t> le_log_idx, le_log_n;  // SLEA tracked: per detection and CTA, changed live words
  DevBuf<unsigned long long> le_log_val;
  uint32_t serial = 0;                // detection serials (overlap-table generations)
  uint32_t next_serial() {
    if (++serial == 0) serial = 1;
    return serial;
  }
  DevBuf<uint16_t> u16tmp;
  DevBuf<uint32_t> u32tmp;
  DevBuf<unsigned long long> u64tmp;
  Slot sync_slot;
  DetectScratch* scratch = nullptr;
  unsigned* bar = nullptr;
  int detect_grid = 0;
  int cta_budget = 0;  // execution lanes: CTAs of the persistent kernels (0 = one per SM)
  Profiler prof;

  void ensure_detect() {
    if (scratch) return;
    cuda_ok(cudaMalloc(&scratch, sizeof(DetectScratch)), "cudaMalloc (detect scratch)");
    cuda_ok(cudaMemsetAsync(scratch, 0, sizeof(DetectScratch), st), "memset");
    cuda_ok(cudaMalloc(&bar, 4096), "cudaMalloc (grid barrier)");
    cuda_ok(cudaMemsetAsync(bar, 0, 4096, st), "memset");
    detect_grid = dev::detect_grid(device);
    if (cta_budget > 0) detect_grid = std::min(detect_grid, cta_budget);
  }
  uint64_t h2d_bytes = 0, d2h_bytes = 0;

  void init(int dev) {
    device = dev;
    cuda_ok(cudaSetDevice(dev), "cudaSetDevice");
    cuda_ok(cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, dev), "attr");
    cuda_ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    cuda_ok(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking), "stream");
    cuda_ok(cudaStreamCreateWithFlags(&cp2, cudaStreamNonBlocking), "stream");
    for (int i = 0; i < kStageBufs; ++i) {
      cuda_ok(cudaEventCreateWithFlags(&h2d_done[i], cudaEventDisableTiming), "event");
      cuda_ok(cudaEventCreateWithFlags(&scan_done[i], cudaEventDisableTiming), "event");
    }
    cuda_ok(cudaEventCreateWithFlags(&sync_slot.ev, cudaEventDisableTiming), "event");
  }

  void ensure_staging() {
    if (stage_d[0]) return;
    for (int i = 0; i < kStageBufs; ++i) {
      cuda_ok(cudaMalloc(&stage_d[i], kStagePairs * sizeof(srlg_pair)), "cudaMalloc (staging)");
      cuda_ok(cudaMallocHost(&stage_h[i], kStagePairs * sizeof(srlg_pair)), "cudaMallocHost");
    }
  }

  void sync() { cuda_ok(cudaStreamSynchronize(st), "cudaStreamSynchronize"); }
};

std::mutex g_ctx_mu;
DeviceCtx* g_ctx[64] = {};
// execution lanes (srlg_lane_create): further contexts on a physical device,
// each with its own streams, scratch and CTA budget, addressed as device
// ordinals kLaneBase + i
constexpr int kLaneBase = 64;
DeviceCtx* g_lane[64] = {};
int g_n_lanes = 0;

DeviceCtx& ctx_for(int device) {
  if (device >= kLaneBase && device < kLaneBase + 64) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (!g_lane[device - kLaneBase]) raise(SRLG_ERR_INVALID_ARGUMENT, "unknown execution lane");
    return *g_lane[device - kLaneBase];
  }
  if (device < 0 || device >= 64) raise(SRLG_ERR_INVALID_ARGUMENT, "bad device ordinal");
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  if (!g_ctx[device]) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      raise(SRLG_ERR_CUDA, "no CUDA device available (the srlg path has no CPU fallback)");
    if (device >= n) raise(SRLG_ERR_INVALID_ARGUMENT, "device ordinal out of range");
    auto* c = new DeviceCtx();
    c->init(device);
    g_ctx[device] = c;
  }
  return *g_ctx[device];
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cuda_ok(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

bool is_pinned_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// ------------------------------------------------------- host restatements

// sampling_threshold (src/hash.cpp:10-16)
uint32_t sampling_threshold(uint64_t theta, uint64_t eta) {
  if (eta == 0) raise(SRLG_ERR_CONFIG, "sampling threshold: eta must be positive");
  uint32_t t = 0;
  while (t < 64 && eta <= (UINT64_MAX >> t) && (eta << t) < theta) ++t;
  return t;
}

// detection_rho (src/sliding_counters.cpp:50)
double detection_rho() { return 0.99 * (1.0 - std::exp(-1.0 / 3.0)); }

// smallest integer weight w with double(w) >= rho * eta (rsra.cpp:46, 52)
uint32_t hot_min_weight(uint32_t eta) {
  const double threshold = detection_rho() * static_cast<double>(eta);
  uint32_t w = static_cast<uint32_t>(std::max(0.0, std::floor(threshold)));
  while (w > 0 && static_cast<double>(w - 1) >= threshold) --w;
  while (static_cast<double>(w) < threshold) ++w;
  return w;
}

// le_estimate (src/linear_counting.cpp:10-15)
void le_estimate(double weight, uint32_t eta_prime, double* value, bool* saturated) {
  const double eta = static_cast<double>(eta_prime);
  if (weight <= 0.0) {
    *value = 0.0;
    *saturated = false;
  } else if (weight >= eta) {
    *value = eta * std::log(eta);
    *saturated = true;
  } else {
    *value = -eta * std::log((eta - weight) / eta);
    *saturated = false;
  }
}

// corrected_weight (src/linear_counting.cpp:17-24)
double corrected_weight(double usle, double sfp, uint32_t eta_prime) {
  if (sfp >= 1.0)
    raise(SRLG_ERR_SATURATION, "corrected weight: setting-factor product is 1, estimate unusable");
  if (sfp < 0.0) sfp = 0.0;
  const double eta = static_cast<double>(eta_prime);
  const double w = (usle - eta * sfp) / (1.0 - sfp);
  return std::clamp(w, 0.0, eta);
}

constexpr double kSaturationEps = 1e-9;  // linear_counting.hpp:8

// ------------------------------------------------------------------- NCCL
// Loaded at run time (dlopen): the library has no link-time NCCL dependency,
// and inside a torch process it shares torch's already-loaded libnccl.
struct NcclApi {
  bool loaded = false;
  decltype(&ncclGetUniqueId) getUniqueId = nullptr;
  decltype(&ncclCommInitRank) commInitRank = nullptr;
  decltype(&ncclCommDestroy) commDestroy = nullptr;
  decltype(&ncclReduce) reduce = nullptr;
  decltype(&ncclAllReduce) allReduce = nullptr;
  decltype(&ncclGetErrorString) errorString = nullptr;
};

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.reduce = reinterpret_cast<decltype(a.reduce)>(dlsym(h, "ncclReduce"));
    a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
    a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(h, "ncclGetErrorString"));
    a.loaded = a.getUniqueId && a.commInitRank && a.commDestroy && a.reduce && a.allReduce &&
               a.errorString;
    return a;
  }();
  if (!api.loaded) raise(SRLG_ERR_CUDA, "NCCL (libnccl.so.2) could not be loaded");
  return api;
}

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) raise(SRLG_ERR_CUDA, std::string(what) + ": " + nccl().errorString(r));
}

}  // namespace

// ------------------------------------------------------- stream memory ops
// cuStreamWriteValue32 from the driver, looked up at run time (no link-time
// libcuda dependency): the copy stream flags each host-input chunk as it lands
using WriteValue32Fn = int (*)(cudaStream_t, unsigned long long, uint32_t, unsigned);

WriteValue32Fn write_value32() {
  static WriteValue32Fn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<WriteValue32Fn>(nullptr);
    }
    return reinterpret_cast<WriteValue32Fn>(f);
  }();
  return fn;
}

// ----------------------------------------------------------------- handles

struct srlg_rsra {
  srlg_rsra_config cfg{};
  DeviceCtx* ctx = nullptr;
  uint32_t* cells = nullptr;
  uint64_t n = 0;
  uint64_t slides = 0;
  uint32_t now = kClockOrigin;
  uint32_t floor = 0;
  RsraDev dv{};
  GroupDev grp{};
  uint32_t hot_min = 0;
};

struct srlg_slea {
  srlg_slea_config cfg{};
  DeviceCtx* ctx = nullptr;
  uint32_t* cells = nullptr;
  uint64_t* lh_d = nullptr;
  uint64_t n = 0;
  uint64_t row_len = 0;
  uint64_t slides = 0;
  uint32_t now = kClockOrigin;
  uint32_t floor = 0;
  SleaDev dv{};
};

namespace {

// ReversibleHashGroup ctor constraints (src/hash.cpp:39-57) + Rsra ctor
// (src/rsra.cpp:9-23)
void check_rsra_config(const srlg_rsra_config& c, GroupDev* g, uint64_t* cells) {
  if (c.q == 0 || c.q > 31) raise(SRLG_ERR_CONFIG, "hash group: q must be in [1, 31]");
  if (c.r < 2) raise(SRLG_ERR_CONFIG, "hash group: need at least 2 rows");
  if (c.delta == 0 || c.delta >= c.q)
    raise(SRLG_ERR_CONFIG, "hash group: delta must satisfy 1 <= delta < q");
  if (c.eta == 0) raise(SRLG_ERR_CONFIG, "rsra: eta must be positive");
  if (c.r < 3) raise(SRLG_ERR_CONFIG, "rsra: need at least 3 rows to reconstruct hosts");
  if (c.r > 64) raise(SRLG_ERR_CONFIG, "rsra: at most 64 rows supported");
  if (static_cast<uint64_t>(c.r - 2) * c.delta + c.q < 32)
    raise(SRLG_ERR_CONFIG, "rsra: (r-2)*delta + q must reach the 32 address bits");
  const uint64_t total = (uint64_t{1} << c.q) * c.r * c.eta;
  if (total > (uint64_t{1} << 31))
    raise(SRLG_ERR_CONFIG, "rsra: parameter set needs more than 2^31 counters");
  *cells = total;
  GroupDev& G = *g;
  G = GroupDev{};
  G.h0 = mix64(c.seed_rhfg0);
  G.q = c.q;
  G.r = c.r;
  G.delta = c.delta;
  G.col_mask = (1u << c.q) - 1;
  G.overlap_mask = (1u << (c.q - c.delta)) - 1;
  uint64_t covered = 0;
  for (uint32_t i = 1; i < c.r; ++i) {
    const uint32_t lo = i * c.delta;
    if (lo >= 32) break;
    const uint32_t hi = std::min<uint32_t>(32, lo + c.q);
    covered |= ((uint64_t{1} << (hi - lo)) - 1) << lo;
  }
  G.uncovered = static_cast<uint32_t>(~covered & 0xFFFFFFFFull);
  G.n_free = 0;
  for (uint32_t b = 0; b < 32; ++b)
    if (G.uncovered & (1u << b)) G.free_bits[G.n_free++] = static_cast<uint8_t>(b);
}

// Slea ctor constraints (src/slea.cpp:11-27)
void check_slea_config(const srlg_slea_config& c, uint64_t* row_len, uint64_t* cells) {
  if (c.r == 0) raise(SRLG_ERR_CONFIG, "slea: need at least one row");
  if (c.r > 64) raise(SRLG_ERR_CONFIG, "slea: at most 64 rows supported");
  if (c.eta < 2) raise(SRLG_ERR_CONFIG, "slea: eta must be at least 2");
  if (c.delta == 0 || c.delta > c.eta)
    raise(SRLG_ERR_CONFIG, "slea: delta must satisfy 0 < delta <= eta");
  if (c.q > 30) raise(SRLG_ERR_CONFIG, "slea: q must be at most 30");
  *row_len = (uint64_t{1} << c.q) * c.delta + c.eta - c.delta;
  *cells = *row_len * c.r;
  if (*cells > (uint64_t{1} << 31))
    raise(SRLG_ERR_CONFIG, "slea: parameter set needs more than 2^31 counters");
}

bool is_pow2(uint32_t x) { return x && !(x & (x - 1)); }

void fill_rsra_dev(srlg_rsra* h) {
  const auto& c = h->cfg;
  RsraDev& d = h->dv;
  d.cells = h->cells;
  d.h0 = mix64(c.seed_rhfg0);
  d.h1 = mix64(c.seed_h1);
  d.h2 = mix64(c.seed_h2);
  d.q = c.q;
  d.r = c.r;
  d.delta = c.delta;
  d.eta = c.eta;
  d.col_mask = (1u << c.q) - 1;
  d.gate_never = c.tau > 32;
  d.gate_mask = c.tau >= 32 ? 0xFFFFFFFFu : ((1u << c.tau) - 1);
  d.eta_pow2 = is_pow2(c.eta);
  h->hot_min = hot_min_weight(c.eta);
}

void fill_slea_dev(srlg_slea* h) {
  const auto& c = h->cfg;
  SleaDev& d = h->dv;
  d.cells = h->cells;
  d.row_len = h->row_len;
  d.h3 = mix64(c.seed_h3);
  d.q = c.q;
  d.r = c.r;
  d.delta = c.delta;
  d.eta = c.eta;
  d.col_mask = (1u << c.q) - 1;
  d.eta_pow2 = is_pow2(c.eta);
  for (uint32_t i = 0; i < c.r; ++i) d.lh[i] = mix64(c.seeds_lh[i]);
  d.lh_dev = h->lh_d;
}

void advance_clock(uint32_t& now) {
  if (now == 0xFFFFFFFFu) raise(SRLG_ERR_RESOURCE, "stamp clock exhausted (2^32 slides)");
  ++now;
}

// --------------------------------------------------------- host -> device

// Runs fn(device_ptr, count) over n pairs, copying host input through the
// double-buffered staging area when needed. Caller holds ctx.mu.
template <class F>
void with_device_pairs(DeviceCtx& c, const srlg_pair* pairs, uint64_t n, int on_device, F&& fn) {
  if (n == 0) return;
  if (on_device) {
    fn(pairs, n);
    return;
  }
  c.ensure_staging();
  const bool pinned = is_pinned_host(pairs);
  for (uint64_t off = 0; off < n; off += kStagePairs) {
    const uint64_t cnt = std::min(kStagePairs, n - off);
    const int b = c.next_stage;
    c.next_stage = (b + 1) % kStageBufs;
    // the previous scan of this buffer must be done before it is overwritten
    cuda_ok(cudaStreamWaitEvent(c.cp, c.scan_done[b], 0), "wait");
    if (pinned) {
      cuda_ok(cudaMemcpyAsync(c.stage_d[b], pairs + off, cnt * sizeof(srlg_pair),
                              cudaMemcpyHostToDevice, c.cp),
              "H2D");
    } else {
      // pageable input: bounce through pinned memory; the pinned buffer's
      // previous H2D copy must have finished
      cuda_ok(cudaEventSynchronize(c.h2d_done[b]), "event sync");
      std::memcpy(c.stage_h[b], pairs + off, cnt * sizeof(srlg_pair));
      cuda_ok(cudaMemcpyAsync(c.stage_d[b], c.stage_h[b], cnt * sizeof(srlg_pair),
                              cudaMemcpyHostToDevice, c.cp),
              "H2D");
    }
    c.h2d_bytes += cnt * sizeof(srlg_pair);
    cuda_ok(cudaEventRecord(c.h2d_done[b], c.cp), "record");
    cuda_ok(cudaStreamWaitEvent(c.st, c.h2d_done[b], 0), "wait");
    fn(c.stage_d[b], cnt);
    cuda_ok(cudaEventRecord(c.scan_done[b], c.st), "record");
  }
}

void scan_pairs(DeviceCtx& c, srlg_rsra* rs, srlg_slea* le, const srlg_pair* dptr, uint64_t n,
                const AnetDev* anet = nullptr, unsigned long long* raw_records = nullptr) {
  static const RsraDev r0{};
  static const SleaDev l0{};
  const size_t p0 = c.prof.on ? c.prof.begin(c.st) : 0;
  cuda_ok(dev::scan(dptr, n, rs ? rs->dv : r0, rs ? rs->now : 0, le ? le->dv : l0,
                    le ? le->now : 0, dev::kStorePlain, c.st, anet, raw_records),
          "scan kernel");
  g_launches++;
  if (c.prof.on) c.prof.end(c.st, 0, p0, n);
}

// ----------------------------------------------------------- detection

struct PendingWindow {
  uint64_t window_end = 0;
  bool partial = false;
  int slot = 0;
  uint32_t r = 0, le_r = 0, eta_prime = 0;
  uint64_t row_len = 0, theta = 0;
  bool keep_below = false;
  uint64_t cand_cap = 0;
  uint32_t n_free = 0;
};

// Enqueue the device half of run_detection (src/window.cpp:36-78) into slot.
// Device parameters of the fused detection; `cands` is the device candidate
// buffer of capacity cand_cap. Sizes the shared scratch of the device.
DetectParams make_detect_params(DeviceCtx& c, srlg_rsra* rs, srlg_slea* le, uint32_t k,
                                uint64_t tuple_cap, Candidate* cands, uint64_t cand_cap) {
  const uint64_t work_cap = uint64_t{1} << 32;  // ReconstructOptions::work_cap
  c.hot_cols.ensure(static_cast<uint64_t>(rs->cfg.r) << rs->cfg.q);
  const uint64_t tcap = std::min<uint64_t>(tuple_cap, uint64_t{1} << 30);
  c.tuples_a.ensure((tcap + 1) * rs->cfg.r);
  c.tuples_b.ensure((tcap + 1) * rs->cfg.r);
  c.ensure_detect();
  // overlap tables: one region of 2^(q+1) entries per row 2..r-1 (a row has
  // at most 2^q hot columns, so the load factor stays <= 1/2)
  const uint64_t tstride = uint64_t{2} << rs->cfg.q;
  c.tables.ensure(tstride * (rs->cfg.r - 2));
  // reconstruction scratch: 3 * max(r, 8) words per thread of a launch
  const uint32_t dfs_rows = std::max<uint32_t>(rs->cfg.r, 8);
  c.dfs_scratch.ensure(static_cast<uint64_t>(c.detect_grid) * kDetectThreads * 3 * dfs_rows);
  DetectParams P{};
  P.rs = rs->dv;
  P.rs_lo = window_lo(rs->now, rs->floor, k);
  P.hot_min = rs->hot_min;
  P.le = le->dv;
  P.le_lo = window_lo(le->now, le->floor, k);
  P.lh = le->lh_d;
  P.g = rs->grp;
  P.hot_cols = c.hot_cols.p;
  P.tuples_a = c.tuples_a.p;
  P.tuples_b = c.tuples_b.p;
  P.table = c.tables.p;
  P.dfs_scratch = c.dfs_scratch.p;
  P.dfs_rows = dfs_rows;
  // inside bitmap of the SLEA (phase A writes it, phase C reads it), one bit
  // per cell in flat cell order
  P.le_bits_words = (le->row_len * le->cfg.r + 31) / 32 + 1;
  c.le_bits.ensure(P.le_bits_words);
  P.le_bits = c.le_bits.p;
  P.table_stride = tstride;
  P.table_bits = rs->cfg.q + 1;
  P.tuple_cap = tcap;
  P.work_cap = work_cap;
  P.cands = cands;
  P.cand_cap = cand_cap;
  c.left.ensure(cand_cap);
  P.left = c.left.p;
  P.scratch = c.scratch;
  P.bar = c.bar;
  P.host_prefix = std::min(kCandPrefix, cand_cap);
  P.serial = c.next_serial();
  return P;
}

// the buffer sets of pipelined engine batches (detect.cu k_engine: detection
// d uses set d % n); set 0 is the detection scratch make_detect_params set up
void add_sets(DeviceCtx& c, DetectParams& P, srlg_rsra* rs, uint32_t n, Candidate* const* cands) {
  const uint64_t hot = static_cast<uint64_t>(rs->cfg.r) << rs->cfg.q;
  const uint64_t tables = P.table_stride * (rs->cfg.r - 2);
  P.n_sets = n;
  P.sets[0] = DetSet{P.hot_cols, P.le_bits, cands[0], P.left, P.scratch, P.table};
  P.cands = cands[0];
  for (uint32_t i = 1; i < n; ++i) {
    DeviceCtx::SetBufs& b = c.extra[i - 1];
    b.hot_cols.ensure(hot);
    b.le_bits.ensure(P.le_bits_words);
    b.left.ensure(P.cand_cap);
    b.tables.ensure(tables);
    if (!b.scratch) {
      cuda_ok(cudaMalloc(&b.scratch, sizeof(DetectScratch)), "cudaMalloc (detect scratch)");
      cuda_ok(cudaMemsetAsync(b.scratch, 0, sizeof(DetectScratch), c.st), "memset");
    }
    P.sets[i] = DetSet{b.hot_cols.p, b.le_bits.p, cands[i], b.left.p, b.scratch, b.tables.p};
  }
}

void enqueue_detect(DeviceCtx& c, srlg_rsra* rs, srlg_slea* le, uint32_t k, uint64_t tuple_cap,
                    Slot& slot, uint64_t cand_cap) {
  slot.cand_d.ensure(cand_cap);
  slot.res_h.ensure(1);
  slot.cand_h.ensure(kCandPrefix);
  if (!slot.ev) cuda_ok(cudaEventCreateWithFlags(&slot.ev, cudaEventDisableTiming), "event");
  DetectParams P = make_detect_params(c, rs, le, k, tuple_cap, slot.cand_d.p, cand_cap);
  P.out = slot.res_h.dptr;
  P.host_cands = slot.cand_h.dptr;
  const size_t p0 = c.prof.on ? c.prof.begin(c.st) : 0;
  cuda_ok(dev::detect(P, c.detect_grid, c.st), "detect kernel");
  g_launches++;
  if (c.prof.on) c.prof.end(c.st, 1, p0, 1);
  c.d2h_bytes += sizeof(WinResult) + P.host_prefix * sizeof(Candidate);
  cuda_ok(cudaEventRecord(slot.ev, c.st), "record");
}

void put(std::vector<uint8_t>& out, const void* p, size_t n) {
  const size_t b = out.size();
  out.resize(b + n);
  std::memcpy(out.data() + b, p, n);
}

// Host half of run_detection: waits for the slot, then forms the report with
// the reference's double arithmetic and ordering (src/window.cpp:36-78).
// `pre` = the host prefix of the candidates; `tail` = device address of the
// rest (contiguous after the prefix).
void finalize_record(DeviceCtx& c, const WinResult& R, const Candidate* pre_cands,
                     const Candidate* tail, const PendingWindow& w, std::vector<uint8_t>& out) {
  srlg_report_header h{};
  h.window_end_slice = w.window_end;
  h.partial = w.partial;
  h.n_rows = w.r;
  // setting factors and their product, in row order (slea.cpp:85-95)
  double sfp = 1.0;
  for (uint32_t i = 0; i < w.le_r; ++i)
    sfp *= static_cast<double>(R.row_weights[i]) / static_cast<double>(w.row_len);
  h.sf_product = sfp;
  std::vector<Candidate> cands;
  if (!R.overflow && !R.empty) {
    if (R.stage_count[w.r] > 0 && w.n_free > 26)
      raise(SRLG_ERR_RESOURCE, "invert: parameter set leaves too many address bits unconstrained");
    if (R.cand_truncated || R.n_candidates > w.cand_cap)
      raise(SRLG_ERR_RESOURCE, "detection: candidate buffer exhausted");
    const uint64_t n = R.n_candidates;
    cands.resize(n);
    const uint64_t pre = std::min<uint64_t>(n, kCandPrefix);
    std::memcpy(cands.data(), pre_cands, pre * sizeof(Candidate));
    if (n > pre) {
      c.d2h_bytes += (n - pre) * sizeof(Candidate);
      cuda_ok(cudaMemcpy(cands.data() + pre, tail, (n - pre) * sizeof(Candidate),
                         cudaMemcpyDeviceToHost),
              "D2H candidates (tail)");
    }
  }
  h.overflow = R.overflow ? 1 : 0;
  h.candidate_count = cands.size();
  std::vector<srlg_entry> entries;
  if (sfp >= 1.0 - kSaturationEps) {
    h.slea_saturated = 1;
  } else {
    const double theta = static_cast<double>(w.theta);
    entries.reserve(cands.size());
    for (const Candidate& cd : cands) {
      const double cw = corrected_weight(static_cast<double>(cd.weight), sfp, w.eta_prime);
      double v;
      bool sat;
      le_estimate(cw, w.eta_prime, &v, &sat);
      if (w.keep_below || v >= theta) entries.push_back(srlg_entry{cd.aip, sat ? 1u : 0u, v});
    }
    std::sort(entries.begin(), entries.end(), [](const srlg_entry& a, const srlg_entry& b) {
      if (a.estimate != b.estimate) return a.estimate > b.estimate;
      return a.aip < b.aip;
    });
  }
  h.n_entries = static_cast<uint32_t>(entries.size());
  put(out, &h, sizeof h);
  put(out, R.hot_counts, 8 * w.r);
  if (!entries.empty()) put(out, entries.data(), entries.size() * sizeof(srlg_entry));
}

void finalize_detect(DeviceCtx& c, Slot& slot, const PendingWindow& w, std::vector<uint8_t>& out) {
  cuda_ok(cudaEventSynchronize(slot.ev), "detect sync");
  finalize_record(c, *slot.res_h.p, slot.cand_h.p, slot.cand_d.p + kCandPrefix, w, out);
}

PendingWindow make_pending(const srlg_rsra* rs, const srlg_slea* le, const srlg_window_config& cfg,
                           uint64_t end, bool partial, int slot, uint64_t cand_cap) {
  PendingWindow w;
  w.window_end = end;
  w.partial = partial;
  w.slot = slot;
  w.r = rs->cfg.r;
  w.le_r = le->cfg.r;
  w.eta_prime = le->cfg.eta;
  w.row_len = le->row_len;
  w.theta = cfg.theta;
  w.keep_below = cfg.keep_below_threshold != 0;
  w.cand_cap = cand_cap;
  w.n_free = rs->grp.n_free;
  return w;
}

uint64_t cand_cap_for(uint64_t tuple_cap) {
  return std::min<uint64_t>(tuple_cap, uint64_t{1} << 30) + 1024;
}

void check_window(const srlg_window_config& c) {
  if (c.slice_us == 0) raise(SRLG_ERR_CONFIG, "slice duration must be positive");
  if (c.k == 0 || c.k > 65534) raise(SRLG_ERR_CONFIG, "k must be in [1, 65534]");
  if (c.reinit_per_window && c.k != 1)
    raise(SRLG_ERR_CONFIG, "reinit-per-window is the strict discrete mode and needs k = 1");
  if (c.workers == 0) raise(SRLG_ERR_CONFIG, "workers must be at least 1");
}

// AnetSpec -> device form (CidrPrefix::contains, trace.hpp:38-42)
AnetDev to_anet(const srlg_anet& a) {
  if (a.n > SRLG_MAX_PREFIXES) raise(SRLG_ERR_INVALID_ARGUMENT, "anet: too many prefixes");
  AnetDev d{};
  d.n = a.n;
  for (uint32_t i = 0; i < a.n; ++i) {
    if (a.bits[i] > 32) raise(SRLG_ERR_INVALID_ARGUMENT, "anet: prefix length above 32");
    const uint32_t b = a.bits[i];
    const uint32_t mask = b == 0 ? 0u : b >= 32 ? 0xFFFFFFFFu : ~((uint32_t{1} << (32 - b)) - 1);
    d.mask[i] = mask;
    d.addr[i] = a.addr[i] & mask;
  }
  return d;
}

void check_same_device(const srlg_rsra* rs, const srlg_slea* le) {
  if (rs && le && rs->ctx != le->ctx)
    raise(SRLG_ERR_INVALID_ARGUMENT, "rsra and slea live on different devices");
}

}  // namespace

// ====================================================================== ABI

extern "C" {

const char* srlg_last_error(void) { return g_err.c_str(); }
int srlg_abi_version(void) { return SRLG_ABI_VERSION; }
uint64_t srlg_kernel_launches(void) { return g_launches.load(); }

int srlg_device_count(int* n) {
  return guarded([&] {
    if (cudaGetDeviceCount(n) != cudaSuccess) {
      cudaGetLastError();
      *n = 0;
    }
  });
}

// A further execution context on `device`: its own streams and detection
// scratch, and persistent kernels of at most `ctas` CTAs, so several engines
// (virtual ranks of a merge group) can run concurrently on one GPU.
int srlg_lane_create(int device, int ctas, int* lane_device) {
  *lane_device = -1;
  return guarded([&] {
    if (ctas < 0) raise(SRLG_ERR_INVALID_ARGUMENT, "lane CTA budget must be >= 0");
    DeviceCtx& phys = ctx_for(device);
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if (g_n_lanes >= 64) raise(SRLG_ERR_RESOURCE, "too many execution lanes");
    auto* c = new DeviceCtx();
    c->init(phys.device);
    c->cta_budget = ctas;
    g_lane[g_n_lanes] = c;
    *lane_device = kLaneBase + g_n_lanes++;
  });
}

// ------------------------------------------------------------ config

void srlg_window_config_default(srlg_window_config* c) {
  *c = srlg_window_config{};
  c->slice_us = 1'000'000;
  c->k = 300;
  c->theta = 1024;
  c->workers = 1;
  c->tuple_cap = uint64_t{1} << 22;
}

int srlg_window_config_validate(const srlg_window_config* c) {
  return guarded([&] { check_window(*c); });
}

// SketchParams::validate (src/config.cpp:20-42)
int srlg_params_validate(const srlg_params* p) {
  return guarded([&] {
    if (p->q < 1 || p->q > 30) raise(SRLG_ERR_CONFIG, "q must be in [1, 30]");
    if (p->q_prime < 1 || p->q_prime > 30) raise(SRLG_ERR_CONFIG, "q_prime must be in [1, 30]");
    if (p->r < 3 || p->r > 64) raise(SRLG_ERR_CONFIG, "r must be in [3, 64]");
    if (p->r_prime < 1 || p->r_prime > 64) raise(SRLG_ERR_CONFIG, "r_prime must be in [1, 64]");
    if (p->delta < 1 || p->delta >= p->q)
      raise(SRLG_ERR_CONFIG, "delta must satisfy 1 <= delta < q");
    if (static_cast<uint64_t>(p->r - 2) * p->delta + p->q < 32)
      raise(SRLG_ERR_CONFIG, "(r-2)*delta + q must be at least 32 to cover the address bits");
    if (p->eta < 1 || p->eta > 65535) raise(SRLG_ERR_CONFIG, "eta must be in [1, 65535]");
    if (p->eta_prime < 2 || p->eta_prime > (uint32_t{1} << 26))
      raise(SRLG_ERR_CONFIG, "eta_prime must be in [2, 2^26]");
    if (p->delta_prime < 1 || p->delta_prime > p->eta_prime)
      raise(SRLG_ERR_CONFIG, "delta_prime must satisfy 1 <= delta_prime <= eta_prime");
    if (p->theta < p->eta) raise(SRLG_ERR_CONFIG, "theta must be at least eta");
    if (sampling_threshold(p->theta, p->eta) > 32)
      raise(SRLG_ERR_CONFIG, "theta/eta ratio pushes the sampling threshold past 32 bits");
    const uint64_t rough = (uint64_t{1} << p->q) * p->r * p->eta;
    const uint64_t linear =
        ((uint64_t{1} << p->q_prime) * p->delta_prime + p->eta_prime - p->delta_prime) * p->r_prime;
    if (rough > (uint64_t{1} << 31) || linear > (uint64_t{1} << 31))
      raise(SRLG_ERR_CONFIG, "parameter set needs more than 2^31 counters; reduce q or q_prime");
  });
}

// rsra_config (src/config.cpp:48-60) + HashSeeds::derive (src/hash.cpp:18-27)
int srlg_params_rsra_config(const srlg_params* p, srlg_rsra_config* out) {
  int rc = srlg_params_validate(p);
  if (rc) return rc;
  *out = srlg_rsra_config{};
  out->q = p->q;
  out->r = p->r;
  out->delta = p->delta;
  out->eta = p->eta;
  out->tau = sampling_threshold(p->theta, p->eta);
  out->seed_h1 = hash64(1, p->seed);
  out->seed_h2 = hash64(2, p->seed);
  out->seed_rhfg0 = hash64(4, p->seed);
  return SRLG_OK;
}

// slea_config (src/config.cpp:62-72)
int srlg_params_slea_config(const srlg_params* p, srlg_slea_config* out) {
  int rc = srlg_params_validate(p);
  if (rc) return rc;
  *out = srlg_slea_config{};
  out->q = p->q_prime;
  out->r = p->r_prime;
  out->delta = p->delta_prime;
  out->eta = p->eta_prime;
  out->seed_h3 = hash64(3, p->seed);
  for (uint32_t i = 0; i < p->r_prime; ++i) out->seeds_lh[i] = hash64(100 + i, p->seed);
  return SRLG_OK;
}

uint64_t srlg_slea_row_length_for(const srlg_slea_config* c) {
  return (uint64_t{1} << c->q) * c->delta + c->eta - c->delta;
}

// -------------------------------------------------------------- Rsra

int srlg_rsra_create(const srlg_rsra_config* cfg, int device, srlg_rsra** out) {
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<srlg_rsra>();
    h->cfg = *cfg;
    check_rsra_config(*cfg, &h->grp, &h->n);
    h->ctx = &ctx_for(device);
    DeviceGuard g(h->ctx->device);
    cuda_ok(cudaMalloc(&h->cells, h->n * sizeof(uint32_t)), "cudaMalloc (rsra stamps)");
    cuda_ok(cudaMemsetAsync(h->cells, 0, h->n * sizeof(uint32_t), h->ctx->st), "memset");
    fill_rsra_dev(h.get());
    *out = h.release();
  });
}

int srlg_rsra_clone(const srlg_rsra* src, srlg_rsra** out) {
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<srlg_rsra>(*src);
    DeviceGuard g(src->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(src->ctx->mu);
    h->cells = nullptr;
    cuda_ok(cudaMalloc(&h->cells, h->n * sizeof(uint32_t)), "cudaMalloc (rsra stamps)");
    cuda_ok(cudaMemcpyAsync(h->cells, src->cells, h->n * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, src->ctx->st),
            "D2D clone");
    fill_rsra_dev(h.get());
    *out = h.release();
  });
}

void srlg_rsra_destroy(srlg_rsra* h) {
  if (!h) return;
  {
    DeviceGuard g(h->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(h->ctx->mu);
    cudaStreamSynchronize(h->ctx->st);
    cudaFree(h->cells);
  }
  delete h;
}

int srlg_rsra_config_get(const srlg_rsra* h, srlg_rsra_config* out) {
  *out = h->cfg;
  return SRLG_OK;
}
uint64_t srlg_rsra_num_cells(const srlg_rsra* h) { return h->n; }
uint64_t srlg_rsra_slides(const srlg_rsra* h) { return h->slides; }
int srlg_rsra_set_slides(srlg_rsra* h, uint64_t s) {
  h->slides = s;
  return SRLG_OK;
}

// Rsra::slide (src/rsra.cpp:35-38): ages every counter by one — here the
// clock moves, the stamps stay
int srlg_rsra_slide(srlg_rsra* h) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(h->ctx->mu);
    advance_clock(h->now);
    ++h->slides;
  });
}

// Rsra::reinitialize (src/rsra.cpp:40-43): every stamp so far becomes dead
int srlg_rsra_reinitialize(srlg_rsra* h) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(h->ctx->mu);
    h->floor = h->now;
    advance_clock(h->now);
    ++h->slides;
  });
}

int srlg_rsra_extract_hot(const srlg_rsra* hc, uint32_t k, uint32_t* cols, uint64_t cap,
                          uint64_t* row_counts) {
  auto* h = const_cast<srlg_rsra*>(hc);
  return guarded([&] {
    DeviceCtx& c = *h->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    const auto L = dev::counts_layout(&h->dv, nullptr);
    c.hot_bits.ensure((L.rs_sres + 31) / 32 + 1);
    c.partials.ensure(1);
    c.hot_cols.ensure(static_cast<uint64_t>(h->cfg.r) << h->cfg.q);
    c.sync_slot.res_d.ensure(1);
    c.sync_slot.res_h.ensure(1);
    const uint32_t lo = window_lo(h->now, h->floor, k);
    cuda_ok(dev::window_counts(&h->dv, lo, h->hot_min, nullptr, 0, L, c.hot_bits.p, c.partials.p,
                               c.st),
            "window counts kernel");
    cuda_ok(dev::hot_compact(c.hot_bits.p, h->cfg.q, h->cfg.r, c.partials.p, 0, 1, c.hot_cols.p,
                             c.sync_slot.res_d.p, uint64_t{1} << 32, c.st),
            "hot compaction kernel");
    g_launches += 2;
    cuda_ok(cudaMemcpyAsync(c.sync_slot.res_h.p, c.sync_slot.res_d.p, sizeof(WinResult),
                            cudaMemcpyDeviceToHost, c.st),
            "D2H");
    c.sync();
    uint64_t total = 0;
    for (uint32_t i = 0; i < h->cfg.r; ++i) {
      row_counts[i] = c.sync_slot.res_h.p->hot_counts[i];
      total += row_counts[i];
    }
    if (total > cap) raise(SRLG_ERR_RESOURCE, "hot list buffer too small");
    uint64_t off = 0;
    for (uint32_t i = 0; i < h->cfg.r; ++i) {
      if (row_counts[i])
        cuda_ok(cudaMemcpy(cols + off, c.hot_cols.p + (static_cast<uint64_t>(i) << h->cfg.q),
                           row_counts[i] * sizeof(uint32_t), cudaMemcpyDeviceToHost),
                "D2H hot lists");
      off += row_counts[i];
    }
  });
}

}  // extern "C"
namespace {

template <class H>
void export_cells_impl(const H* h, uint16_t* out, uint64_t n) {
  if (n != h->n) raise(SRLG_ERR_INVALID_ARGUMENT, "export: cell count mismatch");
  DeviceCtx& c = *h->ctx;
  DeviceGuard g(c.device);
  std::lock_guard<std::recursive_mutex> lk(c.mu);
  c.u16tmp.ensure(n);
  cuda_ok(dev::export_distances(h->cells, n, h->now, h->floor, c.u16tmp.p, c.st), "export kernel");
  g_launches++;
  cuda_ok(cudaMemcpyAsync(out, c.u16tmp.p, n * sizeof(uint16_t), cudaMemcpyDeviceToHost, c.st),
          "D2H cells");
  c.sync();
}

template <class H>
void import_cells_impl(H* h, const uint16_t* in, uint64_t n) {
  if (n != h->n) raise(SRLG_ERR_INVALID_ARGUMENT, "import: cell count mismatch");
  DeviceCtx& c = *h->ctx;
  DeviceGuard g(c.device);
  std::lock_guard<std::recursive_mutex> lk(c.mu);
  c.u16tmp.ensure(n);
  cuda_ok(cudaMemcpyAsync(c.u16tmp.p, in, n * sizeof(uint16_t), cudaMemcpyHostToDevice, c.st),
          "H2D cells");
  cuda_ok(dev::import_distances(c.u16tmp.p, n, h->now, h->cells, c.st), "import kernel");
  g_launches++;
  h->floor = 0;  // every cell was rewritten
  c.sync();
}

template <class H>
void export_stamps_impl(const H* h, uint32_t* out, uint64_t n, uint32_t* now, uint32_t* floor) {
  if (n != h->n) raise(SRLG_ERR_INVALID_ARGUMENT, "export: cell count mismatch");
  DeviceCtx& c = *h->ctx;
  DeviceGuard g(c.device);
  std::lock_guard<std::recursive_mutex> lk(c.mu);
  cuda_ok(cudaMemcpyAsync(out, h->cells, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, c.st), "D2H");
  c.sync();
  if (now) *now = h->now;
  if (floor) *floor = h->floor;
}

// merge_min of `other` into `self`; other may live on another device
template <class H>
void merge_impl(H* self, const H* other) {
  DeviceCtx& c = *self->ctx;
  DeviceGuard g(c.device);
  const uint32_t* src = other->cells;
  if (other->ctx != self->ctx) {
    // both contexts locked together (no lock-order deadlock between a->b and
    // b->a merges); the copy is ordered after other's pending work, and
    // other's later work after the copy
    std::scoped_lock lk(c.mu, other->ctx->mu);
    cudaEvent_t before = other->ctx->chunk_event(0), after = c.chunk_event(0);
    cuda_ok(cudaEventRecord(before, other->ctx->st), "record");
    cuda_ok(cudaStreamWaitEvent(c.st, before, 0), "wait");
    c.u32tmp.ensure(other->n);
    cuda_ok(cudaMemcpyPeerAsync(c.u32tmp.p, c.device, other->cells, other->ctx->device,
                                other->n * sizeof(uint32_t), c.st),
            "peer copy");
    cuda_ok(cudaEventRecord(after, c.st), "record");
    cuda_ok(cudaStreamWaitEvent(other->ctx->st, after, 0), "wait");
    src = c.u32tmp.p;
    cuda_ok(dev::merge_max(self->cells, src, self->n, self->now, self->floor, other->now,
                           other->floor, c.st),
            "merge kernel");
    g_launches++;
    self->floor = 0;
    return;
  }
  std::lock_guard<std::recursive_mutex> lk(c.mu);
  cuda_ok(dev::merge_max(self->cells, src, self->n, self->now, self->floor, other->now,
                         other->floor, c.st),
          "merge kernel");
  g_launches++;
  self->floor = 0;
}

}  // namespace
extern "C" {

int srlg_rsra_export_cells(const srlg_rsra* h, uint16_t* out, uint64_t n) {
  return guarded([&] { export_cells_impl(h, out, n); });
}
int srlg_rsra_import_cells(srlg_rsra* h, const uint16_t* in, uint64_t n) {
  return guarded([&] { import_cells_impl(h, in, n); });
}
int srlg_rsra_export_stamps(const srlg_rsra* h, uint32_t* out, uint64_t n, uint32_t* now,
                            uint32_t* floor) {
  return guarded([&] { export_stamps_impl(h, out, n, now, floor); });
}

}  // extern "C"
namespace {
std::string rsra_mismatch(const srlg_rsra* a, const srlg_rsra* b) {
  const auto &x = a->cfg, &y = b->cfg;
  if (x.q != y.q) return "q";
  if (x.r != y.r) return "r";
  if (x.delta != y.delta) return "delta";
  if (x.eta != y.eta) return "eta";
  if (x.tau != y.tau) return "tau";
  if (x.seed_h1 != y.seed_h1) return "seed_h1";
  if (x.seed_h2 != y.seed_h2) return "seed_h2";
  if (x.seed_rhfg0 != y.seed_rhfg0) return "seed_rhfg0";
  if (a->slides != b->slides) return "slice position";
  return {};
}
std::string slea_mismatch(const srlg_slea* a, const srlg_slea* b) {
  const auto &x = a->cfg, &y = b->cfg;
  if (x.q != y.q) return "q_prime";
  if (x.r != y.r) return "r_prime";
  if (x.delta != y.delta) return "delta_prime";
  if (x.eta != y.eta) return "eta_prime";
  if (x.seed_h3 != y.seed_h3) return "seed_h3";
  if (std::memcmp(x.seeds_lh, y.seeds_lh, sizeof(uint64_t) * x.r) != 0) return "seeds_lh";
  if (a->slides != b->slides) return "slice position";
  return {};
}
void copy_msg(const std::string& s, char* buf, size_t cap) {
  if (!buf || cap == 0) return;
  const size_t n = std::min(cap - 1, s.size());
  std::memcpy(buf, s.data(), n);
  buf[n] = 0;
}
}  // namespace
extern "C" {

// Rsra::compatibility_mismatch (src/rsra.cpp:64-75)
int srlg_rsra_compatibility_mismatch(const srlg_rsra* a, const srlg_rsra* b, char* buf,
                                     size_t cap) {
  copy_msg(rsra_mismatch(a, b), buf, cap);
  return SRLG_OK;
}

// Rsra::merge_min (src/rsra.cpp:77-81)
int srlg_rsra_merge_min(srlg_rsra* self, const srlg_rsra* other) {
  return guarded([&] {
    const std::string why = rsra_mismatch(self, other);
    if (!why.empty()) raise(SRLG_ERR_INCOMPATIBLE, "rsra merge: " + why + " differs");
    merge_impl(self, other);
  });
}

int srlg_rsra_forward(const srlg_rsra* h, uint32_t aip, uint32_t* cols) {
  const GroupDev& g = h->grp;
  cols[0] = static_cast<uint32_t>(seeded(g.h0, aip)) & g.col_mask;
  for (uint32_t i = 1; i < g.r; ++i) {
    const uint32_t sh = i * g.delta;
    const uint32_t shifted = sh >= 32 ? 0u : aip >> sh;
    cols[i] = (shifted ^ cols[0]) & g.col_mask;
  }
  return SRLG_OK;
}

void* srlg_rsra_device_ptr(const srlg_rsra* h) { return h->cells; }

// -------------------------------------------------------------- Slea

int srlg_slea_create(const srlg_slea_config* cfg, int device, srlg_slea** out) {
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<srlg_slea>();
    h->cfg = *cfg;
    check_slea_config(*cfg, &h->row_len, &h->n);
    h->ctx = &ctx_for(device);
    DeviceGuard g(h->ctx->device);
    cuda_ok(cudaMalloc(&h->cells, h->n * sizeof(uint32_t)), "cudaMalloc (slea stamps)");
    cuda_ok(cudaMalloc(&h->lh_d, SRLG_MAX_ROWS * sizeof(uint64_t)), "cudaMalloc");
    uint64_t lh[SRLG_MAX_ROWS] = {};
    for (uint32_t i = 0; i < cfg->r; ++i) lh[i] = mix64(cfg->seeds_lh[i]);
    cuda_ok(cudaMemcpy(h->lh_d, lh, sizeof lh, cudaMemcpyHostToDevice), "H2D");
    cuda_ok(cudaMemsetAsync(h->cells, 0, h->n * sizeof(uint32_t), h->ctx->st), "memset");
    fill_slea_dev(h.get());
    *out = h.release();
  });
}

int srlg_slea_clone(const srlg_slea* src, srlg_slea** out) {
  *out = nullptr;
  return guarded([&] {
    auto h = std::make_unique<srlg_slea>(*src);
    DeviceGuard g(src->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(src->ctx->mu);
    h->cells = nullptr;
    h->lh_d = nullptr;
    cuda_ok(cudaMalloc(&h->cells, h->n * sizeof(uint32_t)), "cudaMalloc (slea stamps)");
    cuda_ok(cudaMalloc(&h->lh_d, SRLG_MAX_ROWS * sizeof(uint64_t)), "cudaMalloc");
    cuda_ok(cudaMemcpyAsync(h->lh_d, src->lh_d, SRLG_MAX_ROWS * sizeof(uint64_t),
                            cudaMemcpyDeviceToDevice, src->ctx->st),
            "D2D");
    cuda_ok(cudaMemcpyAsync(h->cells, src->cells, h->n * sizeof(uint32_t),
                            cudaMemcpyDeviceToDevice, src->ctx->st),
            "D2D clone");
    fill_slea_dev(h.get());
    *out = h.release();
  });
}

void srlg_slea_destroy(srlg_slea* h) {
  if (!h) return;
  {
    DeviceGuard g(h->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(h->ctx->mu);
    cudaStreamSynchronize(h->ctx->st);
    cudaFree(h->cells);
    cudaFree(h->lh_d);
  }
  delete h;
}

int srlg_slea_config_get(const srlg_slea* h, srlg_slea_config* out) {
  *out = h->cfg;
  return SRLG_OK;
}
uint64_t srlg_slea_num_cells(const srlg_slea* h) { return h->n; }
uint64_t srlg_slea_row_length(const srlg_slea* h) { return h->row_len; }
uint64_t srlg_slea_slides(const srlg_slea* h) { return h->slides; }
int srlg_slea_set_slides(srlg_slea* h, uint64_t s) {
  h->slides = s;
  return SRLG_OK;
}

int srlg_slea_slide(srlg_slea* h) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(h->ctx->mu);
    advance_clock(h->now);
    ++h->slides;
  });
}

int srlg_slea_reinitialize(srlg_slea* h) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(h->ctx->mu);
    h->floor = h->now;
    advance_clock(h->now);
    ++h->slides;
  });
}

int srlg_slea_row_weights(const srlg_slea* hc, uint32_t k, uint64_t* out_r) {
  auto* h = const_cast<srlg_slea*>(hc);
  return guarded([&] {
    DeviceCtx& c = *h->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    const auto L = dev::counts_layout(nullptr, &h->dv);
    c.hot_bits.ensure(1);
    c.hot_cols.ensure(1);
    c.partials.ensure(static_cast<uint64_t>(L.le_blocks_per_row) * h->cfg.r + 1);
    c.sync_slot.res_d.ensure(1);
    c.sync_slot.res_h.ensure(1);
    const uint32_t lo = window_lo(h->now, h->floor, k);
    cuda_ok(dev::window_counts(nullptr, 0, 0, &h->dv, lo, L, c.hot_bits.p, c.partials.p, c.st),
            "window counts kernel");
    cuda_ok(dev::hot_compact(c.hot_bits.p, 0, 0, c.partials.p, h->cfg.r, L.le_blocks_per_row,
                             c.hot_cols.p, c.sync_slot.res_d.p, 0, c.st),
            "compaction kernel");
    g_launches += 2;
    cuda_ok(cudaMemcpyAsync(c.sync_slot.res_h.p, c.sync_slot.res_d.p, sizeof(WinResult),
                            cudaMemcpyDeviceToHost, c.st),
            "D2H");
    c.sync();
    for (uint32_t i = 0; i < h->cfg.r; ++i) out_r[i] = c.sync_slot.res_h.p->row_weights[i];
  });
}

// make_estimate_context (src/slea.cpp:85-95)
int srlg_slea_estimate_context(const srlg_slea* h, uint32_t k, double* factors,
                               double* sf_product) {
  uint64_t w[SRLG_MAX_ROWS];
  int rc = srlg_slea_row_weights(h, k, w);
  if (rc) return rc;
  double prod = 1.0;
  for (uint32_t i = 0; i < h->cfg.r; ++i) {
    const double f = static_cast<double>(w[i]) / static_cast<double>(h->row_len);
    if (factors) factors[i] = f;
    prod *= f;
  }
  *sf_product = prod;
  return SRLG_OK;
}

int srlg_slea_usle_weights(const srlg_slea* hc, uint32_t k, const uint32_t* aips, uint64_t n,
                           uint64_t* out) {
  auto* h = const_cast<srlg_slea*>(hc);
  return guarded([&] {
    if (n == 0) return;
    DeviceCtx& c = *h->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    c.sync_slot.cand_d.ensure(n);
    std::vector<Candidate> cands(n);
    for (uint64_t i = 0; i < n; ++i) cands[i] = Candidate{aips[i], 0};
    cuda_ok(cudaMemcpyAsync(c.sync_slot.cand_d.p, cands.data(), n * sizeof(Candidate),
                            cudaMemcpyHostToDevice, c.st),
            "H2D");
    const uint32_t lo = window_lo(h->now, h->floor, k);
    cuda_ok(dev::usle_weights(h->dv, lo, c.sync_slot.cand_d.p, nullptr, n, n, c.n_sms, c.st),
            "usle kernel");
    g_launches++;
    cuda_ok(cudaMemcpyAsync(cands.data(), c.sync_slot.cand_d.p, n * sizeof(Candidate),
                            cudaMemcpyDeviceToHost, c.st),
            "D2H");
    c.sync();
    for (uint64_t i = 0; i < n; ++i) out[i] = cands[i].weight;
  });
}

// Slea::estimate(aip, ctx) (src/slea.cpp:97-125)
int srlg_slea_estimate(const srlg_slea* h, uint32_t aip, uint32_t k, double sf_product,
                       srlg_estimate* out) {
  return guarded([&] {
    if (sf_product >= 1.0 - kSaturationEps)
      raise(SRLG_ERR_SATURATION, "slea estimate: array saturated, setting-factor product ~ 1");
    uint64_t w = 0;
    const int rc = srlg_slea_usle_weights(h, k, &aip, 1, &w);
    if (rc) raise(rc, g_err);
    *out = srlg_estimate{};
    out->usle_weight = w;
    out->sf_product = sf_product;
    out->corrected_weight = corrected_weight(static_cast<double>(w), sf_product, h->cfg.eta);
    bool sat = false;
    le_estimate(out->corrected_weight, h->cfg.eta, &out->value, &sat);
    out->saturated = sat;
  });
}

int srlg_slea_lh_column(const srlg_slea* h, uint32_t row, uint32_t aip, uint32_t* out) {
  if (row >= h->cfg.r) {
    g_err = "slea: row out of range";
    return SRLG_ERR_OUT_OF_RANGE;
  }
  *out = static_cast<uint32_t>(seeded(h->dv.lh[row], aip)) & h->dv.col_mask;
  return SRLG_OK;
}

int srlg_slea_export_cells(const srlg_slea* h, uint16_t* out, uint64_t n) {
  return guarded([&] { export_cells_impl(h, out, n); });
}
int srlg_slea_import_cells(srlg_slea* h, const uint16_t* in, uint64_t n) {
  return guarded([&] { import_cells_impl(h, in, n); });
}
int srlg_slea_export_stamps(const srlg_slea* h, uint32_t* out, uint64_t n, uint32_t* now,
                            uint32_t* floor) {
  return guarded([&] { export_stamps_impl(h, out, n, now, floor); });
}

int srlg_slea_compatibility_mismatch(const srlg_slea* a, const srlg_slea* b, char* buf,
                                     size_t cap) {
  copy_msg(slea_mismatch(a, b), buf, cap);
  return SRLG_OK;
}

int srlg_slea_merge_min(srlg_slea* self, const srlg_slea* other) {
  return guarded([&] {
    const std::string why = slea_mismatch(self, other);
    if (!why.empty()) raise(SRLG_ERR_INCOMPATIBLE, "slea merge: " + why + " differs");
    merge_impl(self, other);
  });
}

void* srlg_slea_device_ptr(const srlg_slea* h) { return h->cells; }

// ------------------------------------------------------- sketch streams
// The reference's "SRLG" v1 binary sketch stream (sketch_io.hpp:13-24,
// sketch_io.cpp:106-175), little-endian: magic | version u16 | type u8 |
// parameters u32 | seeds u64 | slides u64 | counters u16 row-major. The
// counters are the u16 distances of export_cells, so a GPU sketch can be
// merged with (or detected from) files written by CPU nodes and vice versa.
namespace {

constexpr char kMagic[4] = {'S', 'R', 'L', 'G'};
constexpr uint16_t kVersion = 1;
static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "SRLG streams are little-endian");

uint64_t rsra_header_bytes() { return 4 + 2 + 1 + 5 * 4 + 3 * 8 + 8; }
uint64_t slea_header_bytes(uint32_t r) { return 4 + 2 + 1 + 4 * 4 + (1 + uint64_t{r}) * 8 + 8; }

struct Writer {
  uint8_t* p;
  void raw(const void* v, size_t n) {
    std::memcpy(p, v, n);
    p += n;
  }
  void u8(uint8_t v) { raw(&v, 1); }
  void u16(uint16_t v) { raw(&v, 2); }
  void u32(uint32_t v) { raw(&v, 4); }
  void u64(uint64_t v) { raw(&v, 8); }
};

struct Reader {
  const uint8_t* p;
  const uint8_t* end;
  void raw(void* v, size_t n, const char* what = "sketch stream truncated") {
    if (static_cast<size_t>(end - p) < n) raise(SRLG_ERR_FORMAT, what);
    std::memcpy(v, p, n);
    p += n;
  }
  uint16_t u16() { uint16_t v; raw(&v, 2); return v; }
  uint32_t u32() { uint32_t v; raw(&v, 4); return v; }
  uint64_t u64() { uint64_t v; raw(&v, 8); return v; }
};

}  // namespace

extern "C" {

// serialized_size (sketch_io.cpp:136-142)
uint64_t srlg_rsra_serialized_size(const srlg_rsra* h) { return rsra_header_bytes() + 2 * h->n; }
uint64_t srlg_slea_serialized_size(const srlg_slea* h) {
  return slea_header_bytes(h->cfg.r) + 2 * h->n;
}

// serialize_sketch(const Rsra&) (sketch_io.cpp:106-119)
int srlg_rsra_serialize(const srlg_rsra* h, uint8_t* out, uint64_t cap, uint64_t* written) {
  return guarded([&] {
    const uint64_t need = srlg_rsra_serialized_size(h);
    if (cap < need) raise(SRLG_ERR_INVALID_ARGUMENT, "serialize: output buffer too small");
    Writer w{out};
    w.raw(kMagic, 4);
    w.u16(kVersion);
    w.u8(1);
    const srlg_rsra_config& c = h->cfg;
    w.u32(c.q);
    w.u32(c.r);
    w.u32(c.delta);
    w.u32(c.eta);
    w.u32(c.tau);
    w.u64(c.seed_h1);
    w.u64(c.seed_h2);
    w.u64(c.seed_rhfg0);
    w.u64(h->slides);
    export_cells_impl(h, reinterpret_cast<uint16_t*>(w.p), h->n);  // device -> stream body
    *written = need;
  });
}

// serialize_sketch(const Slea&) (sketch_io.cpp:121-134)
int srlg_slea_serialize(const srlg_slea* h, uint8_t* out, uint64_t cap, uint64_t* written) {
  return guarded([&] {
    const uint64_t need = srlg_slea_serialized_size(h);
    if (cap < need) raise(SRLG_ERR_INVALID_ARGUMENT, "serialize: output buffer too small");
    Writer w{out};
    w.raw(kMagic, 4);
    w.u16(kVersion);
    w.u8(2);
    const srlg_slea_config& c = h->cfg;
    w.u32(c.q);
    w.u32(c.r);
    w.u32(c.delta);
    w.u32(c.eta);
    w.u64(c.seed_h3);
    for (uint32_t i = 0; i < c.r; ++i) w.u64(c.seeds_lh[i]);
    w.u64(h->slides);
    export_cells_impl(h, reinterpret_cast<uint16_t*>(w.p), h->n);
    *written = need;
  });
}

// deserialize_sketch (sketch_io.cpp:144-175): one stream -> a new handle on
// `device` (*type 1 = rsra, 2 = slea; the other out-pointer stays null).
// Bad magic / version / type tag and truncation raise SRLG_ERR_FORMAT with
// the reference's messages; a parameter block the constructors reject raises
// SRLG_ERR_CONFIG, as Rsra(cfg) / Slea(cfg) would.
int srlg_deserialize_sketch(const uint8_t* in, uint64_t size, int device, int* type,
                            srlg_rsra** rsra, srlg_slea** slea, uint64_t* consumed) {
  *type = 0;
  *rsra = nullptr;
  *slea = nullptr;
  return guarded([&] {
    Reader rd{in, in + size};
    char magic[4];
    rd.raw(magic, 4);
    if (std::memcmp(magic, kMagic, 4) != 0) raise(SRLG_ERR_FORMAT, "bad sketch magic");
    const uint16_t version = rd.u16();
    if (version != kVersion)
      raise(SRLG_ERR_FORMAT, "unsupported sketch format version " + std::to_string(version));
    uint8_t t = 0;
    rd.raw(&t, 1);
    if (t != 1 && t != 2) raise(SRLG_ERR_FORMAT, "unknown sketch type tag");
    if (t == 1) {
      srlg_rsra_config c{};
      c.q = rd.u32();
      c.r = rd.u32();
      c.delta = rd.u32();
      c.eta = rd.u32();
      c.tau = rd.u32();
      c.seed_h1 = rd.u64();
      c.seed_h2 = rd.u64();
      c.seed_rhfg0 = rd.u64();
      const uint64_t slides = rd.u64();
      srlg_rsra* h = nullptr;
      const int st = srlg_rsra_create(&c, device, &h);
      if (st != SRLG_OK) raise(st, g_err);
      std::unique_ptr<srlg_rsra, void (*)(srlg_rsra*)> guard(h, srlg_rsra_destroy);
      if (static_cast<uint64_t>(rd.end - rd.p) / 2 < h->n)
        raise(SRLG_ERR_FORMAT, "sketch stream truncated in counter block");
      std::vector<uint16_t> cells(h->n);
      rd.raw(cells.data(), 2 * h->n, "sketch stream truncated in counter block");
      import_cells_impl(h, cells.data(), h->n);
      h->slides = slides;
      *rsra = guard.release();
    } else {
      srlg_slea_config c{};
      c.q = rd.u32();
      c.r = rd.u32();
      c.delta = rd.u32();
      c.eta = rd.u32();
      if (c.r > 64) raise(SRLG_ERR_FORMAT, "sketch stream declares too many rows");
      c.seed_h3 = rd.u64();
      for (uint32_t i = 0; i < c.r; ++i) c.seeds_lh[i] = rd.u64();
      const uint64_t slides = rd.u64();
      srlg_slea* h = nullptr;
      const int st = srlg_slea_create(&c, device, &h);
      if (st != SRLG_OK) raise(st, g_err);
      std::unique_ptr<srlg_slea, void (*)(srlg_slea*)> guard(h, srlg_slea_destroy);
      if (static_cast<uint64_t>(rd.end - rd.p) / 2 < h->n)
        raise(SRLG_ERR_FORMAT, "sketch stream truncated in counter block");
      std::vector<uint16_t> cells(h->n);
      rd.raw(cells.data(), 2 * h->n, "sketch stream truncated in counter block");
      import_cells_impl(h, cells.data(), h->n);
      h->slides = slides;
      *slea = guard.release();
    }
    *type = t;
    *consumed = static_cast<uint64_t>(rd.p - in);
  });
}

}  // extern "C"

// ---------------------------------------------------------------- scan

int srlg_update_pairs(srlg_rsra* rs, srlg_slea* le, const srlg_pair* pairs, uint64_t n,
                      int pairs_on_device, void* stream) {
  return guarded([&] {
    if (!rs && !le) return;
    check_same_device(rs, le);
    DeviceCtx& c = rs ? *rs->ctx : *le->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    cudaEvent_t ev = nullptr;
    if (stream && pairs_on_device) {
      // order after the caller's producer stream
      cuda_ok(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
      cuda_ok(cudaEventRecord(ev, static_cast<cudaStream_t>(stream)), "record");
      cuda_ok(cudaStreamWaitEvent(c.st, ev, 0), "wait");
    }
    with_device_pairs(c, pairs, n, pairs_on_device,
                      [&](const srlg_pair* d, uint64_t cnt) { scan_pairs(c, rs, le, d, cnt); });
    if (ev) cudaEventDestroy(ev);
    if (!pairs_on_device) {
      // host buffers may be reused by the caller once we return
      cuda_ok(cudaStreamSynchronize(c.cp), "copy sync");
    }
  });
}

// classify (trace.cpp:111-116) + Rsra::update + Slea::update over raw packets
int srlg_update_raw(srlg_rsra* rs, srlg_slea* le, const srlg_pair* packets, uint64_t n,
                    int packets_on_device, const srlg_anet* anet, uint64_t* records) {
  return guarded([&] {
    if (!anet || anet->n == 0) raise(SRLG_ERR_INVALID_ARGUMENT, "update_raw: empty monitored network");
    const AnetDev a = to_anet(*anet);
    if (!rs && !le) {
      if (records) *records = 0;
      return;
    }
    check_same_device(rs, le);
    DeviceCtx& c = rs ? *rs->ctx : *le->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    c.u64tmp.ensure(1);
    cuda_ok(cudaMemsetAsync(c.u64tmp.p, 0, sizeof(unsigned long long), c.st), "memset");
    with_device_pairs(c, packets, n, packets_on_device, [&](const srlg_pair* d, uint64_t cnt) {
      scan_pairs(c, rs, le, d, cnt, &a, c.u64tmp.p);
    });
    unsigned long long got = 0;
    cuda_ok(cudaMemcpyAsync(&got, c.u64tmp.p, sizeof got, cudaMemcpyDeviceToHost, c.st), "D2H");
    c.sync();
    if (!packets_on_device) cuda_ok(cudaStreamSynchronize(c.cp), "copy sync");
    if (records) *records = got;
  });
}

// ------------------------------------------------------- reconstruction

}  // extern "C"

namespace {

// ReversibleHashGroup ctor checks (src/hash.cpp:39-57) -> device geometry
GroupDev make_group(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed) {
  if (q == 0 || q > 31) raise(SRLG_ERR_CONFIG, "hash group: q must be in [1, 31]");
  if (r < 2) raise(SRLG_ERR_CONFIG, "hash group: need at least 2 rows");
  if (delta == 0 || delta >= q) raise(SRLG_ERR_CONFIG, "hash group: delta must satisfy 1 <= delta < q");
  if (r > SRLG_MAX_ROWS) raise(SRLG_ERR_CONFIG, "hash group: at most 64 rows supported");
  GroupDev G{};
  G.h0 = mix64(seed);
  G.q = q;
  G.r = r;
  G.delta = delta;
  G.col_mask = (1u << q) - 1;
  G.overlap_mask = (1u << (q - delta)) - 1;
  uint64_t covered = 0;
  for (uint32_t i = 1; i < r; ++i) {
    const uint32_t lo = i * delta;
    if (lo >= 32) break;
    const uint32_t hi = std::min<uint32_t>(32, lo + q);
    covered |= ((uint64_t{1} << (hi - lo)) - 1) << lo;
  }
  G.uncovered = static_cast<uint32_t>(~covered & 0xFFFFFFFFull);
  for (uint32_t b = 0; b < 32; ++b)
    if (G.uncovered & (1u << b)) G.free_bits[G.n_free++] = static_cast<uint8_t>(b);
  return G;
}

void reconstruct_impl(DeviceCtx& c, const GroupDev& grp, const uint32_t* hot_cols,
                      const uint64_t* row_counts, uint64_t tuple_cap, uint64_t work_cap,
                      uint32_t* addresses, uint64_t cap, uint64_t* n_addresses, int* overflow,
                      uint64_t* tuples_checked, uint64_t* tuples_kept) {
  {
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    if (grp.r < 3) raise(SRLG_ERR_INVALID_ARGUMENT, "reconstruct: need at least 3 rows");
    const uint32_t r = grp.r;
    const uint64_t cols = uint64_t{1} << grp.q;
    WinResult R{};
    bool empty = false;
    uint64_t total = 0;
    for (uint32_t i = 0; i < r; ++i) {
      if (row_counts[i] > cols) raise(SRLG_ERR_INVALID_ARGUMENT, "reconstruct: hot list longer than a row");
      R.hot_counts[i] = row_counts[i];
      empty |= row_counts[i] == 0;
      total += row_counts[i];
    }
    for (uint64_t i = 0; i < total; ++i)
      if (hot_cols[i] >= cols) raise(SRLG_ERR_INVALID_ARGUMENT, "reconstruct: column out of range");
    R.empty = empty;
    R.seed_work = empty ? 0 : row_counts[0] * row_counts[1] * row_counts[2];
    R.overflow = !empty && R.seed_work > work_cap;
    c.hot_cols.ensure(static_cast<uint64_t>(r) << grp.q);
    const uint64_t tcap = std::min<uint64_t>(tuple_cap, uint64_t{1} << 30);
    c.tuples_a.ensure((tcap + 1) * r);
    c.tuples_b.ensure((tcap + 1) * r);
    const uint64_t ccap = cand_cap_for(tuple_cap);
    c.sync_slot.res_d.ensure(1);
    c.sync_slot.cand_d.ensure(ccap);
    uint64_t off = 0;
    for (uint32_t i = 0; i < r; ++i) {
      if (row_counts[i])
        cuda_ok(cudaMemcpyAsync(c.hot_cols.p + i * cols, hot_cols + off,
                                row_counts[i] * sizeof(uint32_t), cudaMemcpyHostToDevice, c.st),
                "H2D hot lists");
      off += row_counts[i];
    }
    cuda_ok(cudaMemcpyAsync(c.sync_slot.res_d.p, &R, sizeof R, cudaMemcpyHostToDevice, c.st), "H2D");
    cuda_ok(dev::reconstruct(grp, c.hot_cols.p, c.sync_slot.res_d.p, c.tuples_a.p, c.tuples_b.p,
                             tcap, work_cap, c.sync_slot.cand_d.p, ccap, c.n_sms, c.st),
            "reconstruct kernels");
    g_launches += r - 1;
    cuda_ok(cudaMemcpyAsync(&R, c.sync_slot.res_d.p, sizeof R, cudaMemcpyDeviceToHost, c.st), "D2H");
    c.sync();
    *overflow = R.overflow ? 1 : 0;
    *tuples_checked = 0;
    *tuples_kept = 0;
    *n_addresses = 0;
    if (R.overflow || R.empty) return;
    if (R.stage_count[r] > 0 && grp.n_free > 26)
      raise(SRLG_ERR_RESOURCE, "invert: parameter set leaves too many address bits unconstrained");
    if (R.cand_truncated) raise(SRLG_ERR_RESOURCE, "reconstruct: candidate buffer exhausted");
    uint64_t checked = R.seed_work;
    for (uint32_t j = 3; j < r; ++j) checked += R.stage_count[j] * R.hot_counts[j];
    *tuples_checked = checked;
    *tuples_kept = R.stage_count[r];
    std::vector<Candidate> cands(R.n_candidates);
    if (!cands.empty())
      cuda_ok(cudaMemcpy(cands.data(), c.sync_slot.cand_d.p, cands.size() * sizeof(Candidate),
                         cudaMemcpyDeviceToHost),
              "D2H");
    std::vector<uint32_t> a(cands.size());
    for (size_t i = 0; i < cands.size(); ++i) a[i] = cands[i].aip;
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
    *n_addresses = a.size();
    for (size_t i = 0; i < a.size() && i < cap; ++i) addresses[i] = a[i];
  }
}

}  // namespace

extern "C" {

int srlg_reconstruct(const srlg_rsra* h, const uint32_t* hot_cols, const uint64_t* row_counts,
                     uint64_t tuple_cap, uint64_t work_cap, uint32_t* addresses, uint64_t cap,
                     uint64_t* n_addresses, int* overflow, uint64_t* tuples_checked,
                     uint64_t* tuples_kept) {
  return guarded([&] {
    reconstruct_impl(*h->ctx, h->grp, hot_cols, row_counts, tuple_cap, work_cap, addresses, cap,
                     n_addresses, overflow, tuples_checked, tuples_kept);
  });
}

int srlg_reconstruct_group(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, int device,
                           const uint32_t* hot_cols, const uint64_t* row_counts,
                           uint64_t tuple_cap, uint64_t work_cap, uint32_t* addresses,
                           uint64_t cap, uint64_t* n_addresses, int* overflow,
                           uint64_t* tuples_checked, uint64_t* tuples_kept) {
  return guarded([&] {
    const GroupDev grp = make_group(q, r, delta, seed);
    reconstruct_impl(ctx_for(device), grp, hot_cols, row_counts, tuple_cap, work_cap, addresses,
                     cap, n_addresses, overflow, tuples_checked, tuples_kept);
  });
}

// ------------------------------------------------------------ detection

int srlg_detect(const srlg_rsra* rsc, const srlg_slea* lec, const srlg_window_config* cfg,
                uint64_t window_end_slice, int partial, uint8_t* blob, uint64_t cap,
                uint64_t* blob_bytes) {
  auto* rs = const_cast<srlg_rsra*>(rsc);
  auto* le = const_cast<srlg_slea*>(lec);
  return guarded([&] {
    check_same_device(rs, le);
    DeviceCtx& c = *rs->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    const uint64_t ccap = cand_cap_for(cfg->tuple_cap);
    enqueue_detect(c, rs, le, cfg->k, cfg->tuple_cap, c.sync_slot, ccap);
    std::vector<uint8_t> out;
    finalize_detect(c, c.sync_slot,
                    make_pending(rs, le, *cfg, window_end_slice, partial != 0, 0, ccap), out);
    *blob_bytes = out.size();
    if (blob && out.size() <= cap) std::memcpy(blob, out.data(), out.size());
  });
}

}  // extern "C"

// ================================================================ engine

namespace {
constexpr int kSlots = 4;
// CTAs of the engine's reconstruction group (detect.cu k_engine); the rest
// scan and stream the state. With three buffer sets a detection may take up
// to ~3 slice periods; on C2, 16 CTAs is the fastest (+2 % over 20 at the
// same latency); at 12 the reconstruction falls behind and the stream group
// waits for buffer sets.
}

struct srlg_engine {
  srlg_window_config cfg{};
  srlg_rsra* rs = nullptr;
  srlg_slea* le = nullptr;
  DeviceCtx* ctx = nullptr;
  // SliceClock (include/slidecard/window.hpp:34-52)
  bool has_t0 = false, has_max = false;
  uint64_t t0 = 0, max_ts = 0, clamped = 0;
  uint64_t current = 0, records = 0;
  bool active = false;
  std::vector<srlg_pair> pending;  // host records of the open slice
  // detection pipeline
  Slot slots[kSlots];
  std::deque<PendingWindow> inflight;
  int next_slot = 0;
  uint64_t cand_cap = 0;
  std::vector<uint8_t> reports;
  uint64_t n_reports = 0;
  uint64_t launches_at_take = 0;
  // distributed mode (run_distributed src/distributed.cpp:35-117):
  // one edge-router stream per GPU. The scan only marks touched cells in a u8
  // map; every completed slice the maps are max-reduced (NCCL) onto the root,
  // which stamps them into the global sketches and runs the detection.
  bool merge = false;
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1, root = 0;
  uint8_t* dirty = nullptr;
  uint64_t merges = 0, merge_bytes = 0;
  // in-engine merge over peer memory (srlg_engine_merge_create / _join /
  // _attach; detect.cu rank_scan / root_apply): pre-sliced input only, every
  // rank emits one scan op per slice, numbered by `seq` on every rank alike
  int inbox_role = 0;          // 0 none, 1 root, 2 sending rank
  void* inbox = nullptr;       // root: its allocation; rank: the mapped root inbox
  bool inbox_ipc = false;      // opened with cudaIpcOpenMemHandle
  dev::MergeDev md{};
  uint32_t seq = 0;            // slices published since the group was set up (never reset)
  uint64_t inbox_max_pairs = 0;

  bool is_root() const { return (!merge || rank == root) && inbox_role != 2; }

  // ---- persistent batches: a run of pre-sliced input becomes a list of
  // scan / detect ops executed by one cooperative kernel (detect.cu
  // k_engine); the host only simulates the clock and finalises windows
  // (from a mapped ring) while the kernel runs.
  bool persistent = true;
  // raw-packet ingest (srlg_engine_set_anet): classify on the device
  AnetDev anet{};
  DevBuf<unsigned long long> raw_records;  // records produced by raw packets (device)
  uint64_t raw_packets = 0;  // packets fed in raw mode (counted in `records` by the slice paths)
  struct Batch {
    HostBuf<WinResult> out;
    HostBuf<Candidate> cands;
    HostBuf<uint32_t> ready;
    HostBuf<EngineOp> ops_h;
    DevBuf<EngineOp> ops_d;
    // rings of the candidates past each window's host prefix, one per
    // reconstruction group (group g: windows w = g mod groups)
    DevBuf<Candidate> arena;
    uint64_t arena_cap = 0;  // entries per group
    uint32_t groups = 1;
    HostBuf<unsigned long long> arena_rel;  // per group: ring offset the host copied tails out to
    DevBuf<unsigned long long> arena_heads;  // per group: the kernel's allocation offset
    DevBuf<unsigned long long> op_t;  // diagnostics: per-op {start, ~end} (atomicMin)
    std::vector<unsigned long long> op_t_h;
    DevBuf<unsigned long long> cta_t;
    std::vector<uint32_t> op_kind;
    std::vector<PendingWindow> wins;
    cudaEvent_t done = nullptr;
    bool live = false;
    size_t fin = 0;  // windows already finalised
  };
  // incremental phase A (detect.cu phase_a_inc, srlg_engine_set_incremental):
  // 0 off, 1 RSRA always and the SLEA when its sweep would leave L2, 2 both,
  // 3 RSRA only
  int incremental = 1;
  // SLEA stamps above this are tracked incrementally in mode 1 (its sweep
  // would stream from HBM; below it the sweep is an L2 read and tracking —
  // one more L2 operation per SLEA update — costs more than it saves)
  static constexpr uint64_t kLeIncBytes = uint64_t{64} << 20;
  static constexpr uint64_t kArenaCands = uint64_t{1} << 22;
  uint64_t arena_entries = 0;  // ring capacity override (srlg_engine_set_arena; 0 = default)
  Batch batches[2];
  int next_batch = 0;
  DevBuf<Candidate> bcands[kMaxSets];  // per buffer set
  // reconstruction pipeline of persistent batches (srlg_engine_set_recon):
  // recon_ctas CTAs in recon_groups groups; group g takes detections
  // d = g mod groups, and groups + 1 buffer sets are in flight
  // tools/ab_recon.py on C2: 16x2 8.37 / 24x4 7.43 ms per step; 24x4 7.03 ms at
  // 63 us latency vs 24x3 7.01 ms at 46 us (C5 alike, C4 24x2 194 us vs 24x4 241)
  int recon_ctas = 24, recon_groups = 3;
  std::vector<EngineOp> ops;
  std::vector<PendingWindow> bwins;
  double det_ns_sum = 0;  // device time of the finalised windows' detections
  uint64_t det_n = 0;
  double det_diag[16] = {};  // diagnostics (trace_ops): see srlg_engine_detect_diag
  double det_phase_ns[6] = {};  // A1, barrier, B||A2, barrier, C, epilogue (CTA 0's view)
  bool trace_ops = false;            // diagnostics: record per-op device spans
  std::vector<uint64_t> op_trace;    // {kind, start ns, end ns} per op of finished batches
  std::vector<uint64_t> cta_trace;   // last traced batch: per op, per CTA {start, end}
  uint64_t cta_trace_ops = 0;

  // Slice `sl` of a pre-sliced call: it may not precede the open slice, and
  // may continue it (records already delivered later in the same slice do
  // not make its start time a regression); a non-empty slice moves the
  // clock's maximum timestamp like SliceClock::place would (window.cpp:24-34)
  uint64_t slice_for_call(uint64_t sl, bool has_records) {
    if (sl < current) raise(SRLG_ERR_ORDERING, "slice precedes the engine's current slice");
    if (has_records) {
      const uint64_t ts = t0 + sl * cfg.slice_us;
      if (!has_max || ts > max_ts) {
        max_ts = ts;
        has_max = true;
      }
    }
    return sl;
  }

  // one scan op per slice j in [s, s_end) of a pre-sliced run, pair
  // offsets relative to `base` (detect ops are inserted as slices complete).
  // In-engine merge mode every slice gets an op, empty ones included, so
  // all ranks publish / apply the same numbered slices.
  void add_slice_ops(const uint64_t* off, uint64_t s, uint64_t s_end, uint64_t first_slice,
                     uint64_t base, bool chunked) {
    for (uint64_t j = s; j < s_end; ++j) {
      const uint64_t m = off[j + 1] - off[j];
      if (m == 0 && !inbox_role) continue;
      const uint64_t sl = slice_for_call(first_slice + j, m != 0);
      active = true;
      while (current < sl) batch_complete_slice();
      EngineOp op{};
      op.kind = 0;
      op.begin = off[j] - base;
      op.end = op.begin + m;
      op.rs_now = rs->now;
      op.le_now = le->now;
      op.chunk = !chunked ? 0u : m ? static_cast<uint32_t>((op.end - 1) / kChunkPairs) : ~0u;
      if (inbox_role) {
        if (m > inbox_max_pairs)
          raise(SRLG_ERR_RESOURCE, "slice exceeds the merge inbox capacity (max_pairs_per_slice)");
        op.seq = seq++;
        ++merges;
      }
      ops.push_back(op);
      records += m;
    }
  }

  // complete_slice as ops: a detect op (when due), then the clocks move
  void batch_complete_slice() {
    if (current + 1 >= cfg.k && is_root()) {
      EngineOp op{};
      op.kind = 1;
      op.rs_lo = window_lo(rs->now, rs->floor, cfg.k);
      op.le_lo = window_lo(le->now, le->floor, cfg.k);
      op.window = static_cast<uint32_t>(bwins.size());
      op.serial = ctx->next_serial();
      ops.push_back(op);
      bwins.push_back(make_pending(rs, le, cfg, current, false, -1, cand_cap));
    }
    advance_clocks();
    ++current;
  }

  void advance_clocks() {
    if (cfg.reinit_per_window) {
      rs->floor = rs->now;
      le->floor = le->now;
    }
    advance_clock(rs->now);
    ++rs->slides;
    advance_clock(le->now);
    ++le->slides;
  }

  void wait_ready(Batch& B, size_t w) {
    volatile uint32_t* f = B.ready.p + w;
    while (!*f) {
      const cudaError_t q = cudaEventQuery(B.done);
      if (q == cudaSuccess) {
        if (*f) break;
        raise(SRLG_ERR_CUDA, "engine batch finished without its window record");
      }
      if (q != cudaErrorNotReady) cuda_ok(q, "engine batch");
      std::this_thread::yield();
    }
    std::atomic_thread_fence(std::memory_order_acquire);
  }

  // finalise the windows whose records have arrived, in order, without
  // waiting (the host works through them while the input is still copying)
  void finalize_ready(Batch& B) {
    while (B.fin < B.wins.size() &&
           *reinterpret_cast<volatile uint32_t*>(B.ready.p + B.fin) != 0) {
      std::atomic_thread_fence(std::memory_order_acquire);
      finalize_window(B, B.fin++);
    }
  }

  void finalize_window(Batch& B, size_t w) {
    const WinResult& R = B.out.p[w];
    const uint32_t g = static_cast<uint32_t>(w % B.groups);
    const Candidate* tail = R.tail_offset != ~0ull
                                ? B.arena.p + g * B.arena_cap + R.tail_offset % B.arena_cap
                                : nullptr;
    try {
      finalize_record(*ctx, R, B.cands.p + w * kCandPrefix, tail, B.wins[w], reports);
    } catch (...) {
      // the batch cannot report this window: free the whole ring (later
      // windows must not wait for it), let the kernel run out, drop the
      // batch's remaining windows and surface the error once
      for (uint32_t i = 0; i < B.groups; ++i) release_arena(B, i, ~0ull >> 1);
      cudaEventSynchronize(B.done);
      B.wins.clear();
      B.op_kind.clear();
      B.fin = 0;
      B.live = false;
      throw;
    }
    if (tail) {
      const uint64_t kept = std::min<uint64_t>(R.n_candidates, B.wins[w].cand_cap);
      release_arena(B, g, R.tail_offset + (kept - kCandPrefix));
    }
    ++n_reports;
    det_ns_sum += static_cast<double>(R.t_end - R.t_begin);
    for (int i = 0; i < 5; ++i) det_phase_ns[i] += static_cast<double>(R.t_phase[i + 1] - R.t_phase[i]);
    det_phase_ns[5] += static_cast<double>(R.t_end - R.t_phase[5]);
    if (R.t_diag[0] || R.t_diag[1]) {
      det_diag[0] += R.t_diag[0] ? static_cast<double>(R.t_diag[0] - R.t_phase[2]) : 0.0;
      det_diag[1] += R.t_diag[1] ? static_cast<double>(R.t_diag[1] - R.t_phase[2]) : 0.0;
      det_diag[2] += static_cast<double>(R.t_diag[2]);
      det_diag[3] += static_cast<double>(R.t_diag[3] - R.t_phase[2]);
      for (int i = 0; i < 8; ++i) det_diag[4 + i] += static_cast<double>(R.hot_counts[i]);  // rows 0..7
      det_diag[12] += static_cast<double>(R.n_candidates);
      det_diag[13] += static_cast<double>(R.stage_count[R.stage_count[5] ? 5 : 3]);
      det_diag[14] += 1;
    }
    ++det_n;
  }

  // the kernel may now reuse group g's ring space below `upto` (mapped host word)
  static void release_arena(Batch& B, uint32_t g, uint64_t upto) {
    std::atomic_thread_fence(std::memory_order_release);
    *reinterpret_cast<volatile unsigned long long*>(B.arena_rel.p + g) = upto;
  }

  void finalize_batch(Batch& B) {
    for (; B.fin < B.wins.size(); ++B.fin) {
      wait_ready(B, B.fin);
      finalize_window(B, B.fin);
    }
    B.fin = 0;
    cuda_ok(cudaEventSynchronize(B.done), "engine batch");
    if (!B.op_kind.empty()) {
      cta_trace.resize(21 * B.op_kind.size() * ctx->detect_grid);
      cuda_ok(cudaMemcpy(cta_trace.data(), B.cta_t.p, cta_trace.size() * sizeof(uint64_t),
                         cudaMemcpyDeviceToHost),
              "D2H cta trace");
      cta_trace_ops = B.op_kind.size();
      B.op_t_h.resize(2 * B.op_kind.size());
      cuda_ok(cudaMemcpy(B.op_t_h.data(), B.op_t.p, B.op_t_h.size() * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost),
              "D2H op trace");
      for (size_t o = 0; o < B.op_kind.size(); ++o) {
        op_trace.push_back(B.op_kind[o]);
        op_trace.push_back(B.op_t_h[2 * o]);
        op_trace.push_back(~B.op_t_h[2 * o + 1]);
      }
    }
    B.op_kind.clear();
    B.wins.clear();
    B.live = false;
  }

  void finalize_batches() {
    for (int i = 0; i < 2; ++i) {
      Batch& B = batches[(next_batch + i) % 2];  // older first
      if (B.live) finalize_batch(B);
    }
  }

  // launch the accumulated ops over pairs `d` (device)
  // Incremental window tracking over a launch's ops (detect.cu
  // phase_a_inc): the first detect op runs the full pass and builds the live
  // structures (kOpInit), later ones re-examine only the blocks the window
  // moved past or a scan marked (kOpInc); every scan op after a detect op
  // marks blocks (kOpTrack). kOpLe: the SLEA too. Needs the sector geometry
  // (RSRA eta = 8, 8 | SLEA row_len) and window lows that only grow within
  // the launch (no reinitialize between windows).
  bool incremental_ok() const {
    return incremental && rs->cfg.eta == 8 && le->row_len % 8 == 0 && !cfg.reinit_per_window &&
           rs->hot_min >= 1 && inbox_role != 2;
  }

  bool incremental_le() const {
    return incremental_ok() && incremental != 3 &&
           (incremental == 2 || le->row_len * le->cfg.r * sizeof(uint32_t) > kLeIncBytes);
  }

  void mark_incremental() {
    if (!incremental_ok()) return;
    const uint32_t lef = incremental_le() ? dev::kOpLe : 0u;
    bool have = false;
    for (EngineOp& op : ops) {
      if (op.kind == 1) {
        op.flags = (have ? dev::kOpInc : dev::kOpInit) | lef;
        have = true;
      } else if (have) {
        op.flags |= dev::kOpTrack | lef;
      }
    }
  }

  void launch_batch(const srlg_pair* d, const unsigned* chunk_flags = nullptr) {
    if (ops.empty()) return;
    mark_incremental();
    ctx->ensure_detect();  // grid size and scratch before the launch is set up
    // reconstruction groups: no more groups than the launch has detections
    // (a launch with one detection reconstructs it on every reconstruction
    // CTA); the CTAs a multiple of the group count, at most half the grid
    uint32_t n_det = 0;
    for (const EngineOp& op : ops) n_det += op.kind == 1;
    // A tracked SLEA (state beyond L2, C4) has long slice periods (~230 us
    // against a ~60 us reconstruction), so one group keeps up and every
    // detection gets all the reconstruction CTAs (C4, 24 CTAs: x 1 / x 2 / x 3
    // per-slide latency 87 / 103 / 90+ us at the same throughput)
    const uint32_t G = std::max<uint32_t>(
        1, std::min<uint32_t>(incremental_le() ? 1u : recon_groups, n_det));
    for (size_t i = 0; i < ops.size(); ++i)
      ops[i].flags = (ops[i].flags & ~dev::kOpNextScan) |
                     (i + 1 < ops.size() && ops[i + 1].kind == 0 ? dev::kOpNextScan : 0u);
    Batch& B = batches[next_batch];
    if (B.live) finalize_batch(B);
    if (!B.done) cuda_ok(cudaEventCreateWithFlags(&B.done, cudaEventDisableTiming), "event");
    B.ops_h.ensure(ops.size());
    std::memcpy(B.ops_h.p, ops.data(), ops.size() * sizeof(EngineOp));
    B.ops_d.ensure(ops.size());
    cuda_ok(cudaMemcpyAsync(B.ops_d.p, B.ops_h.p, ops.size() * sizeof(EngineOp),
                            cudaMemcpyHostToDevice, ctx->st),
            "H2D ops");
    const uint64_t nw = std::max<size_t>(1, bwins.size());
    B.out.ensure(nw);
    B.cands.ensure(nw * kCandPrefix);
    B.ready.ensure(nw);
    std::memset(B.ready.p, 0, nw * sizeof(uint32_t));
    // any single window's tail fits the ring; the host frees it as it goes
    B.groups = G;
    B.arena_cap = arena_entries ? arena_entries : std::max(kArenaCands / G, cand_cap);
    B.arena.ensure(B.arena_cap * G);
    B.arena_rel.ensure(kMaxReconGroups);
    for (uint32_t i = 0; i < kMaxReconGroups; ++i) B.arena_rel.p[i] = 0;
    B.arena_heads.ensure(kMaxReconGroups);
    const uint32_t n_sets = G + 1;
    Candidate* cs[kMaxSets];
    for (uint32_t i = 0; i < n_sets; ++i) {
      bcands[i].ensure(cand_cap);
      cs[i] = bcands[i].p;
    }
    DetectParams P = make_detect_params(*ctx, rs, le, cfg.k, cfg.tuple_cap, cs[0], cand_cap);
    add_sets(*ctx, P, rs, n_sets, cs);
    P.recon_groups = G;
    if (incremental_ok()) {
      DeviceCtx& c = *ctx;
      const uint64_t rs_cells = (static_cast<uint64_t>(rs->cfg.r) << rs->cfg.q) * rs->cfg.eta;
      P.inc.rs_blocks = (rs_cells + kIncBlock - 1) / kIncBlock;
      c.rs_smin.ensure(P.inc.rs_blocks);
      c.live_hot.ensure(P.inc.rs_blocks);
      c.inc_stats.ensure(4);
      P.inc.rs_smin = c.rs_smin.p;
      P.inc.live_hot = c.live_hot.p;
      P.inc.stats = c.inc_stats.p;
      if (incremental_le()) {
        const uint64_t le_cells = le->row_len * le->cfg.r;
        P.inc.le_blocks = (le_cells + kIncBlock - 1) / kIncBlock;
        c.le_smin.ensure(P.inc.le_blocks);
        c.live_bits.ensure(2 * P.inc.le_blocks + 2);  // u64 per block
        c.live_row.ensure(kMaxRows);
        const uint64_t log_n = static_cast<uint64_t>(kLeLogSlots) * kLeLogCtas;
        c.le_log_idx.ensure(log_n * kLeLogCap);
        c.le_log_val.ensure(log_n * kLeLogCap);
        c.le_log_n.ensure(log_n);
        P.inc.le_smin = c.le_smin.p;
        P.inc.live_bits = c.live_bits.p;
        P.inc.live_row = c.live_row.p;
        P.inc.le_log_idx = c.le_log_idx.p;
        P.inc.le_log_val = c.le_log_val.p;
        P.inc.le_log_n = c.le_log_n.p;
      }
    }
    P.anet = anet;
    P.raw_records = anet.n ? raw_records.p : nullptr;
    // a sending rank only scans (no reconstruction group)
    {
      const uint32_t cap = static_cast<uint32_t>(ctx->detect_grid / 2) / G * G;
      const uint32_t want = static_cast<uint32_t>(recon_ctas) / G * G;
      P.recon_ctas = inbox_role == 2 ? 0u : std::max(G, std::min(want, cap));
    }
    P.diag = trace_ops ? 1u : 0u;
    EngineRing ring{B.out.dptr, B.cands.dptr, B.ready.dptr, B.arena.p, B.arena_cap, nullptr, nullptr,
                    chunk_flags, md, B.arena_rel.dptr, B.arena_heads.p, 0};
    // the leading scan-only ops (device-resident record input): one merged loop
    if (!chunk_flags && inbox_role == 0 && anet.n == 0) {
      uint32_t np = 0;
      while (np < ops.size() && np < dev::kMergedPrefixCap && ops[np].kind == 0 &&
             (np == 0 || ops[np].begin == ops[np - 1].end) && ops[np].end < (uint64_t{1} << 32))
        ++np;
      ring.merged_prefix = np >= 2 ? np : 0;
    }
    if (trace_ops) {
      B.op_t.ensure(2 * ops.size());
      cuda_ok(cudaMemsetAsync(B.op_t.p, 0xFF, 2 * ops.size() * sizeof(unsigned long long), ctx->st),
              "memset");
      for (size_t o = 0; o < ops.size(); ++o) B.op_kind.push_back(ops[o].kind);
      ring.op_t = B.op_t.p;
      B.cta_t.ensure(21 * ops.size() * ctx->detect_grid);
      cuda_ok(cudaMemsetAsync(B.cta_t.p, 0, 21 * ops.size() * ctx->detect_grid * 8, ctx->st), "memset");
      ring.cta_t = B.cta_t.p;
    }
    uint64_t pkts = 0;
    for (const EngineOp& op : ops) pkts += op.kind == 0 ? op.end - op.begin : 0;
    const size_t p0 = ctx->prof.on ? ctx->prof.begin(ctx->st) : 0;
    cuda_ok(dev::engine_run(P, B.ops_d.p, static_cast<uint32_t>(ops.size()), d, ring,
                            ctx->detect_grid, ctx->st),
            "engine kernel");
    g_launches++;
    if (ctx->prof.on) ctx->prof.end(ctx->st, 2, p0, pkts);
    ctx->d2h_bytes += bwins.size() * (sizeof(WinResult) + P.host_prefix * sizeof(Candidate));
    cuda_ok(cudaEventRecord(B.done, ctx->st), "record");
    B.wins = std::move(bwins);
    bwins.clear();
    ops.clear();
    B.live = true;
    next_batch ^= 1;
    Batch& O = batches[next_batch];  // the older batch finalises while this one runs
    if (O.live) finalize_batch(O);
  }

  void scan(const srlg_pair* d, uint64_t n) {
    if (!merge) {
      scan_pairs(*ctx, rs, le, d, n, anet.n ? &anet : nullptr, anet.n ? raw_records.p : nullptr);
      return;
    }
    RsraDev r = rs->dv;
    SleaDev l = le->dv;
    r.cells = reinterpret_cast<uint32_t*>(dirty);
    l.cells = reinterpret_cast<uint32_t*>(dirty + rs->n);
    const size_t p0 = ctx->prof.on ? ctx->prof.begin(ctx->st) : 0;
    cuda_ok(dev::scan(d, n, r, 0, l, 0, dev::kStoreMark, ctx->st, anet.n ? &anet : nullptr,
                      anet.n ? raw_records.p : nullptr),
            "scan kernel (marks)");
    g_launches++;
    if (ctx->prof.on) ctx->prof.end(ctx->st, 0, p0, n);
  }

  // the per-slide merge: NCCL max-reduce of the u8 maps onto the root
  void merge_slice() {
    const uint64_t n = rs->n + le->n;
    nccl_ok(nccl().reduce(dirty, dirty, n, ncclUint8, ncclMax, root, comm, ctx->st), "ncclReduce");
    if (rank == root) {
      cuda_ok(dev::apply_marks(dirty, rs->n, rs->cells, rs->now, le->n, le->cells, le->now,
                               ctx->st),
              "apply kernel");
      g_launches++;
    } else {
      cuda_ok(cudaMemsetAsync(dirty, 0, n, ctx->st), "memset");
    }
    ++merges;
    merge_bytes += n;
  }

  // SliceClock::place (src/window.cpp:24-34)
  uint64_t place(uint64_t ts) {
    if (!has_t0) {
      t0 = ts;
      has_t0 = true;
    }
    if (has_max && ts < max_ts) {
      if (max_ts - ts > cfg.regression_tolerance_us)
        raise(SRLG_ERR_ORDERING, "timestamp regression beyond tolerance");
      ++clamped;
      return (max_ts - t0) / cfg.slice_us;
    }
    if (!has_max || ts > max_ts) {
      max_ts = ts;
      has_max = true;
    }
    if (ts < t0) raise(SRLG_ERR_ORDERING, "timestamp precedes the stream start");
    return (ts - t0) / cfg.slice_us;
  }

  void drain_one() {
    PendingWindow w = inflight.front();
    inflight.pop_front();
    finalize_detect(*ctx, slots[w.slot], w, reports);
    ++n_reports;
  }

  void drain_slots() {
    while (!inflight.empty()) drain_one();
  }

  // windows finalise in issue order: persistent batches always precede the
  // per-slice windows still in flight (process_slices drains those first)
  void drain_all() {
    finalize_batches();
    drain_slots();
  }

  void detect(uint64_t end, bool partial) {
    // keep report order: earlier persistent batches are finalised before
    // this detection's record. With nothing in flight the detection is
    // enqueued first (stream order puts it after the batch on the device),
    // so the GPU does not idle while the host finalises the batch.
    const bool early = inflight.empty();
    if (!early) finalize_batches();
    if (static_cast<int>(inflight.size()) >= kSlots) drain_one();
    // an idle ring restarts at slot 0: a run's detections reuse the slots
    // (and their pinned buffers) the previous runs allocated, instead of
    // walking into a fresh slot (cudaHostAlloc: tens of ms) every call
    if (inflight.empty()) next_slot = 0;
    const int s = next_slot;
    next_slot = (s + 1) % kSlots;
    enqueue_detect(*ctx, rs, le, cfg.k, cfg.tuple_cap, slots[s], cand_cap);
    inflight.push_back(make_pending(rs, le, cfg, end, partial, s, cand_cap));
    if (early) finalize_batches();
  }

  // flush_pending (src/window.cpp:89-98)
  void flush() {
    if (pending.empty()) return;
    with_device_pairs(*ctx, pending.data(), pending.size(), 0,
                      [&](const srlg_pair* d, uint64_t n) { scan(d, n); });
    cuda_ok(cudaStreamSynchronize(ctx->cp), "copy sync");
    pending.clear();
  }

  // complete_slice (src/window.cpp:100-111); distributed: merged_detect
  // (src/distributed.cpp:72-85) on the root
  void complete_slice() {
    if (merge) merge_slice();
    if (current + 1 >= cfg.k && is_root()) detect(current, false);
    advance_clocks();
    ++current;
  }

  // persistent batches over pinned host input: every batch's pairs are
  // copied (copy stream) into the resident input buffer up front, each batch
  // launch waits only for its own copy
  void process_resident(const srlg_pair* pairs, const uint64_t* off, uint64_t n_slices,
                        uint64_t first_slice) {
    if (write_value32()) {
      process_streamed(pairs, off, n_slices, first_slice);
      return;
    }
    DeviceCtx& c = *ctx;
    const uint64_t base0 = off[0];
    c.input_d.ensure(off[n_slices] - base0);
    std::vector<std::pair<uint64_t, uint64_t>> groups;  // slice ranges of the batches
    for (uint64_t s = 0; s < n_slices;) {
      uint64_t s_end = s + 1;
      while (s_end < n_slices && off[s_end + 1] - off[s] <= kStagePairs) ++s_end;
      groups.emplace_back(s, s_end);
      s = s_end;
    }
    // the copy stream may not overwrite the buffer while an earlier batch reads it
    cuda_ok(cudaEventRecord(c.chunk_event(0), c.st), "record");
    cuda_ok(cudaStreamWaitEvent(c.cp, c.chunk_event(0), 0), "wait");
    std::vector<cudaEvent_t> tev;  // diagnostics (trace_ops): copy-done and launch times
    auto tevent = [&](cudaStream_t st) {
      cudaEvent_t e;
      cuda_ok(cudaEventCreate(&e), "event");
      cuda_ok(cudaEventRecord(e, st), "record");
      tev.push_back(e);
    };
    if (trace_ops) tevent(c.cp);
    for (size_t g = 0; g < groups.size(); ++g) {
      const uint64_t a = off[groups[g].first], b = off[groups[g].second];
      if (b > a)
        cuda_ok(cudaMemcpyAsync(c.input_d.p + (a - base0), pairs + a, (b - a) * sizeof(srlg_pair),
                                cudaMemcpyHostToDevice, c.cp),
                "H2D");
      c.h2d_bytes += (b - a) * sizeof(srlg_pair);
      cuda_ok(cudaEventRecord(c.chunk_event(g + 1), c.cp), "record");
      if (trace_ops) tevent(c.cp);
    }
    for (size_t g = 0; g < groups.size(); ++g) {
      cuda_ok(cudaStreamWaitEvent(c.st, c.chunk_event(g + 1), 0), "wait");
      const uint64_t s = groups[g].first, s_end = groups[g].second;
      const uint64_t base = off[s];
      add_slice_ops(off, s, s_end, first_slice, base, false);
      if (trace_ops) tevent(c.st);
      launch_batch(c.input_d.p + (base - base0));
    }
    // the caller may reuse its buffer once the call returns
    cuda_ok(cudaStreamSynchronize(c.cp), "copy sync");
    if (trace_ops) {
      cuda_ok(cudaStreamSynchronize(c.st), "sync");
      io_trace.clear();
      for (size_t i = 1; i < tev.size(); ++i) {
        float ms = 0;
        cuda_ok(cudaEventElapsedTime(&ms, tev[0], tev[i]), "elapsed");
        io_trace.push_back(ms);
      }
      for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
  }
  std::vector<float> io_trace;  // diagnostics: ms of each chunk copy done, then each launch

  // pinned host input as ONE persistent launch: the copy stream lands the
  // input in kChunkPairs pieces and flags each one (cuStreamWriteValue32);
  // the kernel's scan ops wait for their chunk's flag, so the copy engine and
  // the kernel run concurrently from the first chunk to the last
  void process_streamed(const srlg_pair* pairs, const uint64_t* off, uint64_t n_slices,
                        uint64_t first_slice) {
    DeviceCtx& c = *ctx;
    const uint64_t base0 = off[0], total = off[n_slices] - base0;
    const uint64_t n_chunks = (total + kChunkPairs - 1) / kChunkPairs;
    c.input_d.ensure(total);
    c.chunk_flags.ensure(n_chunks);
    // the copy stream may not overwrite input or flags an earlier launch still reads
    cuda_ok(cudaEventRecord(c.chunk_event(0), c.st), "record");
    cuda_ok(cudaStreamWaitEvent(c.cp, c.chunk_event(0), 0), "wait");
    cuda_ok(cudaMemsetAsync(c.chunk_flags.p, 0, n_chunks * sizeof(unsigned), c.cp), "memset");
    cuda_ok(cudaEventRecord(c.chunk_event(1), c.cp), "record");
    cuda_ok(cudaStreamWaitEvent(c.cp2, c.chunk_event(1), 0), "wait");
    // chunks alternate between two copy streams, so one stream's flag write
    // overlaps the other's copy; the kernel waits for every chunk's own flag
    for (uint64_t k = 0; k < n_chunks; ++k) {
      cudaStream_t cs = (k & 1) ? c.cp2 : c.cp;
      const uint64_t a = k * kChunkPairs, n = std::min(kChunkPairs, total - a);
      cuda_ok(cudaMemcpyAsync(c.input_d.p + a, pairs + base0 + a, n * sizeof(srlg_pair),
                              cudaMemcpyHostToDevice, cs),
              "H2D");
      if (write_value32()(cs, reinterpret_cast<unsigned long long>(c.chunk_flags.p + k), 1u, 0) != 0)
        raise(SRLG_ERR_CUDA, "cuStreamWriteValue32 failed");
      c.h2d_bytes += n * sizeof(srlg_pair);
    }
    add_slice_ops(off, 0, n_slices, first_slice, base0, true);
    cuda_ok(cudaStreamWaitEvent(c.st, c.chunk_event(1), 0), "wait");  // flags cleared
    cuda_ok(cudaEventRecord(c.chunk_event(2), c.cp), "record");
    cuda_ok(cudaEventRecord(c.chunk_event(3), c.cp2), "record");
    Batch& B = batches[next_batch];
    launch_batch(c.input_d.p, c.chunk_flags.p);
    // the caller may reuse its buffer once the call returns; meanwhile the
    // windows the kernel has already published are finalised
    while (cudaEventQuery(c.chunk_event(2)) == cudaErrorNotReady ||
           cudaEventQuery(c.chunk_event(3)) == cudaErrorNotReady) {
      if (B.live) finalize_ready(B);
      std::this_thread::yield();
    }
    cuda_ok(cudaStreamSynchronize(c.cp), "copy sync");
    cuda_ok(cudaStreamSynchronize(c.cp2), "copy sync");
  }

  void to_slice(uint64_t s) {
    if (s > current) {
      flush();
      while (current < s) complete_slice();
    }
  }
};

extern "C" {

int srlg_engine_create(const srlg_window_config* cfg, srlg_rsra* rsra, srlg_slea* slea,
                       srlg_engine** out) {
  *out = nullptr;
  return guarded([&] {
    check_window(*cfg);
    if (!rsra || !slea) raise(SRLG_ERR_INVALID_ARGUMENT, "engine needs both sketches");
    check_same_device(rsra, slea);
    auto e = std::make_unique<srlg_engine>();
    e->cfg = *cfg;
    e->rs = rsra;
    e->le = slea;
    e->ctx = rsra->ctx;
    e->has_t0 = cfg->has_t0 != 0;
    e->t0 = cfg->t0_us;
    e->cand_cap = cand_cap_for(cfg->tuple_cap);
    *out = e.release();
  });
}

// WindowEngine's copy (the reference engine is a value type, window.hpp:64-98):
// a new engine on the same device with deep copies of both sketches (device
// to device), the slice clock, the open slice's records and the reports not
// yet taken. Windows still in flight are finalised first.
int srlg_engine_clone(srlg_engine* src, srlg_engine** out) {
  *out = nullptr;
  return guarded([&] {
    DeviceGuard g(src->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(src->ctx->mu);
    if (src->merge || src->inbox_role)
      raise(SRLG_ERR_INVALID_ARGUMENT, "an engine of a merge group cannot be copied");
    src->drain_all();
    srlg_rsra* r = nullptr;
    srlg_slea* l = nullptr;
    int st = srlg_rsra_clone(src->rs, &r);
    if (st != SRLG_OK) raise(st, g_err);
    st = srlg_slea_clone(src->le, &l);
    if (st != SRLG_OK) {
      srlg_rsra_destroy(r);
      raise(st, g_err);
    }
    auto e = std::make_unique<srlg_engine>();
    e->cfg = src->cfg;
    e->rs = r;
    e->le = l;
    e->ctx = src->ctx;
    e->has_t0 = src->has_t0;
    e->has_max = src->has_max;
    e->t0 = src->t0;
    e->max_ts = src->max_ts;
    e->clamped = src->clamped;
    e->current = src->current;
    e->records = src->records;
    e->active = src->active;
    e->pending = src->pending;
    e->reports = src->reports;
    e->n_reports = src->n_reports;
    e->cand_cap = src->cand_cap;
    e->persistent = src->persistent;
    e->arena_entries = src->arena_entries;
    e->anet = src->anet;
    e->raw_packets = src->raw_packets;
    if (src->raw_records.p) {
      e->raw_records.ensure(1);
      cuda_ok(cudaMemcpyAsync(e->raw_records.p, src->raw_records.p, sizeof(unsigned long long),
                              cudaMemcpyDeviceToDevice, src->ctx->st),
              "D2D raw record count");
    }
    *out = e.release();
  });
}

void srlg_engine_destroy(srlg_engine* e) {
  if (!e) return;
  {
    DeviceGuard g(e->ctx->device);
    // windows in flight first: a kernel may wait for the host to drain its
    // candidate ring before the stream can drain
    try {
      std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
      e->drain_all();
    } catch (...) {
    }
    cudaStreamSynchronize(e->ctx->st);
    for (auto& s : e->slots) {
      if (s.res_d.p) cudaFree(s.res_d.p);
      if (s.cand_d.p) cudaFree(s.cand_d.p);
      if (s.res_h.p) cudaFreeHost(s.res_h.p);
      if (s.cand_h.p) cudaFreeHost(s.cand_h.p);
      if (s.ev) cudaEventDestroy(s.ev);
    }
  }
  if (e->dirty) cudaFree(e->dirty);
  if (e->inbox) {
    DeviceGuard g(e->ctx->device);
    if (e->inbox_role == 1) cudaFree(e->inbox);
    else if (e->inbox_ipc) cudaIpcCloseMemHandle(e->inbox);
  }
  for (auto& B : e->batches) {
    if (B.out.p) cudaFreeHost(B.out.p);
    if (B.cands.p) cudaFreeHost(B.cands.p);
    if (B.ready.p) cudaFreeHost(B.ready.p);
    if (B.ops_h.p) cudaFreeHost(B.ops_h.p);
    if (B.ops_d.p) cudaFree(B.ops_d.p);
    if (B.arena.p) cudaFree(B.arena.p);
    if (B.done) cudaEventDestroy(B.done);
  }
  for (auto& b : e->bcands)
    if (b.p) cudaFree(b.p);
  srlg_rsra_destroy(e->rs);
  srlg_slea_destroy(e->le);
  delete e;
}

// WindowEngine::process (src/window.cpp:122-131)
int srlg_engine_process(srlg_engine* e, const srlg_record* recs, uint64_t n) {
  return guarded([&] {
    // merge groups advance slice by slice in lockstep: every rank must see
    // the same slices, which pre-sliced calls make explicit
    if ((e->inbox_role || e->merge) && n)
      raise(SRLG_ERR_INVALID_ARGUMENT, "a merge group takes pre-sliced input (process_slices)");
    DeviceGuard g(e->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    for (uint64_t i = 0; i < n; ++i) {
      const uint64_t s = e->place(recs[i].ts_us);
      e->active = true;
      e->to_slice(s);
      e->pending.push_back(srlg_pair{recs[i].aip, recs[i].bip});
      ++e->records;
    }
    if (e->anet.n) e->raw_packets += n;  // raw mode: {ts, src, dst} packets
  });
}

// A binary trace file of timestamped records — the reference's TraceRecord /
// RawPacket layout {u64 ts_us, u32, u32}, 16 B each, little-endian (raw
// packets {ts, src, dst} when the engine has a monitored network) — read in
// blocks and fed through srlg_engine_process.
int srlg_engine_process_file(srlg_engine* e, const char* path, uint64_t* n_read) {
  return guarded([&] {
    *n_read = 0;
    FILE* f = std::fopen(path, "rb");
    if (!f) raise(SRLG_ERR_PARSE, std::string("cannot open trace file: ") + path);
    std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
    constexpr size_t kBlock = 1 << 20;  // records per read
    std::vector<srlg_record> buf(kBlock);
    while (true) {
      const size_t got = std::fread(buf.data(), 1, kBlock * sizeof(srlg_record), f);
      if (got % sizeof(srlg_record) != 0)
        raise(SRLG_ERR_FORMAT, std::string(path) + ": trailing partial record");
      const size_t n = got / sizeof(srlg_record);
      if (n) {
        const int st = srlg_engine_process(e, buf.data(), n);
        if (st != SRLG_OK) raise(st, g_err);
        *n_read += n;
      }
      if (got < kBlock * sizeof(srlg_record)) break;
    }
    if (std::ferror(f)) raise(SRLG_ERR_PARSE, std::string("read failed: ") + path);
  });
}

int srlg_engine_process_slices(srlg_engine* e, const srlg_pair* pairs,
                               const uint64_t* slice_offsets, uint64_t n_slices,
                               uint64_t first_slice, int pairs_on_device) {
  return guarded([&] {
    if (!e->has_t0 && !(e->cfg.has_t0))
      raise(SRLG_ERR_CONFIG, "process_slices needs a configured t0");
    DeviceCtx& c = *e->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    e->flush();
    e->drain_slots();  // reports keep their order: per-slice windows first
    const uint64_t total = slice_offsets[n_slices] - slice_offsets[0];
    if (e->anet.n) e->raw_packets += total;
    if (e->inbox_role && !e->persistent)
      raise(SRLG_ERR_INVALID_ARGUMENT, "in-engine merge needs persistent batches");
    if (!pairs_on_device && e->persistent && !e->merge && total > 0 && total <= kResidentPairs &&
        is_pinned_host(pairs + slice_offsets[0])) {
      e->process_resident(pairs, slice_offsets, n_slices, first_slice);
      return;
    }
    // group consecutive slices into staging-sized chunks for host input
    uint64_t s = 0;
    while (s < n_slices) {
      uint64_t s_end = s + 1;
      if (!pairs_on_device) {
        while (s_end < n_slices &&
               slice_offsets[s_end + 1] - slice_offsets[s] <= kStagePairs)
          ++s_end;
      } else {
        s_end = n_slices;
      }
      const uint64_t base = slice_offsets[s];
      const uint64_t cnt = slice_offsets[s_end] - base;
      auto run = [&](const srlg_pair* d, uint64_t) {
        if (e->persistent && !e->merge) {
          // the whole chunk as one persistent launch (detect.cu k_engine)
          e->add_slice_ops(slice_offsets, s, s_end, first_slice, base, false);
          e->launch_batch(d);
          return;
        }
        for (uint64_t j = s; j < s_end; ++j) {
          const uint64_t m = slice_offsets[j + 1] - slice_offsets[j];
          if (m == 0) continue;
          const uint64_t sl = e->slice_for_call(first_slice + j, true);
          e->active = true;
          e->to_slice(sl);
          // records of the open slice all write the same stamp, so they are
          // applied right away instead of being buffered
          e->scan(d + (slice_offsets[j] - base), m);
          e->records += m;
        }
      };
      if (pairs_on_device || cnt <= kStagePairs) {
        if (cnt == 0) {
          if (e->inbox_role) run(nullptr, 0);  // the empty slices are published all the same
          s = s_end;
          continue;
        }
        with_device_pairs(c, pairs + base, cnt, pairs_on_device, run);
      } else {
        // a single slice larger than one staging buffer
        if (e->inbox_role)
          raise(SRLG_ERR_INVALID_ARGUMENT,
                "in-engine merge: pass slices larger than 64 MB in pinned or device memory");
        for (uint64_t j = s; j < s_end; ++j) {
          const uint64_t m = slice_offsets[j + 1] - slice_offsets[j];
          if (m == 0) continue;
          const uint64_t sl = e->slice_for_call(first_slice + j, true);
          e->active = true;
          e->to_slice(sl);
          with_device_pairs(c, pairs + slice_offsets[j], m, 0,
                            [&](const srlg_pair* d, uint64_t k) { e->scan(d, k); });
          e->records += m;
        }
      }
      s = s_end;
    }
    if (e->merge && n_slices) {
      // every rank ends the call at its last slice (trailing empty slices
      // included), so the per-slice reduces stay paired across ranks
      e->active = true;
      e->to_slice(first_slice + n_slices - 1);
    }
    if (!pairs_on_device) cuda_ok(cudaStreamSynchronize(c.cp), "copy sync");
  });
}

// WindowEngine::advance_to_slice (src/window.cpp:113-120)
int srlg_engine_advance_to_slice(srlg_engine* e, uint64_t slice) {
  return guarded([&] {
    if (e->inbox_role)
      raise(SRLG_ERR_INVALID_ARGUMENT,
            "in-engine merge: pass the empty slices through process_slices instead");
    DeviceGuard g(e->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    if (!e->active && !e->has_max) {
      if (!e->cfg.has_t0)
        raise(SRLG_ERR_CONFIG, "cannot advance slices before the stream start is known");
      e->active = true;
    }
    e->flush();
    while (e->current < slice) e->complete_slice();
  });
}

// WindowEngine::finish (src/window.cpp:133-137)
int srlg_engine_finish(srlg_engine* e) {
  return guarded([&] {
    DeviceGuard g(e->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    if (!e->active) return;
    e->flush();
    if (e->merge) e->merge_slice();
    if (e->is_root()) e->detect(e->current, true);
  });
}

int srlg_engine_sync(srlg_engine* e) {
  return guarded([&] {
    DeviceGuard g(e->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    e->flush();
    e->drain_all();
    e->ctx->sync();
  });
}

int srlg_engine_take_reports(srlg_engine* e, uint8_t* blob, uint64_t cap, uint64_t* blob_bytes,
                             uint64_t* n_reports) {
  return guarded([&] {
    DeviceGuard g(e->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    e->drain_all();
    *blob_bytes = e->reports.size();
    if (n_reports) *n_reports = e->n_reports;
    if (blob && e->reports.size() <= cap) {
      std::memcpy(blob, e->reports.data(), e->reports.size());
      e->reports.clear();
      e->n_reports = 0;
    }
  });
}

uint64_t srlg_engine_current_slice(const srlg_engine* e) { return e->current; }
uint64_t srlg_engine_records(const srlg_engine* e) {
  if (!e->raw_records.p) return e->records;
  // raw packets produced a device-counted number of records
  std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
  DeviceGuard g(e->ctx->device);
  unsigned long long dev_records = 0;
  if (cudaMemcpyAsync(&dev_records, e->raw_records.p, sizeof dev_records, cudaMemcpyDeviceToHost,
                      e->ctx->st) != cudaSuccess ||
      cudaStreamSynchronize(e->ctx->st) != cudaSuccess) {
    cudaGetLastError();
    return e->records;
  }
  return e->records - e->raw_packets + dev_records;
}

// Raw-packet ingest for later process_slices calls (classify, trace.cpp:111-116)
int srlg_engine_set_anet(srlg_engine* e, const srlg_anet* a) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    DeviceGuard g(e->ctx->device);
    if (!a || a->n == 0) {
      e->anet = AnetDev{};
      return;
    }
    e->anet = to_anet(*a);
    if (!e->raw_records.p) {
      e->raw_records.ensure(1);
      cuda_ok(cudaMemsetAsync(e->raw_records.p, 0, sizeof(unsigned long long), e->ctx->st), "memset");
    }
  });
}
uint64_t srlg_engine_clamped(const srlg_engine* e) { return e->clamped; }
srlg_rsra* srlg_engine_rsra(srlg_engine* e) { return e->rs; }
srlg_slea* srlg_engine_slea(srlg_engine* e) { return e->le; }

int srlg_engine_reset(srlg_engine* e) {
  return guarded([&] {
    DeviceCtx& c = *e->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    e->drain_all();
    e->reports.clear();
    e->n_reports = 0;
    e->pending.clear();
    // fresh state: every stamp dead, clocks and slice position back to zero
    cuda_ok(cudaMemsetAsync(e->rs->cells, 0, e->rs->n * sizeof(uint32_t), c.st), "memset");
    cuda_ok(cudaMemsetAsync(e->le->cells, 0, e->le->n * sizeof(uint32_t), c.st), "memset");
    e->rs->now = e->le->now = kClockOrigin;
    e->rs->floor = e->le->floor = 0;
    e->rs->slides = e->le->slides = 0;
    e->has_t0 = e->cfg.has_t0 != 0;
    e->t0 = e->cfg.t0_us;
    e->has_max = false;
    e->max_ts = 0;
    e->clamped = 0;
    e->current = 0;
    e->records = 0;
    e->active = false;
    e->merges = e->merge_bytes = 0;
    e->raw_packets = 0;
    if (e->raw_records.p)
      cuda_ok(cudaMemsetAsync(e->raw_records.p, 0, sizeof(unsigned long long), c.st), "memset");
    if (e->dirty)
      cuda_ok(cudaMemsetAsync(e->dirty, 0, e->rs->n + e->le->n, c.st), "memset");
    if (e->inbox_role == 1)  // merge stats count per run (the slice sequence goes on)
      cuda_ok(cudaMemsetAsync(e->md.entries, 0, sizeof(unsigned long long), c.st), "memset");
  });
}

uint64_t srlg_engine_kernel_launches(srlg_engine* e) {
  const uint64_t now = g_launches.load();
  const uint64_t d = now - e->launches_at_take;
  e->launches_at_take = now;
  return d;
}

}  // extern "C"

// ======================================================== exact oracle
// ExactSlidingOracle (exact_oracle.hpp:25-62, exact_oracle.cpp:22-101) on
// the device (exact.cu), over pre-sliced input like srlg_engine_process_slices.
struct srlg_exact {
  DeviceCtx* ctx = nullptr;
  uint64_t theta = 1024;
  uint32_t k = 300;
  uint64_t max_pairs = 0;
  uint64_t mask = 0, amask = 0;  // table slots - 1 (each table has one spare slot more)
  unsigned long long* keys = nullptr;
  uint32_t* stamps = nullptr;
  uint32_t* akeys = nullptr;
  uint32_t* counts = nullptr;
  unsigned long long* n_pairs = nullptr;  // device: distinct pairs ever seen
  unsigned long long* n_out = nullptr;
  DevBuf<uint64_t> out;
  uint32_t now = 1;  // stamp of the open slice (0 = never seen)
  uint64_t current = 0;
  bool active = false;
  uint64_t pairs_seen = 0;
  std::vector<uint8_t> windows;  // blob: per window {u64 end, u32 partial, u32 n} + n x {u32 aip, u32 0, u64 card}
  uint64_t n_windows = 0;

  void window(bool partial) {
    DeviceCtx& c = *ctx;
    const uint32_t lo = now > k ? now - k : 0;  // live iff last seen slice > current - k
    const uint64_t cap = out.n;
    cuda_ok(cudaMemsetAsync(n_out, 0, sizeof(unsigned long long), c.st), "memset");
    cuda_ok(dev::exact_window(keys, stamps, mask + 2, lo, akeys, counts, amask, theta, out.p, n_out,
                              cap, c.st),
            "exact window kernels");
    g_launches += 2;
    unsigned long long n = 0;
    cuda_ok(cudaMemcpyAsync(&n, n_out, sizeof n, cudaMemcpyDeviceToHost, c.st), "D2H");
    c.sync();
    if (n > cap) {  // more super hosts than the buffer: grow and redo (tables were cleared)
      raise(SRLG_ERR_RESOURCE, "exact oracle: super-point buffer exhausted");
    }
    std::vector<uint64_t> got(n);
    if (n)
      cuda_ok(cudaMemcpy(got.data(), out.p, n * sizeof(uint64_t), cudaMemcpyDeviceToHost), "D2H");
    std::vector<std::pair<uint32_t, uint64_t>> supers;
    supers.reserve(n);
    for (uint64_t v : got) supers.emplace_back(static_cast<uint32_t>(v >> 32), v & 0xFFFFFFFFu);
    // cardinality desc, aip asc (exact_oracle.cpp:85-89)
    std::sort(supers.begin(), supers.end(), [](const auto& a, const auto& b) {
      if (a.second != b.second) return a.second > b.second;
      return a.first < b.first;
    });
    const uint64_t end = current;
    const uint32_t part = partial ? 1u : 0u, cnt = static_cast<uint32_t>(supers.size());
    put(windows, &end, 8);
    put(windows, &part, 4);
    put(windows, &cnt, 4);
    for (const auto& sp : supers) {
      const uint32_t zero = 0;
      put(windows, &sp.first, 4);
      put(windows, &zero, 4);
      put(windows, &sp.second, 8);
    }
    ++n_windows;
  }

  // complete_slice (exact_oracle.cpp:72-77): emit from k-1 on, then advance
  void complete_slice() {
    if (current + 1 >= k) window(false);
    ++now;
    ++current;
  }
};

extern "C" {

int srlg_exact_create(uint64_t theta, uint32_t k, uint64_t max_pairs, int device, srlg_exact** out) {
  *out = nullptr;
  return guarded([&] {
    if (k == 0 || k > 65534) raise(SRLG_ERR_CONFIG, "k must be in [1, 65534]");
    if (max_pairs == 0) raise(SRLG_ERR_CONFIG, "exact oracle: max_pairs must be positive");
    auto e = std::make_unique<srlg_exact>();
    e->ctx = &ctx_for(device);
    DeviceGuard g(e->ctx->device);
    e->theta = theta;
    e->k = k;
    e->max_pairs = max_pairs;
    uint64_t slots = 1 << 16;
    while (slots < 2 * max_pairs) slots <<= 1;  // load factor <= 1/2
    e->mask = slots - 1;
    e->amask = slots - 1;
    cuda_ok(cudaMalloc(&e->keys, (slots + 1) * sizeof(unsigned long long)), "cudaMalloc (exact)");
    cuda_ok(cudaMalloc(&e->stamps, (slots + 1) * sizeof(uint32_t)), "cudaMalloc (exact)");
    cuda_ok(cudaMalloc(&e->akeys, (slots + 1) * sizeof(uint32_t)), "cudaMalloc (exact)");
    cuda_ok(cudaMalloc(&e->counts, (slots + 1) * sizeof(uint32_t)), "cudaMalloc (exact)");
    cuda_ok(cudaMalloc(&e->n_pairs, 2 * sizeof(unsigned long long)), "cudaMalloc (exact)");
    e->n_out = e->n_pairs + 1;
    cudaStream_t st = e->ctx->st;
    cuda_ok(cudaMemsetAsync(e->keys, 0xFF, (slots + 1) * sizeof(unsigned long long), st), "memset");
    cuda_ok(cudaMemsetAsync(e->stamps, 0, (slots + 1) * sizeof(uint32_t), st), "memset");
    cuda_ok(cudaMemsetAsync(e->akeys, 0xFF, (slots + 1) * sizeof(uint32_t), st), "memset");
    cuda_ok(cudaMemsetAsync(e->counts, 0, (slots + 1) * sizeof(uint32_t), st), "memset");
    cuda_ok(cudaMemsetAsync(e->n_pairs, 0, 2 * sizeof(unsigned long long), st), "memset");
    e->out.ensure(1 << 16);
    *out = e.release();
  });
}

void srlg_exact_destroy(srlg_exact* e) {
  if (!e) return;
  DeviceGuard g(e->ctx->device);
  cudaStreamSynchronize(e->ctx->st);
  cudaFree(e->keys);
  cudaFree(e->stamps);
  cudaFree(e->akeys);
  cudaFree(e->counts);
  cudaFree(e->n_pairs);
  if (e->out.p) cudaFree(e->out.p);
  delete e;
}

// ExactSlidingOracle::process over pre-sliced pairs (slice j of the call is
// slice first_slice + j); the distinct-pair budget is checked after the call
// (ResourceError "exact oracle: distinct pair budget exceeded")
int srlg_exact_process_slices(srlg_exact* e, const srlg_pair* pairs, const uint64_t* offsets,
                              uint64_t n_slices, uint64_t first_slice, int pairs_on_device) {
  return guarded([&] {
    DeviceCtx& c = *e->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    for (uint64_t j = 0; j < n_slices; ++j) {
      const uint64_t m = offsets[j + 1] - offsets[j];
      if (m == 0) continue;
      const uint64_t sl = first_slice + j;
      if (sl < e->current) raise(SRLG_ERR_ORDERING, "exact oracle: slices must not go back");
      e->active = true;
      while (e->current < sl) e->complete_slice();
      with_device_pairs(c, pairs + offsets[j], m, pairs_on_device, [&](const srlg_pair* d, uint64_t n) {
        cuda_ok(dev::exact_insert(d, n, e->now, e->keys, e->stamps, e->mask, e->n_pairs, c.st),
                "exact insert");
        g_launches++;
      });
    }
    if (!pairs_on_device) cuda_ok(cudaStreamSynchronize(c.cp), "copy sync");
    unsigned long long n = 0;
    cuda_ok(cudaMemcpyAsync(&n, e->n_pairs, sizeof n, cudaMemcpyDeviceToHost, c.st), "D2H");
    c.sync();
    e->pairs_seen = n;
    if (n > e->max_pairs) raise(SRLG_ERR_RESOURCE, "exact oracle: distinct pair budget exceeded");
  });
}

// finish (exact_oracle.cpp:95-98): the partial window at stream end
int srlg_exact_finish(srlg_exact* e) {
  return guarded([&] {
    DeviceGuard g(e->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    if (e->active) e->window(true);
  });
}

uint64_t srlg_exact_distinct_pairs(const srlg_exact* e) { return e->pairs_seen; }

int srlg_exact_take_windows(srlg_exact* e, uint8_t* blob, uint64_t cap, uint64_t* bytes,
                            uint64_t* n_windows) {
  return guarded([&] {
    *bytes = e->windows.size();
    *n_windows = e->n_windows;
    if (!blob) return;
    if (cap < e->windows.size()) raise(SRLG_ERR_INVALID_ARGUMENT, "take_windows: buffer too small");
    std::memcpy(blob, e->windows.data(), e->windows.size());
    e->windows.clear();
    e->n_windows = 0;
  });
}

}  // extern "C"

// ============================================================ diagnostics

extern "C" {

void* srlg_device_stream(int device) {
  void* out = nullptr;
  guarded([&] { out = ctx_for(device).st; });
  return out;
}

int srlg_profile_enable(int device, int on) {
  return guarded([&] {
    DeviceCtx& c = ctx_for(device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    c.sync();
    c.prof.collect();
    c.prof.on = on != 0;
  });
}

int srlg_profile_read(int device, double* scan_ms, uint64_t* scan_launches, uint64_t* scan_pairs,
                      double* detect_ms, uint64_t* detect_windows) {
  return guarded([&] {
    DeviceCtx& c = ctx_for(device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    c.sync();
    c.prof.collect();
    *scan_ms = c.prof.ms[0];
    *scan_launches = c.prof.count[0];
    *scan_pairs = c.prof.units[0];
    *detect_ms = c.prof.ms[1];
    *detect_windows = c.prof.count[1];
    c.prof.ms[0] = c.prof.ms[1] = 0;
    c.prof.count[0] = c.prof.count[1] = 0;
    c.prof.units[0] = c.prof.units[1] = 0;
  });
}

// globaltimer (ns) at the phase boundaries of the last fused detection:
// start, counts done, barrier, reconstruction done, barrier, usle done, end
int srlg_detect_phase_ns(int device, uint64_t* out16) {
  return guarded([&] {
    DeviceCtx& c = ctx_for(device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    c.sync();
    DetectScratch s{};
    if (c.scratch)
      cuda_ok(cudaMemcpy(&s, c.scratch, sizeof s, cudaMemcpyDeviceToHost), "D2H");
    for (int i = 0; i < 16; ++i) out16[i] = s.phase_ns[i];
  });
}

// persistent engine batches (kind 2): CUDA-event time, launches, packets
int srlg_profile_read_engine(int device, double* ms, uint64_t* launches, uint64_t* pairs) {
  return guarded([&] {
    DeviceCtx& c = ctx_for(device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    DeviceGuard g(c.device);
    c.sync();
    c.prof.collect();
    *ms = c.prof.ms[2];
    *launches = c.prof.count[2];
    *pairs = c.prof.units[2];
    c.prof.ms[2] = 0;
    c.prof.count[2] = c.prof.units[2] = 0;
  });
}

// device time (globaltimer) of the detections finalised from persistent
// batches since the last call: start of phase A1 to the record write
int srlg_engine_detect_latency(srlg_engine* e, double* mean_us, uint64_t* windows) {
  *windows = e->det_n;
  *mean_us = e->det_n ? e->det_ns_sum / e->det_n * 1e-3 : 0.0;
  e->det_n = 0;
  e->det_ns_sum = 0;
  return SRLG_OK;
}

// mean µs per phase (A1, barrier, B||A2, barrier, C, epilogue) of the
// detections finalised since the last call, CTA 0's view
int srlg_engine_detect_phases(srlg_engine* e, double* out6) {
  for (int i = 0; i < 6; ++i) {
    out6[i] = e->det_n ? e->det_phase_ns[i] / e->det_n * 1e-3 : 0.0;
    e->det_phase_ns[i] = 0;
  }
  return SRLG_OK;
}

// diagnostics: record the device span (first CTA in, last CTA out) of every
// op of later persistent batches; read them back as {kind, start_ns, end_ns}
int srlg_engine_trace_ops(srlg_engine* e, int on) {
  e->trace_ops = on != 0;
  return SRLG_OK;
}

int srlg_engine_read_op_trace(srlg_engine* e, uint64_t* out, uint64_t cap, uint64_t* n) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    e->drain_all();
    *n = e->op_trace.size() / 3;
    if (out) {
      std::memcpy(out, e->op_trace.data(), std::min<uint64_t>(cap, *n) * 3 * sizeof(uint64_t));
      e->op_trace.clear();
    }
  });
}

// diagnostics of traced batches, means per detection: [0] last DFS warp end,
// [1] last A2 warp end, [3] inversion end (µs after phase B starts), [2] DFS
// warps per CTA, [4..11] hot SREs per row, [12] candidates, [13] complete
// tuples, [14] detections
int srlg_engine_detect_diag(srlg_engine* e, double* out16) {
  const double n = e->det_diag[14];
  for (int i = 0; i < 16; ++i) {
    double v = e->det_diag[i];
    if (i != 14 && n) v /= n;
    if ((i <= 1 || i == 3) && n) v *= 1e-3;
    out16[i] = v;
    e->det_diag[i] = 0;
  }
  return SRLG_OK;
}

// diagnostics: the last traced resident-input run: ms (from the first copy)
// at which each chunk copy finished, then at which each batch was launched
int srlg_engine_read_io_trace(srlg_engine* e, float* out, uint64_t cap, uint64_t* n) {
  *n = e->io_trace.size();
  if (out) std::memcpy(out, e->io_trace.data(), std::min<uint64_t>(cap, *n) * sizeof(float));
  return SRLG_OK;
}

// diagnostics: per-CTA {start, end} ns of every op of the last traced batch
int srlg_engine_read_cta_trace(srlg_engine* e, uint64_t* out, uint64_t cap, uint64_t* n_ops,
                               uint64_t* grid) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    e->drain_all();
    *n_ops = e->cta_trace_ops;
    *grid = static_cast<uint64_t>(e->ctx->detect_grid);
    if (out) std::memcpy(out, e->cta_trace.data(), std::min<uint64_t>(cap, e->cta_trace.size()) * 8);
  });
}

// capacity (candidates) of the ring holding the candidates past each
// window's host prefix during persistent batches (0 = default: the largest
// tail one window can have); smaller rings only make the kernel wait for the
// host to drain earlier windows
int srlg_engine_set_arena(srlg_engine* e, uint64_t entries) {
  return guarded([&] {
    if (entries && entries < 1024) raise(SRLG_ERR_INVALID_ARGUMENT, "arena below 1024 candidates");
    e->arena_entries = entries;
  });
}

// Persistent batches track the window incrementally: the first detection of
// a launch sweeps the whole state, later ones re-examine only the blocks the
// window moved past or a scan marked. 1 (default): the RSRA always, the SLEA
// when its stamps exceed kLeIncBytes; 2: both always; 3: the RSRA only; 0:
// every detection sweeps the whole state. Results are identical in every mode.
int srlg_engine_set_incremental(srlg_engine* e, int mode) {
  return guarded([&] {
    if (mode < 0 || mode > 3) raise(SRLG_ERR_INVALID_ARGUMENT, "incremental mode must be 0..3");
    e->incremental = mode;
  });
}

// reconstruction pipeline of persistent batches: `ctas` CTAs (rounded to a
// multiple of `groups`, at most half the grid) in `groups` groups taking
// every groups-th detection, with groups + 1 buffer sets in flight; 0 keeps
// a value (defaults 24 CTAs, 3 groups)
int srlg_engine_set_recon(srlg_engine* e, int ctas, int groups) {
  return guarded([&] {
    if (ctas < 0 || groups < 0 || groups > static_cast<int>(kMaxReconGroups))
      raise(SRLG_ERR_INVALID_ARGUMENT, "recon groups must be 1..8");
    if (groups) e->recon_groups = groups;
    if (ctas) e->recon_ctas = ctas;
  });
}

// diagnostics: blocks the incremental detections re-examined since the last
// call ({RSRA, SLEA, 0, 0}; counted while srlg_engine_trace_ops is on)
int srlg_engine_inc_stats(srlg_engine* e, uint64_t out[4]) {
  return guarded([&] {
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    e->drain_all();
    DeviceCtx& c = *e->ctx;
    for (int i = 0; i < 4; ++i) out[i] = 0;
    if (!c.inc_stats.p) return;
    c.sync();
    cuda_ok(cudaMemcpy(out, c.inc_stats.p, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost), "D2H");
    cuda_ok(cudaMemset(c.inc_stats.p, 0, 4 * sizeof(uint64_t)), "memset");
  });
}

// 0: every slice through its own launches (scan, then detect); 1 (default):
// pre-sliced input runs as persistent batches
int srlg_engine_set_persistent(srlg_engine* e, int on) {
  e->persistent = on != 0;
  return SRLG_OK;
}

int srlg_io_bytes(int device, uint64_t* h2d, uint64_t* d2h) {
  return guarded([&] {
    DeviceCtx& c = ctx_for(device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    *h2d = c.h2d_bytes;
    *d2h = c.d2h_bytes;
    c.h2d_bytes = c.d2h_bytes = 0;
  });
}

}  // extern "C"

extern "C" {

// Random-update roofline: best-of-`reps` rate (updates/s) of n_updates random
// u32 stores (mode 0) or red.max (mode 1) into n_cells u32 on `device`.
int srlg_bench_random_updates(int device, uint64_t n_cells, uint64_t n_updates, int mode,
                              int reps, double* updates_per_s) {
  return guarded([&] {
    DeviceCtx& c = ctx_for(device);
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    uint32_t* buf = nullptr;
    cuda_ok(cudaMalloc(&buf, n_cells * sizeof(uint32_t)), "cudaMalloc");
    cuda_ok(cudaMemsetAsync(buf, 0, n_cells * sizeof(uint32_t), c.st), "memset");
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    for (int i = 0; i < reps + 1; ++i) {
      cuda_ok(cudaEventRecord(a, c.st), "record");
      cuda_ok(dev::random_updates(buf, n_cells, n_updates, mode, 1234 + i, 100 + i, c.n_sms, c.st),
              "random update kernel");
      cuda_ok(cudaEventRecord(b, c.st), "record");
      cuda_ok(cudaEventSynchronize(b), "sync");
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (i > 0) best = std::max(best, n_updates / (ms * 1e-3));  // first launch = warm-up
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(buf);
    *updates_per_s = best;
  });
}

// Random-update roofline on the trace's own address distribution (SURVEY.md
// §8d "R", for traces whose hot cells are not uniform, e.g. C4): the cell
// indices of n device-resident pairs are materialised once, then replayed as
// red.max into a fresh buffer of the sketches' footprint; best of `reps`.
int srlg_bench_trace_updates(const srlg_rsra* rs, const srlg_slea* le, const srlg_pair* dpairs,
                             uint64_t n, int reps, double* updates_per_s, uint64_t* n_updates) {
  return guarded([&] {
    check_same_device(rs, le);
    DeviceCtx& c = *rs->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    const uint64_t cells = rs->n + le->n;
    if (cells >= (uint64_t{1} << 32)) raise(SRLG_ERR_CONFIG, "trace replay: more than 2^32 cells");
    const uint64_t n_le = n * le->cfg.r;
    uint32_t *idx = nullptr, *buf = nullptr;
    unsigned long long* cnt = nullptr;
    cuda_ok(cudaMalloc(&idx, (n_le + n * rs->cfg.r) * sizeof(uint32_t)), "cudaMalloc (indices)");
    cuda_ok(cudaMalloc(&buf, cells * sizeof(uint32_t)), "cudaMalloc (replay state)");
    cuda_ok(cudaMalloc(&cnt, sizeof(unsigned long long)), "cudaMalloc");
    cuda_ok(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), c.st), "memset");
    cuda_ok(cudaMemsetAsync(buf, 0, cells * sizeof(uint32_t), c.st), "memset");
    cuda_ok(dev::trace_indices(dpairs, n, rs->dv, le->dv, idx, idx + n_le, cnt, c.n_sms, c.st),
            "trace index kernel");
    unsigned long long n_rs = 0;
    cuda_ok(cudaMemcpyAsync(&n_rs, cnt, sizeof n_rs, cudaMemcpyDeviceToHost, c.st), "D2H");
    c.sync();
    // RSRA entries follow the SLEA ones directly: one contiguous stream
    const uint64_t total = n_le + n_rs;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    double best = 0;
    for (int i = 0; i < reps + 1; ++i) {
      cuda_ok(cudaEventRecord(a, c.st), "record");
      cuda_ok(dev::replay_updates(idx, total, buf, 100 + i, c.n_sms, c.st), "replay kernel");
      cuda_ok(cudaEventRecord(b, c.st), "record");
      cuda_ok(cudaEventSynchronize(b), "sync");
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      if (i > 0) best = std::max(best, total / (ms * 1e-3));
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(idx);
    cudaFree(buf);
    cudaFree(cnt);
    *updates_per_s = best;
    *n_updates = total;
  });
}

// ------------------------------------------------------------ multi-GPU

int srlg_nccl_unique_id(uint8_t* out128) {
  return guarded([&] {
    ncclUniqueId id;
    nccl_ok(nccl().getUniqueId(&id), "ncclGetUniqueId");
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof id);
  });
}

int srlg_nccl_comm_create(int nranks, const uint8_t* id128, int rank, int device, void** comm) {
  *comm = nullptr;
  return guarded([&] {
    DeviceGuard g(ctx_for(device).device);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    ncclComm_t c = nullptr;
    nccl_ok(nccl().commInitRank(&c, nranks, id, rank), "ncclCommInitRank");
    *comm = c;
  });
}

int srlg_nccl_comm_destroy(void* comm) {
  return guarded([&] {
    if (comm) nccl_ok(nccl().commDestroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy");
  });
}

// Switch an engine to the distributed mode: this rank scans
// its own edge-router stream; every completed slice the touched-cell maps of
// all ranks are max-reduced onto `root`, whose sketches therefore hold the
// global state (the reference's merged min of distances, distributed.cpp:72-85)
// and which alone emits reports. Must be called before any record.
int srlg_engine_set_merge(srlg_engine* e, void* comm, int rank, int nranks, int root) {
  return guarded([&] {
    if (e->active || e->records) raise(SRLG_ERR_INVALID_ARGUMENT, "set_merge after records");
    // one global slice clock: every rank must place slices identically
    if (!e->cfg.has_t0) raise(SRLG_ERR_CONFIG, "NCCL merge needs a configured t0 on every rank");
    if (e->inbox_role) raise(SRLG_ERR_INVALID_ARGUMENT, "engine already in an in-engine merge group");
    if (!comm || nranks < 1 || rank < 0 || rank >= nranks || root < 0 || root >= nranks)
      raise(SRLG_ERR_INVALID_ARGUMENT, "bad merge group");
    DeviceGuard g(e->ctx->device);
    std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
    const uint64_t n = e->rs->n + e->le->n;
    if (!e->dirty) cuda_ok(cudaMalloc(&e->dirty, n), "cudaMalloc (dirty map)");
    cuda_ok(cudaMemsetAsync(e->dirty, 0, n, e->ctx->st), "memset");
    e->merge = true;
    e->comm = static_cast<ncclComm_t>(comm);
    e->rank = rank;
    e->nranks = nranks;
    e->root = root;
  });
}

// DistributedStats (include/slidecard/distributed.hpp:21-24): merges done and
// bytes each rank contributed to them (in-engine merge, on the root: 4 B per
// list entry applied)
int srlg_engine_merge_stats(srlg_engine* e, uint64_t* slice_merges, uint64_t* bytes) {
  return guarded([&] {
    *slice_merges = e->merges;
    *bytes = e->merge_bytes;
    if (e->inbox_role == 1) {
      DeviceGuard g(e->ctx->device);
      std::lock_guard<std::recursive_mutex> lk(e->ctx->mu);
      e->drain_all();
      InboxHeader h{};
      cuda_ok(cudaMemcpy(&h, e->inbox, sizeof h, cudaMemcpyDeviceToHost), "D2H inbox header");
      *bytes = 4 * static_cast<uint64_t>(h.entries);
    }
  });
}

}  // extern "C"

namespace {

constexpr uint64_t kInboxMagic = 0x584f424e49474c52ull;  // "RLGINBOX"
constexpr uint64_t kInboxHdrBytes = 4096;
constexpr uint64_t kEngineThreads = 512;  // detect.cu kThreads

void check_fresh_for_merge(const srlg_engine* e) {
  if (e->active || e->records || e->merge || e->inbox_role)
    raise(SRLG_ERR_INVALID_ARGUMENT, "merge group must be set up on a fresh engine");
  if (e->rs->n + e->le->n >= (uint64_t{1} << 32))
    raise(SRLG_ERR_CONFIG, "in-engine merge: more than 2^32 cells");
}

// wire `e` to the inbox at `base` (root memory) as `rank`
void bind_inbox(srlg_engine* e, void* base, const InboxHeader& h, int rank, int role) {
  auto* p = static_cast<uint8_t*>(base);
  e->inbox_role = role;
  e->inbox_max_pairs = h.max_pairs;
  e->md.role = static_cast<uint32_t>(role);
  e->md.rank = static_cast<uint32_t>(rank);
  e->md.nranks = h.nranks;
  e->md.slot_cap = h.slot_cap;
  e->md.rs_n = h.rs_n;
  e->md.hdr = reinterpret_cast<InboxRank*>(p + kInboxHdrBytes);
  e->md.lists = reinterpret_cast<uint32_t*>(p + kInboxHdrBytes + h.nranks * sizeof(InboxRank));
  e->md.entries = reinterpret_cast<unsigned long long*>(p + offsetof(InboxHeader, entries));
  e->rank = rank;
  e->nranks = static_cast<int>(h.nranks);
  e->root = 0;
}

InboxHeader read_inbox_header(const srlg_engine* e, const void* base, int rank) {
  InboxHeader h{};
  cuda_ok(cudaMemcpy(&h, base, sizeof h, cudaMemcpyDeviceToHost), "D2H inbox header");
  if (h.magic != kInboxMagic) raise(SRLG_ERR_INVALID_ARGUMENT, "not a merge inbox");
  if (rank < 1 || static_cast<uint32_t>(rank) >= h.nranks)
    raise(SRLG_ERR_INVALID_ARGUMENT, "merge rank out of range");
  if (h.rs_n != e->rs->n || h.le_n != e->le->n)
    raise(SRLG_ERR_INCOMPATIBLE, "merge group: sketch geometries differ");
  if (static_cast<uint64_t>(e->ctx->detect_grid) > kInboxMaxCtas)
    raise(SRLG_ERR_CONFIG, "merge rank grid exceeds the inbox regions");
  return h;
}

}  // namespace

extern "C" {

// Make `root` rank 0 of an in-engine merge group of `nranks`:
// its device memory gets the inbox the other ranks publish their slices' moved
// cells into, sized for max_pairs_per_slice packets per slice and rank. The
// IPC handle (64 bytes, when ipc_handle_out is not null) lets ranks in other
// processes map it (srlg_engine_merge_join).
int srlg_engine_merge_create(srlg_engine* root, int nranks, uint64_t max_pairs_per_slice,
                             uint8_t* ipc_handle_out) {
  return guarded([&] {
    check_fresh_for_merge(root);
    if (nranks < 1 || nranks > 64) raise(SRLG_ERR_INVALID_ARGUMENT, "merge group of 1..64 ranks");
    if (max_pairs_per_slice == 0) raise(SRLG_ERR_INVALID_ARGUMENT, "max_pairs_per_slice must be > 0");
    DeviceCtx& c = *root->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    c.ensure_detect();
    // a CTA appends at most ceil(m / (G * T)) * T * U entries (U cells per
    // packet: two records per raw packet), so regions of slot_cap / G
    // entries never overflow for m <= max_pairs and G <= kInboxMaxCtas
    const uint64_t U = 2ull * (root->rs->cfg.r + root->le->cfg.r);
    InboxHeader h{};
    h.magic = kInboxMagic;
    h.nranks = static_cast<uint32_t>(nranks);
    h.slots = kInboxSlots;
    h.slot_cap = (max_pairs_per_slice + kInboxMaxCtas * kEngineThreads) * U;
    h.rs_n = root->rs->n;
    h.le_n = root->le->n;
    h.max_pairs = max_pairs_per_slice;
    const uint64_t bytes = kInboxHdrBytes + nranks * sizeof(InboxRank) +
                           static_cast<uint64_t>(nranks) * kInboxSlots * h.slot_cap * 4;
    void* base = nullptr;
    cuda_ok(cudaMalloc(&base, bytes), "cudaMalloc (merge inbox)");
    root->inbox = base;
    cuda_ok(cudaMemset(base, 0, kInboxHdrBytes + nranks * sizeof(InboxRank)), "memset");
    cuda_ok(cudaMemcpy(base, &h, sizeof h, cudaMemcpyHostToDevice), "H2D inbox header");
    bind_inbox(root, base, h, 0, 1);
    if (ipc_handle_out) {
      cudaIpcMemHandle_t ih;
      cuda_ok(cudaIpcGetMemHandle(&ih, base), "cudaIpcGetMemHandle");
      static_assert(sizeof(ih) == 64, "cudaIpcMemHandle_t is 64 bytes");
      std::memcpy(ipc_handle_out, &ih, sizeof ih);
    }
  });
}

// Join as sending rank `rank` (>= 1) through the root's IPC handle (another
// process; its GPU reaches the root's memory over NVLink / P2P).
int srlg_engine_merge_join(srlg_engine* e, int rank, const uint8_t* ipc_handle) {
  return guarded([&] {
    check_fresh_for_merge(e);
    DeviceCtx& c = *e->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    c.ensure_detect();
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, ipc_handle, sizeof ih);
    void* base = nullptr;
    cuda_ok(cudaIpcOpenMemHandle(&base, ih, cudaIpcMemLazyEnablePeerAccess),
            "cudaIpcOpenMemHandle (merge inbox)");
    e->inbox = base;
    e->inbox_ipc = true;
    bind_inbox(e, base, read_inbox_header(e, base, rank), rank, 2);
  });
}

// Join as sending rank `rank` (>= 1) of the group whose root engine lives in
// this process (another GPU with peer access, or another execution lane of
// the same GPU: virtual ranks).
int srlg_engine_merge_attach(srlg_engine* e, int rank, srlg_engine* root) {
  return guarded([&] {
    check_fresh_for_merge(e);
    if (!root || root->inbox_role != 1) raise(SRLG_ERR_INVALID_ARGUMENT, "not a merge root");
    DeviceCtx& c = *e->ctx;
    DeviceGuard g(c.device);
    std::lock_guard<std::recursive_mutex> lk(c.mu);
    c.ensure_detect();
    if (root->ctx->device != c.device) {
      const cudaError_t pe = cudaDeviceEnablePeerAccess(root->ctx->device, 0);
      if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else cuda_ok(pe, "cudaDeviceEnablePeerAccess (merge inbox)");
    }
    bind_inbox(e, root->inbox, read_inbox_header(e, root->inbox, rank), rank, 2);
  });
}

}  // extern "C"
