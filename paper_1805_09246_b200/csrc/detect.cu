// detect.cu — the per-slide estimate as phases of ONE persistent cooperative
// kernel, and the persistent engine that interleaves it with the packet scan.
//
// run_detection (src/window.cpp:36-78) needs, per completed slice:
//   A  hot SREs per row (Rsra::extract_hot, src/rsra.cpp:45-57) and the
//      inside-window count of every SLEA row (Slea::setting_factor,
//      src/slea.cpp:57-61)                          -> one pass over the state
//   B  candidate reconstruction (reconstruct_candidates,
//      src/reconstruct.cpp:32-151 + ReversibleHashGroup::invert,
//      src/hash.cpp:77-112)                         -> small, latency bound
//   C  the USLE weight of every candidate (Slea::estimate,
//      src/slea.cpp:103-114)                        -> r' x eta' bits each
// Grid = one 512-thread CTA per SM (cooperative launch, every CTA resident);
// the phases are separated by grid barriers on a release/acquire counter.
//
// Phase A streams the whole state (RSRA + SLEA stamps, 63.2 MB at paper
// geometry, L2-resident) as 32-cell words: a warp keeps 16 coalesced 128 B
// loads in flight per iteration and turns each into one `inside` ballot.
// RSRA words give the SRE weights (popcount of eta-bit groups); SLEA words are
// stored as a flat 1-bit-per-cell bitmap (bit = cell index) and counted per
// row. Phase C then reads r' x eta' bits per candidate instead of stamps.
//
// Reconstruction. A partial tuple (he0, .., he_{L-1}) extends with column he
// of row L iff (he & overlap_mask) == ((he_{L-1} ^ he0) >> delta) ^
// (he0 & overlap_mask) — hash.hpp:101-103 rewritten as an equality on masked
// bits. Every CTA inserts the hot columns of rows >= 2 into private
// shared-memory tables keyed by (col & overlap_mask), and all (row-0, row-1)
// pairs are spread over the grid, each growing its tuples depth-first. It
// yields exactly the reference's tuple set per stage; the per-stage counts
// feed the reference's tuple_cap / work_cap decisions (reconstruct.cpp:60-63,
// 97-99, 110-113) afterwards, in its own brute-force units.
//
// The last CTA to finish writes the result record and the first candidates
// into mapped pinned host memory; the host forms the doubles.
#include <algorithm>

#include "scan_device.cuh"
#include "srlg_internal.cuh"

namespace srlg {
namespace dev {
namespace {

constexpr int kThreads = kDetectThreads;  // 128 registers per thread: phase A keeps 4 x 16 B loads in flight unspilled

// spin reads: relaxed (an acquire load invalidates the SM's L1 on every poll),
// followed by one acquire fence once the condition holds
__device__ __forceinline__ uint32_t ld_relaxed(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acquire() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// CTA 0's view of the phase boundaries (diagnostics: srlg_detect_phase_ns)
__device__ __forceinline__ void stamp_phase(const DetectParams& P, DetectScratch* S, int i) {
  if (P.grank == 0 && threadIdx.x == 0) S->phase_ns[i] = globaltimer();
}

// per-CTA op timestamps (diagnostics): 0 op start, 1 A done, 2 barrier 1
// passed, 3 B done, 4 barrier 2 passed, 5 C done, 6 epilogue done, 7 op end,
// 8 record assembled, 9 host copies issued, 10 scratch reset, 11 `last` known,
// 12 entry barrier passed (engine detect ops), 13 unused, phase B: 14 counts
// read, 15 lists + tables built, 16 DFS done, 17 inversion done, 18 USLE done
constexpr int kCtaT = 21;

__device__ __forceinline__ void publish(unsigned* flag, unsigned v) {
  __threadfence();
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(v) : "memory");
}

__device__ __forceinline__ void stamp_cta(unsigned long long* ct, int i) {
  if (ct && threadIdx.x == 0) ct[i] = globaltimer();
}

// Grid barrier: a monotonically increasing arrival counter (zeroed by the
// host before every launch); CTA thread 0 keeps the running target. The
// release add publishes the CTA's writes (bar.sync orders them before it),
// the acquire poll makes the other CTAs' writes visible. Cross-CTA data is
// read with ld.cg after a barrier, so stale L1 lines never matter. Measured
// 1.3 us per barrier with 148 CTAs (tools/membench.cu) vs 2.6 us for an
// atomic + generation-flag barrier.
// `between` runs on thread 0 after its arrival, before it polls the counter.
struct NoWait {
  __device__ void operator()() const {}
};
template <class F = NoWait>
__device__ __forceinline__ void group_sync(unsigned* ctr, uint32_t group, unsigned& target,
                                           F&& between = NoWait{}) {
  __syncthreads();
  if (threadIdx.x == 0) {
    target += group;
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
    between();
    while (static_cast<int>(ld_relaxed(ctr) - target) < 0) {
    }
    fence_acquire();
  }
  __syncthreads();
}

// ------------------------------------------------------ bounded flag waits
// Flags written by another engine (a peer rank, possibly on another GPU) or
// by a copy stream. A wait that sees no progress for kFlagTimeoutNs traps:
// the launch fails with an error instead of hanging the device when a peer
// or a copy never arrives. The globaltimer is read every 1024 polls, in a
// function kept out of line so the hot kernel body pays no registers for it.
constexpr uint64_t kFlagTimeoutNs = 20ull * 1000 * 1000 * 1000;

__device__ __forceinline__ uint32_t ld_relaxed_sys(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __noinline__ void wait_flag(const unsigned* flag, unsigned v) {
  uint64_t t0 = 0;
  for (uint32_t spins = 1; static_cast<int>(ld_relaxed_sys(flag) - v) < 0; ++spins) {
    if ((spins & 1023) == 0) {
      const uint64_t t = globaltimer();
      if (!t0) {
        t0 = t;
      } else if (t - t0 > kFlagTimeoutNs) {
        __trap();
      }
    }
  }
  fence_sys();
}

// a word the host writes into mapped pinned memory (the candidate arena's
// release offset): the host frees ring space as the caller drains the
// batch's reports, so this wait is bounded generously
constexpr uint64_t kHostTimeoutNs = 120ull * 1000 * 1000 * 1000;

__device__ __noinline__ void wait_host_u64(const unsigned long long* word, uint64_t v) {
  uint64_t t0 = 0;
  for (uint32_t spins = 1;; ++spins) {
    unsigned long long cur;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(cur) : "l"(word) : "memory");
    if (cur >= v) break;
    if ((spins & 255) == 0) {
      const uint64_t t = globaltimer();
      if (!t0) t0 = t;
      else if (t - t0 > kHostTimeoutNs) __trap();
    }
  }
  fence_sys();
}

// every thread of the CTA returns once *flag >= v
__device__ __forceinline__ void cta_wait_flag(const unsigned* flag, unsigned v) {
  if (threadIdx.x == 0) wait_flag(flag, v);
  __syncthreads();
}

// ------------------------------------------------------- overlap tables
// entry = (generation << 32) | (col + 1); any other generation reads empty
__device__ __forceinline__ uint32_t table_slot(uint32_t key, uint32_t bits) {
  return (key * 0x9E3779B1u) >> (32 - bits);
}

__device__ __forceinline__ void table_insert(unsigned long long* T, uint32_t bits, uint32_t gen,
                                             uint32_t key, uint32_t col) {
  const unsigned long long e = (static_cast<unsigned long long>(gen) << 32) | (col + 1u);
  const uint32_t mask = (1u << bits) - 1;
  uint32_t i = table_slot(key, bits);
  unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(T + i);
  while (true) {
    if (static_cast<uint32_t>(cur >> 32) != gen) {
      const unsigned long long old = atomicCAS(T + i, cur, e);
      if (old == cur) return;
      cur = old;  // raced: re-examine the same slot
    } else {
      i = (i + 1) & mask;
      cur = *reinterpret_cast<volatile unsigned long long*>(T + i);
    }
  }
}

// ---------------------------------------------------------------- phase A
constexpr uint32_t kBlockWords = 16;  // 32-cell words per warp iteration; lane u < 16 owns word u

// `inside` ballots of 16 consecutive 32-cell words of `cells` (n cells) from
// word w0: 16 coalesced 128 B loads in flight per warp. Lane u receives the
// ballot of word w0 + u.
__device__ __forceinline__ uint32_t block_ballots(const uint32_t* __restrict__ cells, uint64_t n,
                                                  uint64_t w0, uint32_t lo) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t v[kBlockWords];
#pragma unroll
  for (uint32_t u = 0; u < kBlockWords; ++u) {
    const uint64_t c = (w0 + u) * 32 + lane;
    v[u] = c < n ? ld_state(cells + c) : 0u;  // stamp 0 = never set, never inside
  }
  uint32_t mine = 0;
#pragma unroll
  for (uint32_t u = 0; u < kBlockWords; ++u) {
    const uint32_t m = __ballot_sync(0xFFFFFFFFu, v[u] > lo);
    if (lane == u) mine = m;
  }
  return mine;
}

// RSRA SREs whose eta cells fit 32-cell words without straddling a row
__device__ __forceinline__ bool rsra_words_ok(const RsraDev& rs) {
  return (rs.eta & (rs.eta - 1)) == 0 && rs.eta <= 32 && ((static_cast<uint64_t>(rs.eta) << rs.q) % 32) == 0;
}

__device__ __forceinline__ void append_hot(const DetectParams& P, DetectScratch* S, uint64_t sre) {
  const uint64_t cols = 1ull << P.rs.q;
  const uint32_t row = static_cast<uint32_t>(sre >> P.rs.q);
  const unsigned long long i = atomicAdd(&S->hot_counts[row], 1ull);
  P.hot_cols[row * cols + i] = static_cast<uint32_t>(sre & (cols - 1));
}

// A1 fallback for SRE sizes that do not tile 32-cell words: thread per SRE
__device__ __noinline__ void phase_rsra_generic(const DetectParams& P, DetectScratch* S, uint32_t rs_lo) {
  const uint64_t gtid = static_cast<uint64_t>(P.grank) * blockDim.x + threadIdx.x;
  const uint64_t gsize = static_cast<uint64_t>(P.gsize) * blockDim.x;
  const RsraDev& rs = P.rs;
  const uint64_t sres = static_cast<uint64_t>(rs.r) << rs.q;
  for (uint64_t s = gtid; s < sres; s += gsize) {
    const uint32_t* p = rs.cells + s * rs.eta;
    uint32_t w = 0;
    for (uint32_t z = 0; z < rs.eta; ++z) w += __ldcg(p + z) > rs_lo;
    if (w >= P.hot_min) append_hot(P, S, s);
  }
}

// one 32 B sector (8 stamps) per lane: a single 256-bit load (two 16 B loads
// bypassing L1 would fetch every sector twice from L2)
__device__ __forceinline__ void ld_state8(const uint32_t* p, uint4& a, uint4& b) {
  asm volatile("ld.global.cg.L2::cache_hint.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8], %9;"
               : "=r"(a.x), "=r"(a.y), "=r"(a.z), "=r"(a.w), "=r"(b.x), "=r"(b.y), "=r"(b.z),
                 "=r"(b.w)
               : "l"(p), "l"(policy_evict_last()));
}

__device__ __forceinline__ uint32_t inside8(uint4 a, uint4 b, uint32_t lo) {
  return (a.x > lo) | (a.y > lo) << 1 | (a.z > lo) << 2 | (a.w > lo) << 3 | (b.x > lo) << 4 |
         (b.y > lo) << 5 | (b.z > lo) << 6 | (b.w > lo) << 7;
}

// the smallest stamp of a sector's inside cells (0xFFFFFFFF: none inside)
__device__ __forceinline__ uint32_t inside_min8(uint4 a, uint4 b, uint32_t lo) {
  const auto f = [lo](uint32_t v) { return v > lo ? v : 0xFFFFFFFFu; };
  return min(min(min(f(a.x), f(a.y)), min(f(a.z), f(a.w))),
             min(min(f(b.x), f(b.y)), min(f(b.z), f(b.w))));
}

// min over the 8 lanes of an aligned lane octet (the 8 sectors of a block)
__device__ __forceinline__ uint32_t octet_min(uint32_t v) {
  v = min(v, __shfl_xor_sync(0xFFFFFFFFu, v, 1));
  v = min(v, __shfl_xor_sync(0xFFFFFFFFu, v, 2));
  return min(v, __shfl_xor_sync(0xFFFFFFFFu, v, 4));
}

// Sector path of phase A: every lane loads whole 32 B sectors (8 stamps),
// kSecUnroll sectors in flight, and works on them alone — an SRE of
// eta = 8 is exactly one sector, and 8 SLEA cells are one byte of the flat
// inside bitmap — so the pass needs no cross-lane traffic. (A 16 B-per-lane
// version that formed bitmap words and row sums with shuffles / redux ran
// 3x slower: the cross-lane unit, not memory, was the bound.)
// Requires eta in {1, 2, 4} or eta = 8 * 2^j <= 256, 8 | row_len.
__device__ __forceinline__ bool phase_a_sector_ok(const RsraDev& rs, const SleaDev& le) {
  const bool small = rs.eta == 1 || rs.eta == 2 || rs.eta == 4;
  const uint32_t g = rs.eta / 8;  // lanes per SRE
  const bool big = rs.eta % 8 == 0 && g <= 32 && (g & (g - 1)) == 0;
  return (small || big) && le.row_len % 8 == 0;
}

// 6 sectors in flight per lane: 2 / 4 / 6 / 8 measured -8 % / base / +1.2 %
// / -0.8 % on C2
constexpr int kSecUnrollDefault = 6;

// steady-state scans: equal contiguous slice shares per stream CTA (0: grid
// stride over the stream group; kept for A/B builds)
// scans of at least kDynScanMin pairs per stream CTA claim chunks of
// kDynScanChunk pairs dynamically (a multiple of kThreads)
constexpr uint64_t kDynScanMin = 8192;
// (C4 A/B: 3072 -> 1536 pairs = one group of 3 per thread: 121.4 -> 120.5 ms,
// latency 88 -> 84 us; 1024: +0.3 % time, 79 us; 512: +3 %; groups of 2 or 6
// pairs per thread: no better)
constexpr uint64_t kDynScanChunk = 3 * 512;

#ifndef SRLG_SCAN_GROUPED
#define SRLG_SCAN_GROUPED 1
#endif

// init (kOpInit, eta = 8): also (re)build the live tracking structures
// (IncDev): per block the smallest inside stamp, the live bitmap and the live
// hot bits. A warp's lanes hold consecutive sectors, so a block is an aligned
// lane octet.
// RS / LE: 0 skip the sketch, 1 sweep it, 2 sweep it and (re)build its live
// tracking structures (RS 2 needs eta = 8)
// The pass runs on threads [t0, t0 + nt) of every CTA of the group (t0 and nt
// multiples of 32).
template <int RS, int LE, int kSecUnroll = kSecUnrollDefault>
__device__ void phase_a_sector(const DetectParams& P, DetectScratch* S, uint32_t rs_lo,
                               uint32_t le_lo, unsigned* row_cnt, uint32_t t0 = 0,
                               uint32_t nt = kThreads) {
  const RsraDev& rs = P.rs;
  const SleaDev& le = P.le;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gtid = static_cast<uint64_t>(P.grank) * nt + (threadIdx.x - t0);
  const uint64_t gsize = static_cast<uint64_t>(P.gsize) * nt;
  // ---- RSRA: sector v holds cells [8v, 8v+8)
  if constexpr (RS > 0) {
    const uint64_t cols = 1ull << rs.q;
    const uint64_t ns = ((static_cast<uint64_t>(rs.r) << rs.q) * rs.eta) / 8;
    const uint32_t g = rs.eta >= 8 ? rs.eta / 8 : 1;    // lanes per SRE
    const uint32_t lg = __ffs(g) - 1;
    const uint32_t per = rs.eta >= 8 ? 1 : 8 / rs.eta;  // SREs per sector
    const uint32_t lper = __ffs(per) - 1;
    const uint32_t emask = rs.eta >= 8 ? 0xFFu : (1u << rs.eta) - 1;
    const uint64_t nsw = (ns + 31) & ~uint64_t(31);  // warp-uniform trip count
    for (uint64_t v = gtid; v < nsw; v += kSecUnroll * gsize) {
      uint4 xa[kSecUnroll], xb[kSecUnroll];
#pragma unroll
      for (int u = 0; u < kSecUnroll; ++u) {  // out-of-range lanes re-read the last sector
        const uint64_t vu = v + u * gsize;
        const bool in = vu < ns;
        xa[u] = xb[u] = make_uint4(0, 0, 0, 0);
        if (in) ld_state8(rs.cells + 8 * vu, xa[u], xb[u]);
      }
#pragma unroll
      for (int u = 0; u < kSecUnroll; ++u) {
        const uint64_t vu = v + u * gsize;
        if (vu - lane >= nsw) break;  // warp-uniform
        const uint32_t m = vu < ns ? inside8(xa[u], xb[u], rs_lo) : 0u;
        if constexpr (RS == 2) {  // eta = 8: sector = SRE, lane octet = block
          const uint32_t hot =
              __ballot_sync(0xFFFFFFFFu, vu < ns && static_cast<uint32_t>(__popc(m)) >= P.hot_min);
          const uint32_t mn = octet_min(vu < ns ? inside_min8(xa[u], xb[u], rs_lo) : 0xFFFFFFFFu);
          if ((lane & 7) == 0 && vu < ns) {
            P.inc.live_hot[vu >> 3] = static_cast<uint8_t>(hot >> lane);
            P.inc.rs_smin[vu >> 3] = mn;
          }
        }
        if (g > 1) {  // eta >= 16: the SRE spans g lanes
          uint32_t w = __popc(m);
          for (uint32_t o = 1; o < g; o <<= 1) w += __shfl_xor_sync(0xFFFFFFFFu, w, o);
          if ((lane & (g - 1)) == 0 && vu < ns && w >= P.hot_min) {
            const uint64_t sre = vu >> lg;
            const uint32_t row = static_cast<uint32_t>(sre >> rs.q);
            const unsigned long long i = atomicAdd(&S->hot_counts[row], 1ull);
            P.hot_cols[row * cols + i] = static_cast<uint32_t>(sre & (cols - 1));
          }
        } else if (vu < ns) {
          for (uint32_t j = 0; j < per; ++j) {
            if (static_cast<uint32_t>(__popc((m >> (j * rs.eta)) & emask)) >= P.hot_min) {
              const uint64_t sre = (vu << lper) + j;
              const uint32_t row = static_cast<uint32_t>(sre >> rs.q);
              const unsigned long long i = atomicAdd(&S->hot_counts[row], 1ull);
              P.hot_cols[row * cols + i] = static_cast<uint32_t>(sre & (cols - 1));
            }
          }
        }
      }
    }
  }
  // ---- SLEA: per-row inside counts + the flat bitmap, one byte per sector.
  // Each lane's sector index only grows, so it tracks its row with compares
  // and flushes its count into the CTA's shared row counter on a row change.
  if constexpr (LE > 0) {
    constexpr bool init = LE == 2;
    const uint64_t ns_row = le.row_len / 8;
    const uint64_t ns = ns_row * le.r;
    uint8_t* bytes = reinterpret_cast<uint8_t*>(P.le_bits);
    uint32_t row = 0, cnt = 0;
    uint64_t bnd = ns_row;
    // init: the lane octets' shuffles need whole warps (warp-uniform trip count)
    const uint64_t nsw = init ? (ns + 31) & ~uint64_t(31) : ns;
    for (uint64_t v = gtid; v < nsw; v += kSecUnroll * gsize) {
      uint4 xa[kSecUnroll], xb[kSecUnroll];
#pragma unroll
      for (int u = 0; u < kSecUnroll; ++u) {
        const uint64_t vu = v + u * gsize;
        const bool in = vu < ns;
        xa[u] = xb[u] = make_uint4(0, 0, 0, 0);
        if (in) ld_state8(le.cells + 8 * vu, xa[u], xb[u]);
      }
#pragma unroll
      for (int u = 0; u < kSecUnroll; ++u) {
        const uint64_t vu = v + u * gsize;
        if constexpr (init) {
          if (vu - lane >= ns) break;  // warp-uniform
          const bool in = vu < ns;
          const uint32_t m0 = in ? inside8(xa[u], xb[u], le_lo) : 0u;
          const uint32_t mn = octet_min(in ? inside_min8(xa[u], xb[u], le_lo) : 0xFFFFFFFFu);
          if (in) reinterpret_cast<uint8_t*>(P.inc.live_bits)[vu] = static_cast<uint8_t>(m0);
          if ((lane & 7) == 0 && in) P.inc.le_smin[vu >> 3] = mn;
          if (!in) continue;  // every lane reaches the next u's warp-uniform check
        } else if (vu >= ns) {
          break;
        }
        const uint32_t m = inside8(xa[u], xb[u], le_lo);
        bytes[vu] = static_cast<uint8_t>(m);
        while (vu >= bnd) {
          if (cnt) atomicAdd(&row_cnt[row], cnt);
          cnt = 0;
          ++row;
          bnd += ns_row;
        }
        cnt += __popc(m);
      }
    }
    if (cnt) atomicAdd(&row_cnt[row], cnt);
  }
}

// Phase A: one streaming pass over RSRA and SLEA. Hot SRE columns are
// appended per row (unordered; the reconstruction sorts its output), SLEA
// inside counts accumulate per CTA in `row_cnt` (shared), and the SLEA inside
// bitmap is written.
__device__ void phase_a(const DetectParams& P, DetectScratch* S, uint32_t rs_lo, uint32_t le_lo,
                        unsigned* row_cnt, bool init, bool init_le) {
  if (phase_a_sector_ok(P.rs, P.le)) {
    if (!init || P.rs.eta != 8)
      phase_a_sector<1, 1>(P, S, rs_lo, le_lo, row_cnt);
    else if (init_le)
      phase_a_sector<2, 2>(P, S, rs_lo, le_lo, row_cnt);
    else
      phase_a_sector<2, 1>(P, S, rs_lo, le_lo, row_cnt);
    return;
  }
  const RsraDev& rs = P.rs;
  const SleaDev& le = P.le;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gwarp = (static_cast<uint64_t>(P.grank) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(P.gsize) * blockDim.x) >> 5;
  const bool rs_words = rsra_words_ok(rs);
  if (!rs_words) phase_rsra_generic(P, S, rs_lo);
  const uint64_t rs_cells = (static_cast<uint64_t>(rs.r) << rs.q) * rs.eta;
  const uint64_t rs_nw = rs_words ? rs_cells / 32 : 0;
  const uint64_t rs_blocks = (rs_nw + kBlockWords - 1) / kBlockWords;
  const uint64_t le_cells = le.row_len * le.r;
  const uint64_t le_nw = (le_cells + 31) / 32;
  const uint64_t le_blocks = (le_nw + kBlockWords - 1) / kBlockWords;
  const uint32_t per_word = rs_words ? 32 / rs.eta : 0;
  const uint32_t emask = rs.eta >= 32 ? 0xFFFFFFFFu : (1u << rs.eta) - 1;
  for (uint64_t blk = gwarp; blk < rs_blocks + le_blocks; blk += nwarps) {
    if (blk < rs_blocks) {
      const uint64_t w0 = blk * kBlockWords;
      const uint32_t mine = block_ballots(rs.cells, rs_cells, w0, rs_lo);
      const uint64_t w = w0 + lane;
      if (lane < kBlockWords && w < rs_nw && mine) {
        for (uint32_t j = 0; j < per_word; ++j)
          if (static_cast<uint32_t>(__popc((mine >> (j * rs.eta)) & emask)) >= P.hot_min)
            append_hot(P, S, w * per_word + j);
      } else if (lane < kBlockWords && w < rs_nw && P.hot_min == 0) {
        for (uint32_t j = 0; j < per_word; ++j) append_hot(P, S, w * per_word + j);
      }
    } else {
      const uint64_t w0 = (blk - rs_blocks) * kBlockWords;
      const uint32_t mine = block_ballots(le.cells, le_cells, w0, le_lo);
      const uint64_t w = w0 + lane;
      const bool own = lane < kBlockWords && w < le_nw;
      if (own) P.le_bits[w] = mine;
      // row of the word's first cell; a word may straddle into the next row
      uint32_t row = 0, c0 = 0, c1 = 0;
      bool split = false;
      if (own) {
        const uint64_t cell = w * 32;
        row = static_cast<uint32_t>(cell / le.row_len);
        const uint64_t rem = (static_cast<uint64_t>(row) + 1) * le.row_len - cell;
        if (rem >= 32) {
          c0 = __popc(mine);
        } else {
          split = true;
          c0 = __popc(mine & ((1u << rem) - 1));
          c1 = __popc(mine >> rem);
        }
      }
      const uint32_t row0 = __shfl_sync(0xFFFFFFFFu, row, 0);
      if (__all_sync(0xFFFFFFFFu, !own || (row == row0 && !split))) {
        const uint32_t s = __reduce_add_sync(0xFFFFFFFFu, c0);
        if (lane == 0 && s) atomicAdd(&row_cnt[row0], s);
      } else if (own) {
        if (c0) atomicAdd(&row_cnt[row], c0);
        if (c1 && row + 1 < le.r) atomicAdd(&row_cnt[row + 1], c1);
      }
    }
  }
}

// ------------------------------------------------- incremental phase A
// kOpInc detections (engine): the live structures (IncDev) hold the window of
// the previous detection; blocks whose smallest inside stamp fell to the new
// window's low, and blocks a scan marked (a cell entered), are re-examined —
// at C2 about 2 % of the blocks. Each stream CTA owns a fixed contiguous block
// range (the same in every detection of the launch), so it re-examines,
// compacts its hot bits and copies its bitmap range without grid-wide
// ordering. Requires RSRA eta = 8 and 8 | SLEA row_len (host-checked).
__device__ __forceinline__ void cta_range(uint64_t n, uint32_t g, uint32_t G, uint64_t& a,
                                          uint64_t& b) {
  const uint64_t chunk = ((n + G - 1) / G + 3) & ~uint64_t(3);
  a = min(n, chunk * g);
  b = min(n, a + chunk);
}

// Up to 4 consecutive u32 from x (x % 4 == 0) below n; missing ones = fill
__device__ __forceinline__ uint4 ld_quad(const uint32_t* p, uint64_t x, uint64_t n, uint32_t fill) {
  if (x + 4 <= n) return __ldcg(reinterpret_cast<const uint4*>(p + x));
  uint4 v = make_uint4(fill, fill, fill, fill);
  if (x < n) v.x = __ldcg(p + x);
  if (x + 1 < n) v.y = __ldcg(p + x + 1);
  if (x + 2 < n) v.z = __ldcg(p + x + 2);
  return v;
}

// RSRA block x: hot bits of its 8 SREs and the smallest inside stamp (two
// halves of 4 sectors in flight: 8 would spill the engine kernel)
__device__ void rs_block(const uint32_t* __restrict__ cells, uint32_t hot_min, uint8_t* live_hot,
                         uint32_t* smin, uint64_t x, uint32_t lo) {
  const uint32_t* c = cells + x * kIncBlock;
  uint32_t hot = 0, mn = 0xFFFFFFFFu;
#pragma unroll
  for (int h = 0; h < 8; h += 4) {
    uint4 va[4], vb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) ld_state8(c + 8 * (h + j), va[j], vb[j]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      hot |= static_cast<uint32_t>(static_cast<uint32_t>(__popc(inside8(va[j], vb[j], lo))) >=
                                   hot_min)
             << (h + j);
      mn = min(mn, inside_min8(va[j], vb[j], lo));
    }
  }
  live_hot[x] = static_cast<uint8_t>(hot);
  smin[x] = mn;
}

// SLEA block x (sectors 8x .. 8x + nsec - 1): its 64 live bits, returned with
// the old ones, and the smallest inside stamp (two halves like rs_block)
__device__ __forceinline__ void le_block(const uint32_t* __restrict__ cells, uint32_t nsec,
                                      unsigned long long* live, uint32_t* smin, uint64_t x,
                                      uint32_t lo, unsigned long long* nb_out,
                                      unsigned long long* ob_out) {
  const uint32_t* c = cells + x * kIncBlock;
  const unsigned long long ob = __ldcg(live + x);
  unsigned long long nb = 0;
  uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
  for (int h = 0; h < 8; h += 4) {
    uint4 va[4], vb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      va[j] = vb[j] = make_uint4(0, 0, 0, 0);
      if (h + j < nsec) ld_state8(c + 8 * (h + j), va[j], vb[j]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (h + j >= nsec) break;
      nb |= static_cast<unsigned long long>(inside8(va[j], vb[j], lo)) << (8 * (h + j));
      mn = min(mn, inside_min8(va[j], vb[j], lo));
    }
  }
  if (nb != ob) live[x] = nb;
  smin[x] = mn;
  *nb_out = nb;
  *ob_out = ob;
}

// the row counts of a changed SLEA block
__device__ __forceinline__ void le_block_rows(const SleaDev& le, uint64_t x, uint32_t nsec,
                                              unsigned long long nb, unsigned long long ob,
                                              int* row_delta) {
  if (nb == ob) return;
  const uint64_t ns_row = le.row_len / 8;
  const uint64_t s0 = x * 8;
  const uint32_t r0 = static_cast<uint32_t>(s0 / ns_row);
  const uint64_t bnd = (static_cast<uint64_t>(r0) + 1) * ns_row;  // first sector of row r0 + 1
  if (s0 + nsec <= bnd) {
    atomicAdd(&row_delta[r0], __popcll(nb) - __popcll(ob));
  } else {  // the block straddles two rows
    const unsigned long long lo_mask = (1ull << (8 * (bnd - s0))) - 1;
    atomicAdd(&row_delta[r0], __popcll(nb & lo_mask) - __popcll(ob & lo_mask));
    atomicAdd(&row_delta[r0 + 1], __popcll(nb & ~lo_mask) - __popcll(ob & ~lo_mask));
  }
}

// RSRA incremental pass on the first kRsWarps warps of a stream CTA, while
// the other warps sweep the SLEA (mode 1: the two overlap; the RSRA part is
// a chain of L2 round trips, the sweep is bound by the L2 read rate). Three
// round trips:
//  1. each thread loads up to kRsQuads quads of block minima and the quads'
//     live hot bytes (kept in shared memory), and lists the flagged blocks;
//  2. a lane octet per pair of flagged blocks, one sector (= one SRE at
//     eta 8) per lane and block: hot bits and smallest inside stamp;
//  3. the range's hot bits (shared memory) go to the hot lists.
// Passes are separated by a named barrier of the subset.
constexpr uint32_t kRsWarps = 4;  // 3: same, 6: -3 % on C2 (A/B)
constexpr uint32_t kRsQuads = 2;
constexpr uint32_t kRsFlagCap = 1024;  // flagged blocks listed per CTA (more: sequential path)
constexpr uint32_t kRsHotQuads = 1024; // hot words kept in shared memory per CTA

__device__ __forceinline__ void rs_bar() {
  asm volatile("bar.sync 1, %0;" ::"r"(kRsWarps * 32) : "memory");
}

// live hot bytes of quad x (4 blocks; fewer below b)
__device__ __forceinline__ uint32_t ld_hot_quad(const uint8_t* live_hot, uint64_t x, uint64_t b) {
  if (x + 4 <= b) return __ldcg(reinterpret_cast<const uint32_t*>(live_hot + x));
  uint32_t h = 0;
  for (uint64_t y = x; y < b; ++y) h |= static_cast<uint32_t>(__ldcg(live_hot + y)) << (8 * (y - x));
  return h;
}

// one flagged block by a lane octet (lane & 7 = its sector): the block's hot
// byte and smallest inside stamp
__device__ __forceinline__ void rs_octet_result(uint4 va, uint4 vb, uint32_t lo, uint32_t hot_min,
                                                uint32_t omask, uint32_t lane, uint32_t& byte,
                                                uint32_t& mn) {
  const uint32_t hot =
      __ballot_sync(omask, static_cast<uint32_t>(__popc(inside8(va, vb, lo))) >= hot_min);
  byte = (hot >> (lane & 24)) & 0xFFu;
  mn = inside_min8(va, vb, lo);
  mn = min(mn, __shfl_xor_sync(omask, mn, 1));
  mn = min(mn, __shfl_xor_sync(omask, mn, 2));
  mn = min(mn, __shfl_xor_sync(omask, mn, 4));
}

__device__ void phase_a_rs_warps(const DetectParams& P, DetectScratch* S, uint32_t lo,
                                 uint32_t* flist, unsigned* fcount, uint32_t* hot_s) {
  const IncDev& I = P.inc;
  const uint32_t tid = threadIdx.x, nthr = kRsWarps * 32, lane = tid & 31;
  uint64_t a, b;
  cta_range(I.rs_blocks, P.grank, P.gsize, a, b);
  const uint64_t qr = (b - a + 3) / 4;
  const bool smem_hot = qr <= kRsHotQuads;
  uint8_t* hot_b = reinterpret_cast<uint8_t*>(hot_s);
  for (uint64_t q0 = 0; q0 < qr; q0 += kRsQuads * nthr) {
    uint4 m[kRsQuads];
    uint32_t h[kRsQuads];
#pragma unroll
    for (uint32_t u = 0; u < kRsQuads; ++u) {
      const uint64_t q = q0 + u * nthr + tid;
      m[u] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
      h[u] = 0;
      if (q < qr) {
        m[u] = ld_quad(I.rs_smin, a + 4 * q, b, 0xFFFFFFFFu);
        if (smem_hot) h[u] = ld_hot_quad(I.live_hot, a + 4 * q, b);
      }
    }
#pragma unroll
    for (uint32_t u = 0; u < kRsQuads; ++u) {
      const uint64_t q = q0 + u * nthr + tid;
      if (q >= qr) continue;
      if (smem_hot) hot_s[q] = h[u];
      const uint64_t x = a + 4 * q;
      const uint32_t v[4] = {m[u].x, m[u].y, m[u].z, m[u].w};
#pragma unroll
      for (uint32_t j = 0; j < 4; ++j) {
        if (v[j] > lo) continue;
        const unsigned k = atomicAdd(fcount, 1u);
        if (k < kRsFlagCap) {
          flist[k] = static_cast<uint32_t>(x + j);
        } else {  // more flagged blocks than listed: this thread does it alone
          rs_block(P.rs.cells, P.hot_min, I.live_hot, I.rs_smin, x + j, lo);
          if (smem_hot) hot_b[x + j - a] = __ldcg(I.live_hot + x + j);
        }
      }
    }
  }
  rs_bar();
  const uint32_t n = min(*fcount, kRsFlagCap);
  if (P.diag && I.stats && tid == 0 && *fcount)
    atomicAdd(I.stats, static_cast<unsigned long long>(*fcount));
  const uint32_t omask = 0xFFu << (lane & 24);  // this lane's octet
  const uint32_t octets = nthr / 8;
  for (uint32_t f = tid >> 3; f < n; f += 2 * octets) {  // two blocks per octet in flight
    const uint32_t f2 = f + octets;
    const uint64_t x1 = flist[f], x2 = f2 < n ? flist[f2] : x1;
    uint4 va1, vb1, va2, vb2;
    ld_state8(P.rs.cells + x1 * kIncBlock + 8 * (lane & 7), va1, vb1);
    ld_state8(P.rs.cells + x2 * kIncBlock + 8 * (lane & 7), va2, vb2);
    uint32_t by1, mn1, by2, mn2;
    rs_octet_result(va1, vb1, lo, P.hot_min, omask, lane, by1, mn1);
    rs_octet_result(va2, vb2, lo, P.hot_min, omask, lane, by2, mn2);
    if ((lane & 7) == 0) {
      I.live_hot[x1] = static_cast<uint8_t>(by1);
      I.rs_smin[x1] = mn1;
      if (smem_hot) hot_b[x1 - a] = static_cast<uint8_t>(by1);
      if (f2 < n) {
        I.live_hot[x2] = static_cast<uint8_t>(by2);
        I.rs_smin[x2] = mn2;
        if (smem_hot) hot_b[x2 - a] = static_cast<uint8_t>(by2);
      }
    }
  }
  rs_bar();
  if (tid == 0) *fcount = 0;  // the next use is several CTA barriers away
  for (uint64_t q = tid; q < qr; q += nthr) {
    uint32_t h = smem_hot ? hot_s[q] : ld_hot_quad(I.live_hot, a + 4 * q, b);
    const uint64_t x = a + 4 * q;
    while (h) {
      const uint32_t j = __ffs(h) - 1;
      h &= h - 1;
      append_hot(P, S, x * 8 + j);
    }
  }
}

// Passes over the CTA's ranges: (1) the threads load the quads of block
// minima (RSRA quads, then SLEA quads), kIncQuads per thread in flight, and
// list the flagged blocks in shared memory; (2) every listed block is
// re-examined by one thread (a thread used to walk its quads one dependent
// round trip after another, and re-examine its flagged blocks in between);
// (3) after a CTA barrier, every thread takes a quad again: RSRA live hot
// bits into the hot lists, SLEA live words into the detection's bitmap.
__device__ void phase_a_inc(const DetectParams& P, DetectScratch* S, uint32_t rs_lo, uint32_t le_lo,
                            int* row_delta, bool le_inc, uint32_t det, unsigned* logn,
                            uint32_t* sm_flags, unsigned* nflag) {
  const IncDev& I = P.inc;
  // this detection's log of changed live words (SLEA tracked)
  const uint32_t slot = det % kLeLogSlots;
  const uint64_t lbase = (static_cast<uint64_t>(slot) * kLeLogCtas + P.grank) * kLeLogCap;
  uint64_t a, b, la = 0, lb = 0;
  cta_range(I.rs_blocks, P.grank, P.gsize, a, b);
  if (le_inc) cta_range(I.le_blocks, P.grank, P.gsize, la, lb);
  const uint64_t qr = (b - a + 3) / 4, ql = (lb - la + 3) / 4;
  // (1) block minima, kIncQuads quads per thread in flight: the flagged blocks
  // go to a shared list (SLEA entries tagged by the top bit); (2) one thread
  // per listed block. Past the list's capacity a thread does its block alone.
  constexpr uint32_t kIncQuads = 4;
  constexpr uint32_t kLeTag = 0x80000000u;
  uint32_t* flist = sm_flags;
  const auto do_block = [&](bool rs, uint64_t xb) {
    if (rs) {
      rs_block(P.rs.cells, P.hot_min, I.live_hot, I.rs_smin, xb, rs_lo);
      return;
    }
    const uint64_t ns = P.le.row_len / 8 * P.le.r;  // sectors
    const uint64_t s0 = xb * 8;
    const uint32_t nsec = ns - s0 < 8 ? static_cast<uint32_t>(ns - s0) : 8u;
    unsigned long long nb, ob;
    le_block(P.le.cells, nsec, reinterpret_cast<unsigned long long*>(I.live_bits), I.le_smin, xb,
             le_lo, &nb, &ob);
    le_block_rows(P.le, xb, nsec, nb, ob, row_delta);
    if (nb != ob) {
      const unsigned k = atomicAdd(logn, 1u);
      if (k < kLeLogCap) {
        I.le_log_idx[lbase + k] = static_cast<uint32_t>(xb);
        I.le_log_val[lbase + k] = nb;
      }
    }
  };
  for (uint64_t q0 = 0; q0 < qr + ql; q0 += kIncQuads * blockDim.x) {
    uint4 m[kIncQuads];
#pragma unroll
    for (uint32_t u = 0; u < kIncQuads; ++u) {
      const uint64_t q = q0 + u * blockDim.x + threadIdx.x;
      m[u] = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
      if (q < qr)
        m[u] = ld_quad(I.rs_smin, a + 4 * q, b, 0xFFFFFFFFu);
      else if (q < qr + ql)
        m[u] = ld_quad(I.le_smin, la + 4 * (q - qr), lb, 0xFFFFFFFFu);
    }
#pragma unroll
    for (uint32_t u = 0; u < kIncQuads; ++u) {
      const uint64_t q = q0 + u * blockDim.x + threadIdx.x;
      if (q >= qr + ql) continue;
      const bool rs = q < qr;
      const uint64_t x = rs ? a + 4 * q : la + 4 * (q - qr);
      const uint32_t lo = rs ? rs_lo : le_lo;
      const uint32_t f = (m[u].x <= lo) | (m[u].y <= lo) << 1 | (m[u].z <= lo) << 2 | (m[u].w <= lo) << 3;
      if (!f) continue;
      if (P.diag && I.stats) atomicAdd(I.stats + (rs ? 0 : 1), static_cast<unsigned long long>(__popc(f)));
      for (uint32_t j = 0; j < 4; ++j) {
        if (!((f >> j) & 1)) continue;
        const unsigned k = atomicAdd(nflag, 1u);
        if (k < kRsFlagCap)
          flist[k] = static_cast<uint32_t>(x + j) | (rs ? 0u : kLeTag);
        else
          do_block(rs, x + j);
      }
    }
  }
  __syncthreads();
  const uint32_t nf = min(*nflag, kRsFlagCap);
  for (uint32_t k = threadIdx.x; k < nf; k += blockDim.x) {
    const uint32_t v = flist[k];
    do_block(!(v & kLeTag), v & ~kLeTag);
  }
  __syncthreads();
  if (threadIdx.x == 0) *nflag = 0;
  __syncthreads();  // this CTA's live hot bits and bitmap words are final
  // The detection's bitmap (buffer set det % n_sets) held the live bitmap of
  // detection det - n_sets: replaying the logs of the n_sets detections
  // since brings it up to date. A full copy for the launch's first n_sets
  // detections and when one of those logs overflowed.
  __shared__ bool full_copy;
  if (le_inc && threadIdx.x == 0) {
    const unsigned n = *logn;
    I.le_log_n[slot * kLeLogCtas + P.grank] = n > kLeLogCap ? kLeLogCap + 1 : n;
    *logn = 0;
    bool full = det < P.n_sets;
    for (uint32_t j = 1; !full && j < P.n_sets; ++j)
      full = __ldcg(&I.le_log_n[((det - j) % kLeLogSlots) * kLeLogCtas + P.grank]) > kLeLogCap;
    full_copy = full || n > kLeLogCap;
  }
  __syncthreads();
  const uint64_t qcopy = le_inc && full_copy ? ql : 0;
  const unsigned long long* live = reinterpret_cast<const unsigned long long*>(I.live_bits);
  unsigned long long* out = reinterpret_cast<unsigned long long*>(P.le_bits);
  if (le_inc && !full_copy) {
    for (uint32_t j = P.n_sets; j-- > 0;) {  // oldest log first: later values win
      const uint32_t sl = (det - j) % kLeLogSlots;
      const unsigned n = __ldcg(&I.le_log_n[sl * kLeLogCtas + P.grank]);
      const uint64_t b0 = (static_cast<uint64_t>(sl) * kLeLogCtas + P.grank) * kLeLogCap;
      for (uint32_t k = threadIdx.x; k < n; k += blockDim.x)
        out[__ldcg(I.le_log_idx + b0 + k)] = __ldcg(I.le_log_val + b0 + k);
      __syncthreads();
    }
  }
  for (uint64_t q = threadIdx.x; q < qr + qcopy; q += blockDim.x) {
    if (q < qr) {  // hot SRE columns of 4 blocks, appended per row like the full pass
      const uint64_t x = a + 4 * q;
      uint32_t h;
      if (x + 4 <= b) {
        h = __ldcg(reinterpret_cast<const uint32_t*>(I.live_hot + x));
      } else {
        h = 0;
        for (uint64_t y = x; y < b; ++y) h |= static_cast<uint32_t>(__ldcg(I.live_hot + y)) << (8 * (y - x));
      }
      while (h) {
        const uint32_t j = __ffs(h) - 1;
        h &= h - 1;
        append_hot(P, S, x * 8 + j);
      }
    } else {  // 4 blocks = 32 B of the bitmap
      const uint64_t x = la + 4 * (q - qr);
      if (x + 4 <= lb) {
        const uint4 u = __ldcg(reinterpret_cast<const uint4*>(live + x));
        const uint4 v = __ldcg(reinterpret_cast<const uint4*>(live + x + 2));
        *reinterpret_cast<uint4*>(out + x) = u;
        *reinterpret_cast<uint4*>(out + x + 2) = v;
      } else {
        for (uint64_t y = x; y < lb; ++y) out[y] = __ldcg(live + y);
      }
    }
  }
}

// ---------------------------------------------------------------- phase B

// Where inverted candidates go: the global candidate array (n_cand order) and
// the finding CTA's shared list, whose USLE weights the CTA computes right
// away from the inside bitmap (complete since barrier 1). Candidates beyond
// the shared list are left to the publishing CTA.
constexpr uint32_t kCandCta = 16;

struct CandSink {
  uint2* cs;        // shared: {aip, global index}
  unsigned* ncs;    // shared count
  uint32_t* left;   // global: indices left to the last CTA
  unsigned* left_n;
};

__device__ __forceinline__ void put_candidate(const DetectParams& P, ReconCounters* C,
                                              const CandSink& k, uint32_t cand) {
  const unsigned long long idx = atomicAdd(&C->n_cand, 1ull);
  if (idx >= P.cand_cap) {
    C->truncated = 1;
    return;
  }
  P.cands[idx] = Candidate{cand, 0};
  const unsigned j = atomicAdd(k.ncs, 1u);
  if (j < kCandCta) {
    k.cs[j] = make_uint2(cand, static_cast<uint32_t>(idx));
  } else {
    const unsigned l = atomicAdd(k.left_n, 1u);
    k.left[l] = static_cast<uint32_t>(idx);
  }
}

// invert one complete tuple (ReversibleHashGroup::invert, hash.cpp:77-112):
// assignments v = v0, v0 + vstep, ... of the uncovered address bits (a warp
// splits them across lanes)
__device__ __noinline__ void invert_tuple(const DetectParams& P, ReconCounters* C, const CandSink& k,
                             const uint32_t* cols, uint64_t v0 = 0, uint64_t vstep = 1) {
  const GroupDev& g = P.g;
  const uint32_t c0 = cols[0];
  uint32_t prev = (cols[1] ^ c0) & g.col_mask;
  uint64_t known = static_cast<uint64_t>(prev) << g.delta;
  for (uint32_t i = 2; i < g.r; ++i) {
    const uint32_t wv = (cols[i] ^ c0) & g.col_mask;
    if ((prev >> g.delta) != (wv & g.overlap_mask)) return;  // consistent by construction
    const uint32_t sh = i * g.delta;
    if (sh < 64) known |= static_cast<uint64_t>(wv) << sh;
    prev = wv;
  }
  const uint32_t assembled = static_cast<uint32_t>(known) & ~g.uncovered;
  for (uint64_t v = v0; v < (1ull << g.n_free); v += vstep) {
    uint32_t cand = assembled;
    for (uint32_t b = 0; b < g.n_free; ++b)
      if (v & (1ull << b)) cand |= 1u << g.free_bits[b];
    const uint32_t f0 = static_cast<uint32_t>(seeded(g.h0, cand)) & g.col_mask;
    if (f0 != c0) continue;
    bool match = true;
    for (uint32_t i = 1; i < g.r && match; ++i) {
      const uint32_t sh = i * g.delta;
      match = (((sh >= 32 ? 0u : cand >> sh) ^ f0) & g.col_mask) == cols[i];
    }
    if (match) put_candidate(P, C, k, cand);
  }
}

// Overlap tables for rows 2..r-1. Common case (few hot columns): every CTA
// builds a private copy in shared memory, u32 entries = col + 1 (0 = empty),
// so the depth-first lookups never leave the SM. Otherwise one copy in
// global memory, u64 entries tagged with the launch generation.
// 4096 u32 entries (16 KB): rows 2..r-1 of the paper geometry need ~768 at a
// typical slide; more hot columns fall back to the global tables. Kept small
// so the detect kernel and the scan share one L1/shared carveout (a carveout
// switch between the two launches costs several microseconds per slide).
// Entries are u64 = (detection generation << 32) | (col + 1), in shared and
// in global memory alike, so a table never needs clearing between
// detections (the shared copy is zeroed once per launch).
constexpr uint32_t kSmemTable = 4096;
// the hot lists themselves are copied into shared memory too when they fit
// (one L2 round trip per CTA instead of one per seed pair)
constexpr uint32_t kSmemLists = 4096;
constexpr size_t kDynSmem = kSmemTable * sizeof(unsigned long long) + kSmemLists * sizeof(uint32_t);

struct Tables {
  bool smem;
  const unsigned long long* s;      // shared-memory tables
  const uint32_t* lists;            // shared copies of the hot lists (or null)
  uint32_t loff[kMaxRows];          // row offsets in `lists`
  uint32_t bits[kMaxRows];          // per row (smem) / common (global)
  uint32_t off[kMaxRows];           // smem row offsets
  const unsigned long long* gtab;   // global tables
  uint64_t gstride;
  uint32_t gen;
};

// smallest b >= 5 with 2^b >= 2n (load factor <= 1/2)
__device__ __forceinline__ uint32_t smem_bits(uint64_t n) {
  const uint32_t b = n <= 16 ? 5u : 64u - __clzll(2 * n - 1);
  return b < 5 ? 5u : b;
}

// probe row L from position *slot for the next column with masked key;
// returns col + 1, or 0 when the probe sequence ends
__device__ __forceinline__ uint32_t table_next(const Tables& t, uint32_t L, uint32_t key,
                                               uint32_t ov, uint32_t* slot) {
  const uint32_t mask = (1u << t.bits[L]) - 1;
  while (true) {
    const unsigned long long g =
        t.smem ? t.s[t.off[L] + *slot] : __ldcg(t.gtab + (L - 2) * t.gstride + *slot);
    const uint32_t e = static_cast<uint32_t>(g >> 32) == t.gen ? static_cast<uint32_t>(g) : 0u;
    if (e == 0) return 0;
    *slot = (*slot + 1) & mask;
    if (((e - 1) & ov) == key) return e;
  }
}

// Depth-first growth of every seed pair (rows 0, 1) through rows 2..r-1;
// pairs are spread over all CTAs. Stage counts are accumulated per thread
// and published with one reduction per level at the end.
constexpr unsigned kQueue = 256;      // complete tuples queued per CTA
constexpr uint32_t kQueueWidth = 8;   // queue slots hold tuples of r <= 8 rows

struct DfsCtx {
  const DetectParams* P;
  ReconCounters* C;
  CandSink k;
  const Tables* t;
  unsigned* abort;
  unsigned* cta_stage;
  uint32_t* q_s;
  unsigned* q_n;
  uint32_t m0;
};

// this thread's region of the reconstruction scratch (DetectParams::dfs_scratch)
__device__ __forceinline__ uint32_t* thread_scratch(const DetectParams& P) {
  return P.dfs_scratch + (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 3 * P.dfs_rows;
}

// complete tuple: queue it for a warp-parallel inversion; past the CTA's
// queue, the thread inverts it from its scratch region (a register tuple
// whose address is taken would live in the kernel's stack frame)
template <int R>
__device__ __forceinline__ void emit_tuple(const DfsCtx& d, const uint32_t (&tup)[R]) {
  const unsigned qi = atomicAdd(d.q_n, 1u);
  if (qi < kQueue) {
#pragma unroll
    for (int x = 0; x < R; ++x) d.q_s[qi * kQueueWidth + x] = tup[x];
  } else {
    uint32_t* ts = thread_scratch(*d.P);
#pragma unroll
    for (int x = 0; x < R; ++x) ts[x] = tup[x];
    invert_tuple(*d.P, d.C, d.k, ts);
  }
}

// compile-time depth: the tuple stays in registers (a dynamically indexed
// array would live in local memory, which spills past the L1 left beside the
// shared-memory tables)
// Stage counts accumulate in registers (cnt[L + 1] = tuples alive after row
// L) and reach the CTA counters in batches of kStageBatch: per-extension
// shared atomics on one address serialised whole warps.
constexpr uint32_t kStageBatch = 64;
constexpr uint32_t kAbortPoll = 16;  // seed pairs between two reads of the global abort flag

template <int L>
__device__ __forceinline__ void stage_flush(const DfsCtx& d, uint32_t& c) {
  // a CTA-local count above tuple_cap proves the global one is: the
  // reference overflows, so everyone may stop
  if (static_cast<uint64_t>(atomicAdd(&d.cta_stage[L + 1], c)) + c > d.P->tuple_cap)
    atomicExch(d.abort, 1u);
  c = 0;
}

// The tables' per-level bases, masks and the group constants, held in
// registers for the whole walk: read through the shared Tables block on
// every probe, they were reloaded each time (the walk's shared-memory stores
// may alias them), a dependent shared load chain per probe.
template <int R>
struct DfsReg {
  const unsigned long long* row[R];  // levels 2..R-1: table base (shared or global)
  uint32_t bits[R], mask[R];
  uint32_t gen, delta, ov;
  bool smem;
};

template <int L, int R>
__device__ __forceinline__ uint32_t table_next_r(const DfsReg<R>& t, uint32_t key, uint32_t* slot) {
  while (true) {
    const unsigned long long g = t.smem ? t.row[L][*slot] : __ldcg(t.row[L] + *slot);
    const uint32_t e = static_cast<uint32_t>(g >> 32) == t.gen ? static_cast<uint32_t>(g) : 0u;
    if (e == 0) return 0;
    *slot = (*slot + 1) & t.mask[L];
    if (((e - 1) & t.ov) == key) return e;
  }
}

template <int L, int R>
__device__ __forceinline__ void dfs(const DfsCtx& d, const DfsReg<R>& t, uint32_t (&tup)[R],
                                    uint32_t (&cnt)[R + 1]) {
  const uint32_t key = ((tup[L - 1] ^ tup[0]) >> t.delta) ^ d.m0;
  uint32_t slot = table_slot(key, t.bits[L]);
  while (true) {
    const uint32_t e = table_next_r<L, R>(t, key, &slot);
    if (e == 0) return;
    tup[L] = e - 1;
    if (++cnt[L + 1] == kStageBatch) stage_flush<L>(d, cnt[L + 1]);
    if constexpr (L + 1 == R) {
      emit_tuple<R>(d, tup);
    } else {
      dfs<L + 1, R>(d, t, tup, cnt);
    }
  }
}

template <int L, int R>
__device__ __forceinline__ void stage_flush_all(const DfsCtx& d, uint32_t (&cnt)[R + 1]) {
  if (cnt[L + 1]) stage_flush<L>(d, cnt[L + 1]);
  if constexpr (L + 1 < R) stage_flush_all<L + 1, R>(d, cnt);
}

template <int R>
__device__ void dfs_pairs(DfsCtx d, const uint64_t* n) {
  const DetectParams& P = *d.P;
  const uint64_t cols = 1ull << P.g.q;
  const uint64_t tid = static_cast<uint64_t>(threadIdx.x) * P.gsize + P.grank;
  const uint64_t nthreads = static_cast<uint64_t>(P.gsize) * blockDim.x;
  const uint64_t n1 = n[1];
  const uint64_t pairs = n[0] * n1;
  uint32_t cnt[R + 1];
#pragma unroll
  for (int x = 0; x <= R; ++x) cnt[x] = 0;
  DfsReg<R> t;
  {
    const Tables& tb = *d.t;
    t.smem = tb.smem;
    t.gen = tb.gen;
    t.delta = P.g.delta;
    t.ov = P.g.overlap_mask;
#pragma unroll
    for (int L = 2; L < R; ++L) {
      t.bits[L] = tb.bits[L];
      t.mask[L] = (1u << tb.bits[L]) - 1;
      t.row[L] = tb.smem ? tb.s + tb.off[L] : tb.gtab + (L - 2) * tb.gstride;
    }
  }
  const uint32_t* lists = d.t->lists;
  const uint32_t loff0 = d.t->loff[0], loff1 = d.t->loff[1];
  uint32_t it = 0;
  for (uint64_t p = tid; p < pairs; p += nthreads) {
    // overflow seen elsewhere: checked every kAbortPoll pairs (the flag is
    // global memory, so each check is an L2 round trip — once per pair it
    // made the growth of C4's ~87 k seed pairs 6x slower); an early stop
    // only saves work, the overflow decision comes from the stage counts
    if ((++it & (kAbortPoll - 1)) == 0 && *reinterpret_cast<volatile unsigned*>(d.abort)) break;
    const uint64_t a = (p | n1) >> 32 ? p / n1
                                      : static_cast<uint32_t>(p) / static_cast<uint32_t>(n1);
    uint32_t tup[R];
    if (lists) {
      tup[0] = lists[loff0 + a];
      tup[1] = lists[loff1 + (p - a * n1)];
    } else {
      tup[0] = __ldcg(P.hot_cols + a);
      tup[1] = __ldcg(P.hot_cols + cols + (p - a * n1));
    }
    d.m0 = tup[0] & t.ov;
    dfs<2, R>(d, t, tup, cnt);
  }
  stage_flush_all<2, R>(d, cnt);
}

// Iterative depth-first walk for r > kRegRows, the walk state (tuple, probe
// positions, keys: 3 r words) in the thread's scratch region of global memory
// (kept out of line; r <= kRegRows keeps its tuple in registers)
__device__ __noinline__ void dfs_deep(const DetectParams& P, ReconCounters* C, const CandSink& k,
                                      const uint64_t* n, const Tables& t, unsigned* abort,
                                      unsigned* cta_stage) {
  const GroupDev& g = P.g;
  const uint32_t r = g.r;
  const uint64_t cols = 1ull << g.q;
  const uint64_t tid = static_cast<uint64_t>(threadIdx.x) * P.gsize + P.grank;
  const uint64_t nthreads = static_cast<uint64_t>(P.gsize) * blockDim.x;
  const uint64_t n1 = n[1];
  const uint64_t pairs = n[0] * n1;
  uint32_t* tup = thread_scratch(P);
  uint32_t* slot = tup + r;  // probe position per level
  uint32_t* key = slot + r;
  uint32_t it = 0;
  for (uint64_t p = tid; p < pairs; p += nthreads) {
    // overflow seen elsewhere, every kAbortPoll pairs (see dfs_pairs)
    if ((++it & (kAbortPoll - 1)) == 0 && *reinterpret_cast<volatile unsigned*>(abort)) break;
    const uint64_t a = (p | n1) >> 32 ? p / n1
                                      : static_cast<uint32_t>(p) / static_cast<uint32_t>(n1);
    const uint64_t b = p - a * n1;
    if (t.lists) {
      tup[0] = t.lists[t.loff[0] + a];
      tup[1] = t.lists[t.loff[1] + b];
    } else {
      tup[0] = __ldcg(P.hot_cols + a);
      tup[1] = __ldcg(P.hot_cols + cols + b);
    }
    const uint32_t m0 = tup[0] & g.overlap_mask;
    uint32_t L = 2;
    key[2] = ((tup[1] ^ tup[0]) >> g.delta) ^ m0;
    slot[2] = table_slot(key[2], t.bits[2]);
    while (L >= 2) {
      const uint32_t e = table_next(t, L, key[L], g.overlap_mask, &slot[L]);
      if (e == 0) {  // row L exhausted for this prefix: backtrack
        --L;
        continue;
      }
      tup[L] = e - 1;
      // a CTA-local count above tuple_cap proves the global one is: the
      // reference overflows, so everyone may stop
      if (atomicAdd(&cta_stage[L + 1], 1u) >= P.tuple_cap) atomicExch(abort, 1u);
      if (L + 1 == r) {
        invert_tuple(P, C, k, tup);
      } else {
        ++L;
        key[L] = ((tup[L - 1] ^ tup[0]) >> g.delta) ^ m0;
        slot[L] = table_slot(key[L], t.bits[L]);
      }
    }
  }
}


__device__ void phase_reconstruct(const DetectParams& P, ReconCounters* C, const CandSink& k,
                                  const uint64_t* n, const Tables& t, unsigned* abort,
                                  unsigned* cta_stage, uint32_t* q_s, unsigned* q_n) {
  const GroupDev& g = P.g;
  const uint32_t r = g.r;
  const DfsCtx d{&P, C, k, &t, abort, cta_stage, q_s, q_n, 0};
  // up to kRegRows rows the tuple stays in registers (one instantiation per
  // row count); more rows walk with the state in the scratch region
  switch (r) {
    case 3: dfs_pairs<3>(d, n); break;
    case 4: dfs_pairs<4>(d, n); break;
    case 5: dfs_pairs<5>(d, n); break;
    case 6: dfs_pairs<6>(d, n); break;
    case 7: dfs_pairs<7>(d, n); break;
    case 8: dfs_pairs<8>(d, n); break;
    default: dfs_deep(P, C, k, n, t, abort, cta_stage);
  }
}

// after a __syncthreads: invert the CTA's queued tuples (a warp per tuple)
// and publish the CTA's stage counts
__device__ void finish_reconstruct(const DetectParams& P, ReconCounters* C, const CandSink& k,
                                   const unsigned* cta_stage, const uint32_t* q_s,
                                   unsigned q_n) {
  const unsigned nq = min(q_n, kQueue);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (unsigned t2 = warp; t2 < nq; t2 += blockDim.x >> 5)
    invert_tuple(P, C, k, q_s + t2 * kQueueWidth, lane, 32);
  if (threadIdx.x >= 3 && threadIdx.x <= P.g.r && cta_stage[threadIdx.x])
    atomicAdd(&C->stage[threadIdx.x], static_cast<unsigned long long>(cta_stage[threadIdx.x]));
}

// ------------------------------------------------------ USLE weights
// Slea::estimate's union and count (slea.cpp:103-114) for n candidates held
// in shared memory, by the whole CTA, from the inside bitmap: output word w
// of a candidate holds slots [32w, 32w+32) = the AND over rows i of the
// bitmap at bit i*row_len + col_i*delta' + 32w (funnel shift across the word
// boundary). `coff` (shared, n x r') receives the per-row bit offsets and
// `cw` (shared, n) the weights; the caller writes them out.
__device__ __noinline__ void cta_usle(const DetectParams& P, const uint2* cs, uint32_t n, uint32_t* coff,
                         unsigned* cw) {
  const SleaDev& le = P.le;
  const uint32_t r = le.r;
  for (uint32_t x = threadIdx.x; x < n * r; x += blockDim.x) {
    const uint32_t c = x / r, i = x - c * r;
    const uint32_t col = static_cast<uint32_t>(seeded(P.lh[i], cs[c].x)) & le.col_mask;
    coff[x] = col * le.delta;
  }
  if (threadIdx.x < n) cw[threadIdx.x] = 0;
  __syncthreads();
  // a thread takes kRun consecutive 32-bit words of one candidate: per row
  // kRun + 1 loads (neighbouring words share their funnel-shift halves), and
  // 5 rows' loads in flight at a time (the paper's r') — the pass is L2-latency
  // bound: 8 words per item and 5 rows take half the round trips of 4 and 8
  constexpr uint32_t kRun = 8, kRowsInFlight = 5;
  const uint32_t words = (le.eta + 31) / 32;
  const uint32_t runs = (words + kRun - 1) / kRun;
  const uint64_t nbw = P.le_bits_words;
  for (uint32_t item = threadIdx.x; item < n * runs; item += blockDim.x) {
    const uint32_t c = item / runs, w0 = (item - c * runs) * kRun;
    uint32_t acc[kRun];
#pragma unroll
    for (uint32_t k = 0; k < kRun; ++k) acc[k] = 0xFFFFFFFFu;
    for (uint32_t i0 = 0; i0 < r; i0 += kRowsInFlight) {
      uint32_t v[kRowsInFlight][kRun + 1], sh[kRowsInFlight];
#pragma unroll
      for (uint32_t u = 0; u < kRowsInFlight; ++u) {
        const uint32_t i = i0 + u;
        sh[u] = 0;
        const uint64_t bit = i < r ? i * le.row_len + coff[c * r + i] + 32ull * w0 : 0;
        const uint64_t b = bit >> 5;
        if (i < r) sh[u] = static_cast<uint32_t>(bit & 31);
#pragma unroll
        for (uint32_t k = 0; k <= kRun; ++k)
          v[u][k] = (i < r && b + k < nbw) ? __ldcg(P.le_bits + b + k) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (uint32_t u = 0; u < kRowsInFlight; ++u)
#pragma unroll
        for (uint32_t k = 0; k < kRun; ++k) acc[k] &= __funnelshift_r(v[u][k], v[u][k + 1], sh[u]);
    }
    unsigned cnt = 0;
#pragma unroll
    for (uint32_t k = 0; k < kRun; ++k) {
      const uint32_t w = w0 + k;
      if (w >= words) break;
      const uint32_t valid = le.eta - 32 * w;
      cnt += __popc(valid < 32 ? acc[k] & ((1u << valid) - 1) : acc[k]);
    }
    // lanes holding runs of the same candidate add up first: one shared
    // atomic per candidate and warp (same-address atomics of a warp
    // serialise: they were 60 % of the engine's shared-memory wavefronts)
    const unsigned same = __match_any_sync(__activemask(), c);
    cnt = __reduce_add_sync(same, cnt);
    if (cnt && (threadIdx.x & 31) == static_cast<uint32_t>(__ffs(same) - 1)) atomicAdd(&cw[c], cnt);
  }
  __syncthreads();
}

// Shared memory of one detection (static part; the overlap tables are the
// dynamic part)
struct DetSmem {
  uint64_t n[kMaxRows];
  Tables tabs;
  uint2 cs[kCandCta];                // candidates found by this CTA: {aip, index}
  unsigned ncs;
  unsigned cw[kCandCta];             // their USLE weights
  uint32_t coff[kCandCta * kMaxRows];  // their per-row bit offsets
  // per-CTA stage counts: 32-bit (64-bit shared atomics are CAS loops on
  // sm_100); exact while below tuple_cap <= 2^30, and a count above it aborts
  unsigned cta_stage[kMaxRows + 1];
  uint32_t q_s[kQueue * kQueueWidth];
  unsigned q_n;
  unsigned row_cnt[kMaxRows];
  bool last;
  uint32_t rs_flags[kRsFlagCap];     // incremental RSRA: flagged blocks of this CTA
  uint32_t rs_hot[kRsHotQuads];      // ... and its range's hot bits
  unsigned rs_nflag;
  unsigned le_logn;                  // SLEA tracked: words logged by this CTA in this detection
};

// Where one window's result goes.
struct WinArgs {
  uint32_t rs_lo, le_lo;
  WinResult* out;          // mapped pinned host memory
  Candidate* host_cands;   // mapped pinned host memory, P.host_prefix entries
  uint32_t* ready;         // mapped flag set after the record (or null)
  Candidate* arena;        // device: candidates beyond the prefix (or null)
  uint64_t arena_cap;
  unsigned long long* ct;  // diagnostics: this CTA's kCtaT timestamps of the op (or null)
  unsigned* set_free;      // engine: published (= set_free_val) once phase A may reuse the
  unsigned set_free_val;   // buffer set, before the record's host writes (or null)
  // engine: the arena is one ring per reconstruction group (`arena`, the
  // group's ring; `arena_head`, its allocation offset), which the host frees
  // in the group's window order (mapped word: ring offset up to which it has
  // copied the tails out); a group's detections run one after the other, so
  // no window waits for another group's
  const unsigned long long* arena_released;
  unsigned long long* arena_head;
  uint32_t win;            // the window's index in the batch
  uint32_t flags;          // engine detect op: kOpInit / kOpInc (0: full phase A only)
};

// run_detection (src/window.cpp:36-78) is split in two halves that the
// engine runs on different CTA groups, pipelined across slices:
//   det_a  phase A over the state (needs the scans of the slice complete and
//          the next slice's scan held back: the stream group's barriers)
//   det_b  reconstruction + USLE weights + the published record (reads only
//          the hot lists and the bitmap of its buffer set, so it overlaps the
//          next slice's scan: the reconstruction group)
// k_detect runs both on every CTA with one barrier in between.
__device__ void det_a(const DetectParams& P, const WinArgs& W, DetSmem& sm) {
  DetectScratch* S = P.scratch;
  if (threadIdx.x < kMaxRows) sm.row_cnt[threadIdx.x] = 0;
  __syncthreads();
  stamp_phase(P, S, 0);
  if ((W.flags & kOpInc) && (W.flags & kOpLe)) {
    // both sketches incremental: per-row deltas into the live counts
    int* delta = reinterpret_cast<int*>(sm.row_cnt);
    phase_a_inc(P, S, W.rs_lo, W.le_lo, delta, true, W.win, &sm.le_logn, sm.rs_flags, &sm.rs_nflag);
    __syncthreads();
    if (threadIdx.x < P.le.r && delta[threadIdx.x])
      atomicAdd(&P.inc.live_row[threadIdx.x],
                static_cast<unsigned long long>(static_cast<long long>(delta[threadIdx.x])));
  } else if (W.flags & kOpInc) {  // RSRA incremental on kRsWarps warps, the SLEA swept by the rest
    if (threadIdx.x < kRsWarps * 32) {
      phase_a_rs_warps(P, S, W.rs_lo, sm.rs_flags, &sm.rs_nflag, sm.rs_hot);
      stamp_cta(W.ct, 13);
    } else {
      // 12 of 16 warps, 6 sectors in flight per lane (4: +2.5 %, 8: +3.5 % per C2 step, A/B)
      phase_a_sector<0, 1, 6>(P, S, W.rs_lo, W.le_lo, sm.row_cnt, kRsWarps * 32,
                              blockDim.x - kRsWarps * 32);
    }
    __syncthreads();
    if (threadIdx.x < P.le.r && sm.row_cnt[threadIdx.x])
      atomicAdd(&S->row_weights[threadIdx.x], static_cast<unsigned long long>(sm.row_cnt[threadIdx.x]));
  } else {
    phase_a(P, S, W.rs_lo, W.le_lo, sm.row_cnt, (W.flags & kOpInit) != 0, (W.flags & kOpLe) != 0);
    __syncthreads();
    if (threadIdx.x < P.le.r && sm.row_cnt[threadIdx.x])
      atomicAdd(&S->row_weights[threadIdx.x], static_cast<unsigned long long>(sm.row_cnt[threadIdx.x]));
  }
  stamp_phase(P, S, 1);
  stamp_cta(W.ct, 1);
}

__device__ __noinline__ void det_b(const DetectParams& P, const WinArgs& W, DetSmem& sm,
                                   unsigned long long* stab, unsigned& bar_target) {
  DetectScratch* S = P.scratch;
  const uint32_t r = P.g.r;
  const uint32_t gen = P.serial;  // overlap-table generation (never 0)
  if (threadIdx.x <= kMaxRows) sm.cta_stage[threadIdx.x] = 0;
  if (threadIdx.x == 0) sm.q_n = 0;
  stamp_phase(P, S, 2);
  stamp_cta(W.ct, 2);

  // ---- phase B: reconstruction + the USLE weight of every candidate.
  // Decisions are identical in every CTA.
  if (threadIdx.x < r) sm.n[threadIdx.x] = __ldcg(&S->hot_counts[threadIdx.x]);
  if (threadIdx.x == 0) sm.ncs = 0;
  __syncthreads();
  stamp_cta(W.ct, 14);
  const uint64_t* n = sm.n;
  bool empty = false;
  for (uint32_t i = 0; i < r; ++i) empty |= n[i] == 0;
  const uint64_t seed_work = empty ? 0 : n[0] * n[1] * n[2];
  const bool cap_overflow = !empty && seed_work > P.work_cap;
  const bool recon = !empty && !cap_overflow;
  Tables& tabs = sm.tabs;
  const CandSink sink{sm.cs, &sm.ncs, P.left, &S->left_n};
  if (recon) {
    const uint64_t cols = 1ull << P.g.q;
    uint32_t* slist = reinterpret_cast<uint32_t*>(stab + kSmemTable);
    if (threadIdx.x == 0) {
      uint32_t off = 0;
      for (uint32_t L = 2; L < r; ++L) {
        tabs.bits[L] = smem_bits(n[L]);
        tabs.off[L] = off;
        off += 1u << tabs.bits[L];
      }
      tabs.smem = off <= kSmemTable;
      tabs.s = stab;
      tabs.gtab = P.table;
      tabs.gstride = P.table_stride;
      tabs.gen = gen;
      if (!tabs.smem)
        for (uint32_t L = 2; L < r; ++L) tabs.bits[L] = P.table_bits;
      uint64_t lo = 0;
      for (uint32_t L = 0; L < r; ++L) {
        tabs.loff[L] = static_cast<uint32_t>(lo);
        lo += n[L];
      }
      tabs.lists = lo <= kSmemLists ? slist : nullptr;
    }
    __syncthreads();
    stamp_cta(W.ct, 13);
    if (tabs.lists) {  // all hot lists in one round trip: independent loads
      const uint32_t total = tabs.loff[r - 1] + static_cast<uint32_t>(n[r - 1]);
      for (uint32_t x = threadIdx.x; x < total; x += blockDim.x) {
        uint32_t L = 0;
        while (L + 1 < r && x >= tabs.loff[L + 1]) ++L;
        slist[x] = __ldcg(P.hot_cols + L * cols + (x - tabs.loff[L]));
      }
      __syncthreads();  // the table inserts and the DFS read other threads' copies
      stamp_cta(W.ct, 19);
    }
    if (tabs.smem) {
      // private tables in every CTA: a few hundred inserts, no grid barrier,
      // no clearing (entries of older generations read as empty)
      for (uint32_t L = 2; L < r; ++L)
        for (uint64_t j = threadIdx.x; j < n[L]; j += blockDim.x) {
          const uint32_t col =
              tabs.lists ? slist[tabs.loff[L] + j] : __ldcg(P.hot_cols + L * cols + j);
          table_insert(stab + tabs.off[L], tabs.bits[L], gen, col & P.g.overlap_mask, col);
        }
      __syncthreads();
    } else {
      // one global copy, generation tagged, then everyone waits for it
      const uint64_t gt = static_cast<uint64_t>(P.grank) * blockDim.x + threadIdx.x;
      const uint64_t gn = static_cast<uint64_t>(P.gsize) * blockDim.x;
      for (uint32_t L = 2; L < r; ++L)
        for (uint64_t j = gt; j < n[L]; j += gn) {
          const uint32_t col = __ldcg(P.hot_cols + L * cols + j);
          table_insert(P.table + (L - 2) * P.table_stride, P.table_bits, gen,
                       col & P.g.overlap_mask, col);
        }
      group_sync(P.gbar, P.gsize, bar_target);
    }
    stamp_cta(W.ct, 15);
    phase_reconstruct(P, &S->cnt, sink, n, tabs, &S->abort, sm.cta_stage, sm.q_s, &sm.q_n);
    __syncthreads();
    if (P.diag && threadIdx.x == 0) atomicMax(&S->phase_ns[8], globaltimer());
    stamp_cta(W.ct, 16);
    finish_reconstruct(P, &S->cnt, sink, sm.cta_stage, sm.q_s, sm.q_n);
    __syncthreads();
    stamp_cta(W.ct, 17);
    // USLE weights of this CTA's candidates (the bitmap is complete since
    // barrier 1); the rest go to the publishing CTA
    const uint32_t nl = min(sm.ncs, kCandCta);
    if (nl) {
      cta_usle(P, sm.cs, nl, sm.coff, sm.cw);
      if (threadIdx.x < nl) P.cands[sm.cs[threadIdx.x].y].weight = sm.cw[threadIdx.x];
    }
    stamp_cta(W.ct, 18);
  }
  if (P.diag && threadIdx.x == 0) atomicMax(&S->phase_ns[11], globaltimer());
  stamp_phase(P, S, 3);
  stamp_cta(W.ct, 3);
  stamp_phase(P, S, 4);
  stamp_phase(P, S, 5);
  stamp_cta(W.ct, 4);
  stamp_cta(W.ct, 5);

  // ---- the last CTA to finish publishes the record and resets the scratch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    sm.last = atomicAdd(&S->done, 1u) == P.gsize - 1;
  }
  __syncthreads();
  if (!sm.last) return;
  stamp_cta(W.ct, 11);
  __threadfence();
  const bool aborted = __ldcg(&S->abort) != 0;
  const uint64_t nc = __ldcg(&S->cnt.n_cand);
  {  // candidates the finding CTAs had no room for
    const unsigned nleft = __ldcg(&S->left_n);
    for (unsigned b = 0; b < nleft; b += kCandCta) {
      const uint32_t m = min(kCandCta, nleft - b);
      __syncthreads();
      if (threadIdx.x < m) {
        const uint32_t idx = __ldcg(P.left + b + threadIdx.x);
        sm.cs[threadIdx.x] = make_uint2(__ldcg(&P.cands[idx].aip), idx);
      }
      __syncthreads();
      cta_usle(P, sm.cs, m, sm.coff, sm.cw);
      if (threadIdx.x < m) P.cands[sm.cs[threadIdx.x].y].weight = sm.cw[threadIdx.x];
    }
    __syncthreads();
  }
  // The record is assembled in shared memory and then written to the mapped
  // host buffer by the whole CTA: nothing here reads host memory, the scratch
  // loads are issued in parallel, and so are the PCIe writes (this CTA's
  // epilogue delays the next slice's grid barrier).
  __shared__ WinResult rec;
  __shared__ uint64_t tail_off;
  __shared__ bool ov_s;
  {
    const uint32_t t = threadIdx.x;
    if (t < kMaxRows) {
      rec.hot_counts[t] = t < r ? n[t] : 0;
      rec.row_weights[t] = t < P.le.r ? __ldcg(&S->row_weights[t]) : 0;
    }
    if (t >= 64 && t <= 64 + kMaxRows) rec.stage_count[t - 64] = __ldcg(&S->cnt.stage[t - 64]);
    if (t >= 160 && t < 166) rec.t_phase[t - 160] = __ldcg(&S->phase_ns[t - 160]);
    if (t >= 192 && t < 196) rec.t_diag[t - 192] = __ldcg(&S->phase_ns[8 + t - 192]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    WinResult& R = rec;
    const unsigned long long now_ns = globaltimer();
    S->phase_ns[6] = now_ns;
    R.t_begin = R.t_phase[0];
    R.t_end = now_ns;
    R.seed_work = seed_work;
    R.checked = 0;
    R.n_candidates = nc;
    R.empty = empty;
    R.pad = 0;
    // overflow exactly as the reference's caps decide it, from the counts
    bool ov = cap_overflow || aborted;
    if (!empty && !ov) {
      uint64_t checked = seed_work;
      for (uint32_t row = 3; row <= r && !ov; ++row) {
        const uint64_t cnt = R.stage_count[row];
        if (cnt > P.tuple_cap) ov = true;
        else if (row < r) {
          const uint64_t work = cnt * n[row];
          if (checked + work > P.work_cap) ov = true;
          checked += work;
        }
      }
    }
    R.overflow = ov;
    ov_s = ov;
    bool trunc = __ldcg(&S->cnt.truncated) != 0;
    // candidates beyond the host prefix go to the group's device ring
    // (engine runs): contiguous ring space once the host has copied enough of
    // the group's earlier tails out (the ring offset is virtual: physical =
    // % cap)
    tail_off = ~0ull;
    const uint64_t kept = min(nc, P.cand_cap);
    if (W.arena && !ov && !empty && kept > P.host_prefix) {
      const uint64_t need = kept - P.host_prefix;
      if (need > W.arena_cap) {
        trunc = true;
      } else {
        uint64_t h = __ldcg(W.arena_head);
        const uint64_t pos = h % W.arena_cap;
        if (pos + need > W.arena_cap) h += W.arena_cap - pos;
        if (h + need > W.arena_cap) wait_host_u64(W.arena_released, h + need - W.arena_cap);
        tail_off = h;
        __stcg(W.arena_head, static_cast<unsigned long long>(h + need));
      }
    }
    R.tail_offset = tail_off;
    R.cand_truncated = trunc;
  }
  __syncthreads();
  // Phase A of the detection two slices on reuses this buffer set: it needs
  // the hot lists, the bitmap and the hot / row counters, all read by now.
  // Release them before the host writes (those only read the candidates
  // and the reconstruction counters, which the engine guards separately).
  for (uint32_t i = threadIdx.x; i < kMaxRows; i += blockDim.x) {
    S->hot_counts[i] = 0;
    S->row_weights[i] = 0;
  }
  __syncthreads();
  if (W.set_free && threadIdx.x == 0) publish(W.set_free, W.set_free_val);
  stamp_cta(W.ct, 8);
  {
    static_assert(sizeof(WinResult) % 8 == 0, "record copied as u64 words");
    const uint64_t* src = reinterpret_cast<const uint64_t*>(&rec);
    uint64_t* dst = reinterpret_cast<uint64_t*>(W.out);
    for (uint32_t i = threadIdx.x; i < sizeof(WinResult) / 8; i += blockDim.x) dst[i] = src[i];
  }
  const uint64_t kept = min(nc, P.cand_cap);
  const uint64_t pre = (ov_s || empty) ? 0 : min(kept, P.host_prefix);
  for (uint64_t i = threadIdx.x; i < pre; i += blockDim.x) W.host_cands[i] = P.cands[i];
  if (tail_off != ~0ull) {
    Candidate* ring = W.arena + tail_off % W.arena_cap;
    for (uint64_t i = pre + threadIdx.x; i < kept; i += blockDim.x) ring[i - pre] = P.cands[i];
  }
  stamp_cta(W.ct, 9);
  // reset for the next detection (nothing reads the scratch any more)
  for (uint32_t i = threadIdx.x; i <= kMaxRows; i += blockDim.x) S->cnt.stage[i] = 0;
  if (threadIdx.x < 4) S->phase_ns[8 + threadIdx.x] = 0;
  __syncthreads();
  stamp_cta(W.ct, 10);
  if (threadIdx.x == 0) {
    S->cnt.n_cand = 0;
    S->cnt.truncated = 0;
    S->abort = 0;
    S->left_n = 0;
    S->done = 0;
    __threadfence_system();
    if (W.ready) *reinterpret_cast<volatile uint32_t*>(W.ready) = 1u;
  }
  stamp_cta(W.ct, 6);
}

__device__ __noinline__ void detect_window(const DetectParams& P, const WinArgs& W, DetSmem& sm,
                                           unsigned long long* stab, unsigned& bar_target) {
  det_a(P, W, sm);
  group_sync(P.gbar, P.gsize, bar_target);
  det_b(P, W, sm, stab, bar_target);
}

// The detection reads its parameters from a shared-memory copy: device
// functions then take the block by reference without the compiler spilling
// the whole kernel-parameter block to local memory.
__global__ void __launch_bounds__(kThreads, 1) k_detect(DetectParams P) {
  __shared__ DetSmem sm;
  __shared__ DetectParams sP;
  extern __shared__ unsigned long long stab[];  // kSmemTable entries + the hot lists
  if (threadIdx.x == 0) {
    sP = P;
    sP.grank = blockIdx.x;
    sP.gsize = gridDim.x;
    sP.gbar = P.bar;
  }
  for (uint32_t i = threadIdx.x; i < kSmemTable; i += blockDim.x) stab[i] = 0ull;
  __syncthreads();
  unsigned bar_target = 0;
  const WinArgs W{P.rs_lo, P.le_lo, P.out, P.host_cands, nullptr, nullptr, 0, nullptr,
                  nullptr, 0, nullptr, nullptr, 0, 0};
  detect_window(sP, W, sm, stab, bar_target);
}

// Grid-wide flag words of the engine (after the two group barrier counters;
// the host zeroes the first kBarBytes before every launch).
// Every word on its own 128 B line; per reconstruction group g: a barrier
// counter at kBarRecon + 32 g, b_done at kBDone + 32 g, e_done at kEDone + 32 g.
constexpr uint32_t kBarStream = 0, kBarRecon = 32, kADone = kBarRecon + 32 * kMaxReconGroups,
                   kBDone = kADone + 32, kEDone = kBDone + 32 * kMaxReconGroups,
                   kPrefix = kEDone + 32 * kMaxReconGroups;  // u32 index
constexpr size_t kBarBytes = (kPrefix + 32) * 4;
static_assert(kBarBytes <= 4096, "flag words fit the barrier allocation");

__device__ __forceinline__ void wait_at_least(const unsigned* flag, unsigned v) {
  if (threadIdx.x == 0) {
    while (static_cast<int>(ld_relaxed(flag) - v) < 0) {
    }
    fence_acquire();
  }
  __syncthreads();
}

// shared parameter copy pointed at buffer set (detection % n_sets)
__device__ __forceinline__ void select_slot(DetectParams& sP, const DetectParams& P, uint32_t det) {
  const DetSet& b = P.sets[det % P.n_sets];
  sP.hot_cols = b.hot_cols;
  sP.le_bits = b.le_bits;
  sP.cands = b.cands;
  sP.left = b.left;
  sP.scratch = b.scratch;
  sP.table = b.table;
}

// ------------------------------------------------------- in-engine merge
// (MergeDev, srlg_internal.cuh). Sending rank: one record's cell update with
// the old stamp returned; a cell whose stamp moved in this slice is appended
// to the CTA's region of the inbox slot (warp-aggregated position from a
// shared counter, consecutive lanes write consecutive words). Exactly one
// entry per (cell, slice, rank): the slice's first writer of a cell is the
// only one that sees an older stamp.
__device__ __forceinline__ void outbox_put(uint32_t* cell, uint32_t now, uint32_t entry,
                                           uint32_t* region, uint32_t* n_sm) {
  uint32_t old;
  asm volatile("atom.relaxed.gpu.global.max.L2::cache_hint.u32 %0, [%1], %2, %3;"
               : "=r"(old)
               : "l"(cell), "r"(now), "l"(policy_evict_last())
               : "memory");
  const bool moved = old < now;
  const unsigned act = __activemask();
  const unsigned m = __ballot_sync(act, moved);
  if (!m) return;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane == leader) base = atomicAdd(n_sm, static_cast<uint32_t>(__popc(m)));
  base = __shfl_sync(act, base, leader);
  if (moved) region[base + __popc(m & ((1u << lane) - 1u))] = entry;
}

// A sending rank's scan op: stamp the own state, list the moved cells in
// slot seq % kInboxSlots (waiting until the root has applied the slot's
// previous use), then — once every CTA is done — publish the slice. The
// rank's CTAs keep a barrier per slice so that a cell's first writer in the
// slice is a writer of this slice (no CTA runs ahead into the next one).
template <int ROWS>
__device__ __noinline__ void rank_scan(const DetectParams& P, const MergeDev& M, EngineOp op,
                                       const srlg_pair* pairs, uint32_t* n_sm, unsigned& bar_target) {
  const uint32_t slot = op.seq % kInboxSlots;
  InboxRank* H = M.hdr + M.rank;
  if (threadIdx.x == 0) {
    if (op.seq >= kInboxSlots) wait_flag(&H->consumed, op.seq + 1 - kInboxSlots);
    *n_sm = 0;
    if (blockIdx.x == 0) H->grid = gridDim.x;
  }
  __syncthreads();
  const uint64_t per_cta = M.slot_cap / gridDim.x;
  uint32_t* region = M.lists + (static_cast<uint64_t>(M.rank) * kInboxSlots + slot) * M.slot_cap +
                     blockIdx.x * per_cta;
  const uint32_t le_base = static_cast<uint32_t>(M.rs_n);
  uint32_t records = 0;
  for (uint64_t i = op.begin + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
       i < op.end; i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    records += ingest_with(P.anet, ld_pair_stream(pairs + i), [&](uint32_t aip, uint32_t bip) {
      rsra_cells(P.rs, aip, bip, [&](uint64_t idx) {
        outbox_put(P.rs.cells + idx, op.rs_now, static_cast<uint32_t>(idx), region, n_sm);
      });
      slea_cells<ROWS>(P.le, P.lh, aip, bip, [&](uint64_t idx) {
        outbox_put(P.le.cells + idx, op.le_now, le_base + static_cast<uint32_t>(idx), region, n_sm);
      });
    });
  }
  if (P.anet.n && P.raw_records) {
    records = __reduce_add_sync(__activemask(), records);
    if ((threadIdx.x & 31) == 0 && records)
      atomicAdd(P.raw_records, static_cast<unsigned long long>(records));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    H->counts[slot][blockIdx.x] = *n_sm;
    fence_sys();  // the region's entries and the count reach the root first
  }
  group_sync(P.gbar, P.gsize, bar_target);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    fence_sys();
    st_release_sys(&H->done, op.seq + 1);
  }
}

// The root's share of a slice's merge: after its own scan of the slice, CTA
// g of the n_part CTAs that scanned it applies entries [T g / n, T (g+1) / n)
// of every rank's list (T = the list's length; the per-region counts are
// prefix-summed in shared memory, an entry's region found by bisection) as
// red.max of the slice's stamp. The last CTA to finish a rank's list
// releases the slot to that rank.
__device__ __noinline__ void root_apply(const DetectParams& P, const MergeDev& M, EngineOp op,
                                        uint32_t g, uint32_t n_part, uint32_t* pref) {
  const uint32_t slot = op.seq % kInboxSlots;
  for (uint32_t r = 0; r < M.nranks; ++r) {
    if (r == M.rank) continue;
    InboxRank* H = M.hdr + r;
    cta_wait_flag(&H->done, op.seq + 1);
    const uint32_t G = min(__ldcg(&H->grid), kInboxMaxCtas);
    if (threadIdx.x < 32) {  // exclusive prefix of the G region counts
      const uint32_t lane = threadIdx.x, per = (G + 31) / 32;
      const uint32_t a = min(G, lane * per), b = min(G, a + per);
      uint32_t sum = 0;
      for (uint32_t c = a; c < b; ++c) sum += __ldcg(&H->counts[slot][c]);
      uint32_t incl = sum;
      for (uint32_t d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= d) incl += t;
      }
      uint32_t run = incl - sum;
      for (uint32_t c = a; c < b; ++c) {
        pref[c] = run;
        run += __ldcg(&H->counts[slot][c]);
      }
      if (lane == 31) pref[G] = incl;
    }
    __syncthreads();
    const uint64_t total = pref[G];
    const uint64_t lo = total * g / n_part, hi = total * (g + 1) / n_part;
    if (threadIdx.x == 0 && hi > lo) atomicAdd(M.entries, static_cast<unsigned long long>(hi - lo));
    const uint64_t per_cta = M.slot_cap / max(G, 1u);
    const uint32_t* list = M.lists + (static_cast<uint64_t>(r) * kInboxSlots + slot) * M.slot_cap;
    for (uint64_t f = lo + threadIdx.x; f < hi; f += blockDim.x) {
      uint32_t a = 0, b = G;  // pref[a] <= f < pref[b]
      while (b - a > 1) {
        const uint32_t mid = (a + b) >> 1;
        if (pref[mid] <= f) a = mid;
        else b = mid;
      }
      const uint32_t e = __ldcg(list + a * per_cta + (f - pref[a]));
      if (op.flags & kOpTrack) {  // the merged cells are tracked like scanned ones
        if (e < M.rs_n)
          track_rs_cell(P.rs.cells, P.inc.rs_smin, e, op.rs_now);
        else if (op.flags & kOpLe)
          track_le_cell(P.le, P.inc, e - M.rs_n, op.le_now);
        else
          put_stamp<kStoreRedMax>(P.le.cells + (e - M.rs_n), op.le_now);
      } else if (e < M.rs_n) {
        put_stamp<kStoreRedMax>(P.rs.cells + e, op.rs_now);
      } else {
        put_stamp<kStoreRedMax>(P.le.cells + (e - M.rs_n), op.le_now);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned done_ctas;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                   : "=r"(done_ctas)
                   : "l"(&H->applied[slot])
                   : "memory");
      if (done_ctas == n_part - 1) {
        H->applied[slot] = 0;
        fence_sys();
        st_release_sys(&H->consumed, op.seq + 1);
      }
    }
  }
}

// The persistent engine: a whole batch of slices in one cooperative launch,
// with the CTAs in two roles pipelined across slices.
//   stream group (CTAs >= recon_ctas): the packet scans and phase A. A detect
//     op waits for the slice's scans at a stream barrier, streams the state
//     (det_a), and holds the next slice's scan back with a second barrier,
//     after which detection d is published in a_done.
//   reconstruction groups (CTAs < recon_ctas; CTA c in group c % G, G =
//     recon_groups): group d % G takes detection d: it waits for a_done > d,
//     reconstructs, weighs the candidates, releases the buffer set
//     (b_done[g] = d + 1) and publishes the record (then e_done[g]).
//     Detection d uses buffer set d % S (S = n_sets = G + 1), so phase A of
//     detection d first waits for the release of d - S, and the group
//     reconstructing d for the epilogue of d - S (another group) to finish.
// The reconstruction of slice s thus overlaps the scans and phase A of the
// next slices: each group has G slices' time per detection, and a
// detection's latency may reach S slice periods before phase A waits. Scan
// ops stamp with red.max (CTAs race ahead across scan-only slices; the larger
// stamp wins). The host computes every op's stamps, window lows and serials
// exactly as WindowEngine advances its clocks (capi.cu).
// pull this CTA's share of a scan op's pairs into L2 ahead of time (the
// trace is read once: without it the scan waits on DRAM)
__device__ __forceinline__ void prefetch_pairs(const EngineOp& nx, uint32_t rank, uint32_t size,
                                               const srlg_pair* pairs) {
  const uint64_t a = (nx.begin * sizeof(srlg_pair)) & ~uint64_t(15);
  const uint64_t b = (nx.end * sizeof(srlg_pair) + 15) & ~uint64_t(15);
  const uint64_t share = (((b - a) / size) + 15) & ~uint64_t(15);
  const uint64_t lo = a + share * rank;
  const uint64_t hi = min(b, lo + share);
  if (hi > lo)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(
                     reinterpret_cast<const char*>(pairs) + lo),
                 "r"(static_cast<uint32_t>(hi - lo))
                 : "memory");
}

// A scan op's pairs [i, e) of this thread, stride ls: RSRA + SLEA stamps
// (kOpTrack: with the marks of the incremental detection; P.anet.n: raw
// packets classified first). A thread's pairs go in groups of kScanGroup:
// every pair load of the group is issued before its first update (one L2
// round trip per group).
constexpr int kScanGroup = 3;
template <int ROWS, int kG = kScanGroup>
__device__ __forceinline__ void scan_pairs(const DetectParams& P, const srlg_pair* pairs,
                                           uint32_t rs_now, uint32_t le_now, uint32_t flags,
                                           uint64_t i, uint64_t e, uint64_t lstride) {
        auto load_group = [&](uint2 (&pg)[kG]) {
          uint32_t n = 0;
  #pragma unroll
          for (int k = 0; k < kG; ++k) {
            pg[k] = make_uint2(0, 0);
            if (i + k * lstride < e) {
              pg[k] = ld_pair_stream(pairs + i + k * lstride);
              n = k + 1;
            }
          }
          return n;
        };
        if (flags & kOpTrack) {  // after a detection: mark blocks for the next one (IncDev)
          const IncDev& I = P.inc;
          const bool le = (flags & kOpLe) != 0;
          if (P.anet.n) {
            uint32_t records = 0;
            for (; i < e; i += lstride)
              records += ingest_with(P.anet, ld_pair_stream(pairs + i), [&](uint32_t aip, uint32_t bip) {
                if (le) {
                  const uint2 p1[1] = {make_uint2(aip, bip)};
                  track_records<ROWS, 1>(P.rs, P.le, P.lh, I, rs_now, le_now, p1, 1);
                } else {
                  track_rs_record<ROWS>(P.rs, P.le, P.lh, I, rs_now, le_now, aip, bip);
                }
              });
            records = __reduce_add_sync(0xFFFFFFFFu, records);
            if ((threadIdx.x & 31) == 0 && records && P.raw_records)
              atomicAdd(P.raw_records, static_cast<unsigned long long>(records));
          } else if (le) {
            // reds and bitmap reads of the group, each one round trip
            for (; i < e; i += kG * lstride) {
              uint2 pg[kG];
              const uint32_t n = load_group(pg);
              track_records<ROWS, kG>(P.rs, P.le, P.lh, I, rs_now, le_now, pg, n);
            }
          } else {
            for (; i < e; i += kG * lstride) {
              uint2 pg[kG];
              const uint32_t n = load_group(pg);
  #pragma unroll
              for (int k = 0; k < kG; ++k)
                if (k < n) track_rs_record<ROWS>(P.rs, P.le, P.lh, I, rs_now, le_now, pg[k].x, pg[k].y);
            }
          }
          i = e;
        }
        if (P.anet.n) {  // raw packets: classify (trace.cpp:111-116) fused into the scan
          uint32_t records = 0;
          for (; i < e; i += lstride)
            records += ingest<kStoreRedMax, ROWS>(P.rs, P.le, P.lh, rs_now, le_now, P.anet,
                                                  ld_pair_stream(pairs + i));
          records = __reduce_add_sync(0xFFFFFFFFu, records);
          if ((threadIdx.x & 31) == 0 && records && P.raw_records)
            atomicAdd(P.raw_records, static_cast<unsigned long long>(records));
          i = e;
        }
        for (; i < e; i += kG * lstride) {
          uint2 pg[kG];
          const uint32_t n = load_group(pg);
  #pragma unroll
          for (int k = 0; k < kG; ++k)
            if (k < n) {
              rsra_update<kStoreRedMax>(P.rs, rs_now, pg[k].x, pg[k].y);
              slea_update<kStoreRedMax, ROWS>(P.le, P.lh, le_now, pg[k].x, pg[k].y);
            }
        }
}

// Large scan ops (C4: the updates go to HBM, and CTAs drift apart by tens of
// us over a slice): the stream CTAs claim chunks of kDynScanChunk pairs from
// the op's counter; the next chunk is claimed while the current one is
// scanned (the counter's round trip overlaps it). Out of line: the static
// path's register allocation stays as it was.
template <int ROWS>
__device__ __noinline__ void scan_dynamic(const DetectParams& P, const srlg_pair* pairs,
                                          uint32_t rs_now, uint32_t le_now, uint32_t flags,
                                          uint64_t begin, uint64_t n, unsigned long long* grab,
                                          uint64_t chunk) {
  __shared__ unsigned long long s_chunk;
  if (threadIdx.x == 0) s_chunk = atomicAdd(grab, chunk);
  __syncthreads();
  for (uint64_t c = s_chunk; c < n;) {
    unsigned long long nx = 0;
    if (threadIdx.x == 0) nx = atomicAdd(grab, chunk);
    scan_pairs<ROWS>(P, pairs, rs_now, le_now, flags, begin + c + threadIdx.x,
                     begin + min(c + chunk, n), blockDim.x);
    __syncthreads();
    if (threadIdx.x == 0) s_chunk = nx;
    __syncthreads();
    c = s_chunk;
  }
}

template <int ROWS>
__global__ void __launch_bounds__(kThreads, 1) k_engine(DetectParams P, const EngineOp* ops,
                                                        uint32_t n_ops, const srlg_pair* pairs,
                                                        EngineRing ring) {
  __shared__ DetSmem sm;
  __shared__ DetectParams sP;  // the detection's view (see k_detect); scans use P
  __shared__ uint32_t merge_sm[kInboxMaxCtas + 1];  // merge: outbox count / region prefix
  __shared__ MergeDev sM;  // merge parameters (shared copy: taken by reference out of line)
  extern __shared__ unsigned long long stab[];
  const uint32_t R = P.recon_ctas;  // a multiple of G (0: a merge rank, which only scans)
  const uint32_t G = P.recon_groups;
  const uint32_t NS = P.n_sets;
  const bool recon = blockIdx.x < R;
  const uint32_t group = recon ? blockIdx.x % G : 0;  // reconstruction group
  if (threadIdx.x == 0) {
    sP = P;
    sP.grank = recon ? blockIdx.x / G : blockIdx.x - R;
    sP.gsize = recon ? R / G : gridDim.x - R;
    sP.gbar = P.bar + (recon ? kBarRecon + 32 * group : kBarStream);
    sM = ring.merge;
  }
  for (uint32_t i = threadIdx.x; i < kSmemTable; i += blockDim.x) stab[i] = 0ull;
  if (threadIdx.x == 0) {
    sm.rs_nflag = 0;
    sm.le_logn = 0;
  }
  unsigned bar_target = 0;
  if (blockIdx.x == 0 && threadIdx.x < kMaxReconGroups && ring.arena_heads)
    ring.arena_heads[threadIdx.x] = 0;  // read after a_done waits
  __syncthreads();
  const uint64_t gtid = static_cast<uint64_t>(sP.grank) * blockDim.x + threadIdx.x;
  const uint64_t gsize = static_cast<uint64_t>(sP.gsize) * blockDim.x;
  // scans before the launch's first detect op (the first k - 1 slices) run
  // on every CTA: the reconstruction group has nothing to do yet
  bool prefix = true;
  unsigned* prefix_done = P.bar + kPrefix;  // reconstruction CTAs done with the prefix
  uint32_t chunks_seen = 0;  // host-input chunks known to be resident
  unsigned* a_done = P.bar + kADone;
  unsigned* b_done = P.bar + kBDone;
  unsigned* e_done = P.bar + kEDone;  // per group: detections whose epilogue is complete
  // the next op and the buffer-release flag are loaded one op ahead, so
  // their L2 round trips overlap the current op
  EngineOp nxt = n_ops ? ops[0] : EngineOp{};
  uint32_t dets = 0;    // detect ops passed (thread 0 of a stream CTA)
  unsigned b_seen = 0;  // ... the release flag the next one waits for,
  uint32_t b_for = ~0u; // ... read for detection b_for
  uint32_t o_first = 0;
  if (ring.merged_prefix) {
    // the leading scan ops as one loop over their (contiguous) pairs: each
    // thread follows its pair index through the op boundaries (shared
    // memory, borrowed from the overlap tables and zeroed again after)
    const uint32_t np = ring.merged_prefix;
    uint32_t* s_end = reinterpret_cast<uint32_t*>(stab);
    uint32_t* s_rs = s_end + np;
    uint32_t* s_le = s_rs + np;
    for (uint32_t j = threadIdx.x; j < np; j += blockDim.x) {
      const EngineOp q = ops[j];
      s_end[j] = static_cast<uint32_t>(q.end);
      s_rs[j] = q.rs_now;
      s_le[j] = q.le_now;
    }
    __syncthreads();
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t e_all = s_end[np - 1];
    uint64_t i = nxt.begin + static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    uint32_t ob = 0;
    for (; i + stride < e_all; i += 2 * stride) {
      while (i >= s_end[ob]) ++ob;
      uint32_t ob2 = ob;
      while (i + stride >= s_end[ob2]) ++ob2;
      const uint2 a = ld_pair_stream(pairs + i), b = ld_pair_stream(pairs + i + stride);
      rsra_update<kStoreRedMax>(P.rs, s_rs[ob], a.x, a.y);
      slea_update<kStoreRedMax, ROWS>(P.le, P.lh, s_le[ob], a.x, a.y);
      rsra_update<kStoreRedMax>(P.rs, s_rs[ob2], b.x, b.y);
      slea_update<kStoreRedMax, ROWS>(P.le, P.lh, s_le[ob2], b.x, b.y);
      ob = ob2;
    }
    for (; i < e_all; i += stride) {
      while (i >= s_end[ob]) ++ob;
      const uint2 a = ld_pair_stream(pairs + i);
      rsra_update<kStoreRedMax>(P.rs, s_rs[ob], a.x, a.y);
      slea_update<kStoreRedMax, ROWS>(P.le, P.lh, s_le[ob], a.x, a.y);
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < kSmemTable; j += blockDim.x) stab[j] = 0ull;
    o_first = np;
    if (np < n_ops) {
      nxt = ops[np];
      if (threadIdx.x == 0 && nxt.kind == 0) prefetch_pairs(nxt, blockIdx.x, gridDim.x, pairs);
    }
    __syncthreads();
  }
  for (uint32_t o = o_first; o < n_ops; ++o) {
    const EngineOp op = nxt;
    if (o + 1 < n_ops) nxt = ops[o + 1];
    if (op.kind == 1 && prefix) {
      prefix = false;
      if (recon) {  // this CTA's prefix scans are complete
        __syncthreads();
        if (threadIdx.x == 0)
          asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(prefix_done) : "memory");
      } else if (threadIdx.x == 0) {
        // phase A of the first detection also needs the reconstruction
        // CTAs' scans (acquired by the fence at the end of group_sync)
        while (static_cast<int>(ld_relaxed(prefix_done) - R) < 0) {
        }
      }
    }
    const bool scan_all = prefix && op.kind == 0;  // every CTA scans this op
    if (recon && !scan_all && (op.kind == 0 || op.window % G != group)) continue;
    // (thread 0 waits for this load at once — the value is spilled — and
    // starts its pairs an L2 round trip late; loading the flag at the detect
    // op instead measured 1.6 % slower on C2, A/B)
    if (!recon && threadIdx.x == 0 && op.kind == 0 && dets >= NS) {
      b_seen = ld_relaxed(b_done + 32 * ((dets - NS) % G));
      b_for = dets;
    }
    unsigned long long* ct =
        ring.cta_t ? ring.cta_t + (static_cast<uint64_t>(o) * gridDim.x + blockIdx.x) * kCtaT
                   : nullptr;
    if (ring.op_t && threadIdx.x == 0) {
      const unsigned long long t = globaltimer();
      atomicMin(&ring.op_t[2 * o], t);
      ct[0] = t;
    }
    const uint32_t det = op.window;
    const WinArgs W{op.rs_lo,       op.le_lo,
                    ring.out + det, ring.cands + det * P.host_prefix,
                    ring.ready + det, recon ? ring.arena + group * ring.arena_cap : nullptr,
                    ring.arena_cap, ct,
                    recon ? b_done + 32 * group : nullptr, det + 1,
                    recon ? ring.arena_released + group : nullptr,
                    recon ? ring.arena_heads + group : nullptr,
                    det, op.flags};
    if (recon && !scan_all) {
      wait_at_least(a_done, det + 1);
      // the previous detection on this buffer set (det - NS, another group)
      // has finished its epilogue: candidates and counters are free again
      if (det >= NS) wait_at_least(e_done + 32 * ((det - NS) % G), det - NS + 1);
      if (threadIdx.x == 0) {
        select_slot(sP, P, det);
        sP.serial = op.serial;
      }
      __syncthreads();
      if (ct && threadIdx.x == 0) ct[12] = globaltimer();
      det_b(sP, W, sm, stab, bar_target);
      if (sm.last) {  // the publishing CTA (b_done went out inside det_b)
        __syncthreads();
        if (threadIdx.x == 0) publish(e_done + 32 * group, det + 1);
      }
    } else if (op.kind == 0) {
      const uint64_t first = scan_all ? static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x
                                      : gtid;
      const uint64_t stride = scan_all ? static_cast<uint64_t>(gridDim.x) * blockDim.x : gsize;
      // scan-only runs (the first k - 1 slices): the next scan's pairs now
      if (threadIdx.x == 0 && (op.flags & kOpNextScan)) {
        if (scan_all)
          prefetch_pairs(nxt, blockIdx.x, gridDim.x, pairs);
        else
          prefetch_pairs(nxt, sP.grank, sP.gsize, pairs);
      }
      // the slice's input has arrived: every chunk up to the one holding its
      // last pair (chunks land out of order over two copy streams)
      for (; ring.chunk_flags && static_cast<int>(op.chunk - chunks_seen) >= 0; ++chunks_seen)
        cta_wait_flag(ring.chunk_flags + chunks_seen, 1u);
      if (ring.merge.role == 2) {  // a sending rank: stamp, list, publish
        rank_scan<ROWS>(sP, sM, op, pairs, merge_sm, bar_target);
        goto op_done;
      }
      uint64_t i = op.begin + first;
      uint64_t e = op.end;
#if SRLG_SCAN_GROUPED
      // steady state: every stream CTA takes an equal contiguous share of the
      // slice (a grid stride left ~60 % of the CTAs one pair per thread
      // longer, and the barrier waits for them), and a thread loads its
      // (<= kG) pairs before the first update: one L2 round trip per thread.
      // Large slices (C4: the updates go to HBM, and CTAs drift apart by tens
      // of us) are taken in chunks from a per-op counter instead.
      const uint64_t n_op = op.end - op.begin;
      const bool dyn = !scan_all && n_op >= kDynScanMin * sP.gsize;
      if (!scan_all) {
        i = op.begin + n_op * sP.grank / sP.gsize + threadIdx.x;
        e = op.begin + n_op * (sP.grank + 1) / sP.gsize;
      }
      const uint64_t lstride = scan_all ? stride : blockDim.x;
#else
      constexpr bool dyn = false;
      const uint64_t n_op = 0;
      const uint64_t lstride = stride;
#endif
      if (dyn)
        scan_dynamic<ROWS>(sP, pairs, op.rs_now, op.le_now, op.flags, op.begin, n_op,
                           const_cast<unsigned long long*>(&ops[o].grab), kDynScanChunk);
      else
        scan_pairs<ROWS>(P, pairs, op.rs_now, op.le_now, op.flags, i, e, lstride);
      // the root: the other ranks' cells of this slice, before any phase A
      // reads it (the stream barrier of the slice's detect op follows)
      if (ring.merge.role == 1)
        root_apply(sP, sM, op, scan_all ? blockIdx.x : sP.grank, scan_all ? gridDim.x : sP.gsize,
                   merge_sm);
    } else {
      // buffer set det % NS is free: detection det - NS (group (det - NS) % G)
      // released it. Thread 0's relaxed observation is ordered before phase A
      // by the acquire fence at the end of group_sync.
      // (polled after this CTA's arrival at the barrier: the two waits overlap)
      group_sync(sP.gbar, sP.gsize, bar_target, [&] {  // the slice's scans are complete
        if (det >= NS) {
          const unsigned* f = b_done + 32 * ((det - NS) % G);
          unsigned v = b_for == det ? b_seen : 0u;
          while (static_cast<int>(v - (det - NS + 1)) < 0) v = ld_relaxed(f);
        }
        dets = det + 1;
        if (ct) ct[20] = globaltimer();
      });
      // the next slice's pairs land in L2 during phase A (nxt is already
      // loaded: no extra round trip on warp 0's path)
      if (threadIdx.x == 0 && o + 1 < n_ops && nxt.kind == 0)
        prefetch_pairs(nxt, sP.grank, sP.gsize, pairs);
      if (threadIdx.x == 0) select_slot(sP, P, det);
      __syncthreads();
      if (ct && threadIdx.x == 0) ct[12] = globaltimer();
      det_a(sP, W, sm);
      group_sync(sP.gbar, sP.gsize, bar_target);  // phase A done; the next scan may start
      if (sP.grank == 0 && threadIdx.x == 0) {
        // the SLEA row counts: the live counts follow a full pass, and an
        // incremental pass reports them
        DetectScratch* S = sP.scratch;
        for (uint32_t i = 0; (op.flags & kOpLe) && i < P.le.r; ++i) {
          if (op.flags & kOpInc)
            S->row_weights[i] = __ldcg(&P.inc.live_row[i]);
          else if (op.flags & kOpInit)
            P.inc.live_row[i] = __ldcg(&S->row_weights[i]);
        }
        publish(a_done, det + 1);
      }
    }
  op_done:
    if (ring.op_t) {  // diagnostics: when the last CTA left the op
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned long long t = globaltimer();
        atomicMin(&ring.op_t[2 * o + 1], ~t);  // max end
        ct[7] = t;
      }
    }
  }
}

template <class K>
int grid_for_kernel(K kernel, int device) {
  int per_sm = 0, sms = 0;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kDynSmem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, kDynSmem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return std::max(1, std::min(per_sm, 1)) * sms;
}

}  // namespace

int detect_grid(int device) {
  grid_for_kernel(k_engine<5>, device);
  grid_for_kernel(k_engine<3>, device);
  grid_for_kernel(k_engine<0>, device);
  return grid_for_kernel(k_detect, device);
}

// The grid-barrier counter restarts at zero for every launch.
cudaError_t detect(const DetectParams& P, int grid, cudaStream_t st) {
  DetectParams p = P;
  void* args[] = {&p};
  cudaError_t e = cudaMemsetAsync(P.bar, 0, kBarBytes, st);
  if (e != cudaSuccess) return e;
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_detect), dim3(grid), dim3(kThreads),
                                     args, kDynSmem, st);
}

cudaError_t engine_run(const DetectParams& P, const EngineOp* ops, uint32_t n_ops,
                       const srlg_pair* pairs, const EngineRing& ring, int grid, cudaStream_t st) {
  DetectParams p = P;
  EngineRing g = ring;
  const EngineOp* o = ops;
  uint32_t n = n_ops;
  const srlg_pair* pr = pairs;
  void* args[] = {&p, &o, &n, &pr, &g};
  void* fn = P.le.r == 5   ? reinterpret_cast<void*>(k_engine<5>)
             : P.le.r == 3 ? reinterpret_cast<void*>(k_engine<3>)
                           : reinterpret_cast<void*>(k_engine<0>);
  cudaError_t e = cudaMemsetAsync(P.bar, 0, kBarBytes, st);
  if (e != cudaSuccess) return e;
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, kDynSmem, st);
}

}  // namespace dev
}  // namespace srlg
