// detect.cu — the per-slide estimate as ONE persistent cooperative kernel.
//
// run_detection (src/window.cpp:36-78) needs, per completed slice:
//   A  hot SREs per row (Rsra::extract_hot, src/rsra.cpp:45-57) and the
//      inside-window count of every SLEA row (Slea::setting_factor,
//      src/slea.cpp:57-61)                          -> one pass over the state
//   B  candidate reconstruction (reconstruct_candidates,
//      src/reconstruct.cpp:32-151 + ReversibleHashGroup::invert,
//      src/hash.cpp:77-112)                         -> small, latency bound
//   C  the USLE weight of every candidate (Slea::estimate,
//      src/slea.cpp:103-114)                        -> r' x eta' reads each
// As separate launches these stages are dominated by launch gaps and by
// serial single-CTA work, so they run as phases of one kernel (grid = one CTA
// per SM, cooperative launch so every CTA is resident) with two grid
// barriers.
//
// Reconstruction. A partial tuple (he0, .., he_{L-1}) extends with column he
// of row L iff (he & overlap_mask) == ((he_{L-1} ^ he0) >> delta) ^
// (he0 & overlap_mask) — hash.hpp:101-103 rewritten as an equality on masked
// bits. Phase A therefore inserts every hot column of rows >= 2 into a
// per-row open-addressing table keyed by (col & overlap_mask), and phase B
// walks, for every (row-0, row-1) pair in parallel over the whole grid, the
// tree of consistent extensions depth-first, inverting each complete tuple
// on the spot. It yields exactly the reference's tuple set per stage; the
// per-stage counts feed the reference's tuple_cap / work_cap decisions
// (reconstruct.cpp:60-63, 97-99, 110-113) afterwards, in its own
// brute-force units. Table entries carry a launch generation, so the tables
// never need clearing.
//
// The result record and the first candidates go straight into mapped pinned
// host memory; the host forms the doubles.
#include <algorithm>

#include "srlg_internal.cuh"

namespace srlg {
namespace dev {
namespace {

constexpr int kThreads = 1024;

__device__ __forceinline__ uint32_t ld_acquire(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// CTA 0's view of the phase boundaries (diagnostics: srlg_detect_phase_ns)
__device__ __forceinline__ void stamp_phase(DetectScratch* S, int i) {
  if (blockIdx.x == 0 && threadIdx.x == 0) S->phase_ns[i] = globaltimer();
}

// Grid barrier: the last arriving CTA resets the count and bumps the
// generation. Valid because the launch is cooperative (all CTAs resident).
// The words live in their own allocation so the spinning does not queue in
// front of the counters other CTAs are updating.
__device__ void grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire(&bar[1]);
    __threadfence();
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      unsigned ns = 32;
      while (ld_acquire(&bar[1]) == gen) {
        __nanosleep(ns);
        if (ns < 256) ns *= 2;
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t count_gt4(uint4 v, uint32_t lo) {
  return (v.x > lo) + (v.y > lo) + (v.z > lo) + (v.w > lo);
}

__device__ __forceinline__ uint4 ld4(const uint32_t* p) {
  return *reinterpret_cast<const uint4*>(p);
}

__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xFFFFFFFFu, t, o);
  }
  return t;  // valid in thread 0
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
  unsigned long long cur = __ldcg(T + i);
  while (true) {
    if (static_cast<uint32_t>(cur >> 32) != gen) {
      const unsigned long long old = atomicCAS(T + i, cur, e);
      if (old == cur) return;
      cur = old;  // raced: re-examine the same slot
    } else {
      i = (i + 1) & mask;
      cur = __ldcg(T + i);
    }
  }
}

// ---------------------------------------------------------------- phase A
__device__ void phase_counts(const DetectParams& P, DetectScratch* S, uint32_t* red) {
  const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t gsize = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // RSRA: thread per SRE; a warp covers 32 consecutive SREs of one row when
  // 2^q >= 32, so one aggregated atomic appends its hot columns
  const RsraDev& rs = P.rs;
  const uint64_t cols = 1ull << rs.q;
  const uint64_t sres = static_cast<uint64_t>(rs.r) << rs.q;
  const uint64_t span = (sres + 31) & ~uint64_t(31);
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t s = gtid; s < span; s += gsize) {
    bool hot = false;
    if (s < sres) {
      const uint32_t* p = rs.cells + s * rs.eta;
      uint32_t w = 0;
      if (rs.eta == 8) {
        w = count_gt4(ld4(p), P.rs_lo) + count_gt4(ld4(p + 4), P.rs_lo);
      } else if ((rs.eta & 3) == 0) {
        for (uint32_t z = 0; z < rs.eta; z += 4) w += count_gt4(ld4(p + z), P.rs_lo);
      } else {
        for (uint32_t z = 0; z < rs.eta; ++z) w += p[z] > P.rs_lo;
      }
      hot = w >= P.hot_min;
    }
    const uint32_t row = static_cast<uint32_t>(s >> rs.q);
    const uint32_t col = static_cast<uint32_t>(s & (cols - 1));
    if (cols >= 32) {
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, hot);
      if (m) {
        unsigned long long base = 0;
        if (lane == __ffs(m) - 1)
          base = atomicAdd(&S->hot_counts[row], static_cast<unsigned long long>(__popc(m)));
        base = __shfl_sync(0xFFFFFFFFu, base, __ffs(m) - 1);
        if (hot) P.hot_cols[row * cols + base + __popc(m & ((1u << lane) - 1))] = col;
      }
    } else if (hot) {
      const unsigned long long i = atomicAdd(&S->hot_counts[row], 1ull);
      P.hot_cols[row * cols + i] = col;
    }
  }
  // SLEA: inside counts per row, 4 x uint4 in flight per thread
  const SleaDev& le = P.le;
  for (uint32_t row = 0; row < le.r; ++row) {
    const uint32_t* base = le.cells + row * le.row_len;
    uint32_t cnt = 0;
    uint64_t head = 0;
    if (((row * le.row_len) & 3) != 0) {  // misaligned row start: scalar head
      head = 4 - ((row * le.row_len) & 3);
      if (head > le.row_len) head = le.row_len;
      if (gtid < head) cnt += base[gtid] > P.le_lo;
    }
    const uint64_t nv = (le.row_len - head) / 4;
    const uint32_t* vb = base + head;
    uint64_t v = gtid;
    for (; v + 3 * gsize < nv; v += 4 * gsize) {
      const uint4 a = ld4(vb + 4 * v), b = ld4(vb + 4 * (v + gsize));
      const uint4 c = ld4(vb + 4 * (v + 2 * gsize)), d = ld4(vb + 4 * (v + 3 * gsize));
      cnt += count_gt4(a, P.le_lo) + count_gt4(b, P.le_lo) + count_gt4(c, P.le_lo) +
             count_gt4(d, P.le_lo);
    }
    for (; v < nv; v += gsize) cnt += count_gt4(ld4(vb + 4 * v), P.le_lo);
    for (uint64_t x = head + 4 * nv + gtid; x < le.row_len; x += gsize) cnt += base[x] > P.le_lo;
    const uint32_t t = block_sum(cnt, red);
    if (threadIdx.x == 0 && t) atomicAdd(&S->row_weights[row], static_cast<unsigned long long>(t));
  }
}

// ---------------------------------------------------------------- phase B

// invert one complete tuple (ReversibleHashGroup::invert, hash.cpp:77-112):
// assignments v = v0, v0 + vstep, ... of the uncovered address bits (a warp
// splits them across lanes)
__device__ void invert_tuple(const DetectParams& P, ReconCounters* C, const uint32_t* cols,
                             uint64_t v0 = 0, uint64_t vstep = 1) {
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
    if (!match) continue;
    const unsigned long long idx = atomicAdd(&C->n_cand, 1ull);
    if (idx < P.cand_cap) P.cands[idx] = Candidate{cand, 0};
    else C->truncated = 1;
  }
}

// Overlap tables for rows 2..r-1. Common case (few hot columns): every CTA
// builds a private copy in shared memory, u32 entries = col + 1 (0 = empty),
// so the depth-first lookups never leave the SM. Otherwise one copy in
// global memory, u64 entries tagged with the launch generation.
constexpr uint32_t kSmemTable = 32768;  // u32 entries of shared memory (128 KB)
constexpr size_t kDynSmem = kSmemTable * sizeof(uint32_t);

struct Tables {
  bool smem;
  const uint32_t* s;                // shared-memory tables
  uint32_t bits[kMaxRows];          // per row (smem) / common (global)
  uint32_t off[kMaxRows];           // smem row offsets
  const unsigned long long* gtab;   // global tables
  uint64_t gstride;
  uint32_t gen;
};

__device__ __forceinline__ uint32_t smem_bits(uint64_t n) {
  uint32_t b = 5;
  while ((1ull << b) < 2 * n) ++b;
  return b;
}

// probe row L from position *slot for the next column with masked key;
// returns col + 1, or 0 when the probe sequence ends
__device__ __forceinline__ uint32_t table_next(const Tables& t, uint32_t L, uint32_t key,
                                               uint32_t ov, uint32_t* slot) {
  const uint32_t mask = (1u << t.bits[L]) - 1;
  while (true) {
    uint32_t e;
    if (t.smem) {
      e = t.s[t.off[L] + *slot];
    } else {
      const unsigned long long g = __ldcg(t.gtab + (L - 2) * t.gstride + *slot);
      e = static_cast<uint32_t>(g >> 32) == t.gen ? static_cast<uint32_t>(g) : 0u;
    }
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

__device__ void phase_reconstruct(const DetectParams& P, ReconCounters* C, const uint64_t* n,
                                  const Tables& t, unsigned* abort,
                                  unsigned long long* cta_stage, uint32_t* q_s, unsigned* q_n) {
  const GroupDev& g = P.g;
  const uint32_t r = g.r;
  const uint64_t cols = 1ull << g.q;
  const uint64_t tid = static_cast<uint64_t>(threadIdx.x) * gridDim.x + blockIdx.x;
  const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n1 = n[1];
  const uint64_t pairs = n[0] * n1;
  uint32_t tup[kMaxRows];
  uint32_t slot[kMaxRows];  // probe position per level
  uint32_t key[kMaxRows];
  for (uint64_t p = tid; p < pairs; p += nthreads) {
    if (*reinterpret_cast<volatile unsigned*>(abort)) break;  // overflow seen elsewhere
    const uint64_t a = (p | n1) >> 32 ? p / n1
                                      : static_cast<uint32_t>(p) / static_cast<uint32_t>(n1);
    const uint64_t b = p - a * n1;
    tup[0] = __ldcg(P.hot_cols + a);
    tup[1] = __ldcg(P.hot_cols + cols + b);
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
      if (atomicAdd(&cta_stage[L + 1], 1ull) >= P.tuple_cap) atomicExch(abort, 1u);
      if (L + 1 == r) {
        // complete tuple: queue it for a warp-parallel inversion
        const unsigned qi = r <= kQueueWidth ? atomicAdd(q_n, 1u) : kQueue;
        if (qi < kQueue) {
          for (uint32_t x = 0; x < r; ++x) q_s[qi * kQueueWidth + x] = tup[x];
        } else {
          invert_tuple(P, C, tup);
        }
      } else {
        ++L;
        key[L] = ((tup[L - 1] ^ tup[0]) >> g.delta) ^ m0;
        slot[L] = table_slot(key[L], t.bits[L]);
      }
    }
  }
  __syncthreads();
  const unsigned nq = min(*q_n, kQueue);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (unsigned t2 = warp; t2 < nq; t2 += blockDim.x >> 5)
    invert_tuple(P, C, q_s + t2 * kQueueWidth, lane, 32);
  if (threadIdx.x >= 3 && threadIdx.x <= r && cta_stage[threadIdx.x])
    atomicAdd(&C->stage[threadIdx.x], cta_stage[threadIdx.x]);
}

// ---------------------------------------------------------------- phase C
constexpr uint32_t kUsleChunk = 4096;  // slots per work item

__device__ void phase_usle(const DetectParams& P, uint64_t n, uint32_t* red, uint64_t* off_s) {
  const SleaDev& le = P.le;
  if (n > P.cand_cap) n = P.cand_cap;
  const uint32_t chunks = (le.eta + kUsleChunk - 1) / kUsleChunk;
  const uint64_t items = n * chunks;
  const bool vec = (le.eta & 3) == 0 && (le.delta & 3) == 0 && (le.row_len & 3) == 0;
  for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const uint64_t c = it / chunks;
    const uint32_t z0 = static_cast<uint32_t>(it - c * chunks) * kUsleChunk;
    const uint32_t z1 = min(le.eta, z0 + kUsleChunk);
    const uint32_t aip = __ldcg(&P.cands[c].aip);
    __syncthreads();
    if (threadIdx.x < le.r) {
      const uint32_t col = static_cast<uint32_t>(seeded(P.lh[threadIdx.x], aip)) & le.col_mask;
      off_s[threadIdx.x] = threadIdx.x * le.row_len + static_cast<uint64_t>(col) * le.delta;
    }
    __syncthreads();
    uint32_t cnt = 0;
    if (vec) {
      for (uint32_t z = z0 + 4 * threadIdx.x; z < z1; z += 4 * blockDim.x) {
        uint32_t m0 = 1, m1 = 1, m2 = 1, m3 = 1;
        for (uint32_t i = 0; i < le.r; ++i) {
          const uint4 v = ld4(le.cells + off_s[i] + z);
          m0 &= v.x > P.le_lo;
          m1 &= v.y > P.le_lo;
          m2 &= v.z > P.le_lo;
          m3 &= v.w > P.le_lo;
        }
        cnt += m0 + m1 + m2 + m3;
      }
    } else {
      for (uint32_t z = z0 + threadIdx.x; z < z1; z += blockDim.x) {
        uint32_t m = 1;
        for (uint32_t i = 0; i < le.r; ++i) m &= le.cells[off_s[i] + z] > P.le_lo;
        cnt += m;
      }
    }
    const uint32_t t = block_sum(cnt, red);
    if (threadIdx.x == 0 && t) atomicAdd(&P.cands[c].weight, t);
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_detect(DetectParams P) {
  __shared__ uint32_t red[32];
  __shared__ uint64_t off_s[kMaxRows];
  __shared__ uint64_t n[kMaxRows];
  __shared__ bool last;
  __shared__ Tables tabs;
  __shared__ unsigned long long cta_stage[kMaxRows + 1];
  __shared__ uint32_t q_s[kQueue * kQueueWidth];
  __shared__ unsigned q_n;
  extern __shared__ uint32_t stab[];  // kSmemTable entries
  if (threadIdx.x <= kMaxRows) cta_stage[threadIdx.x] = 0;
  if (threadIdx.x == 0) q_n = 0;
  DetectScratch* S = P.scratch;
  const uint32_t gen = S->gen + 1;  // table generation of this launch (never 0)
  const uint32_t r = P.g.r;

  stamp_phase(S, 0);
  phase_counts(P, S, red);
  stamp_phase(S, 1);
  grid_barrier(P.bar);
  stamp_phase(S, 2);

  // ---- phase B: reconstruction (identical decisions in every CTA)
  if (threadIdx.x < r) n[threadIdx.x] = __ldcg(&S->hot_counts[threadIdx.x]);
  __syncthreads();
  bool empty = false;
  for (uint32_t i = 0; i < r; ++i) empty |= n[i] == 0;
  const uint64_t seed_work = empty ? 0 : n[0] * n[1] * n[2];
  const bool cap_overflow = !empty && seed_work > P.work_cap;
  if (!empty && !cap_overflow) {
    const uint64_t cols = 1ull << P.g.q;
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
    }
    __syncthreads();
    if (tabs.smem) {
      // private copy in every CTA: a few hundred inserts, no grid barrier
      const uint32_t total = tabs.off[r - 1] + (1u << tabs.bits[r - 1]);
      for (uint32_t i = threadIdx.x; i < total; i += blockDim.x) stab[i] = 0u;
      __syncthreads();
      for (uint32_t L = 2; L < r; ++L) {
        const uint32_t mask = (1u << tabs.bits[L]) - 1;
        for (uint64_t j = threadIdx.x; j < n[L]; j += blockDim.x) {
          const uint32_t col = __ldcg(P.hot_cols + L * cols + j);
          uint32_t i = table_slot(col & P.g.overlap_mask, tabs.bits[L]);
          while (atomicCAS(&stab[tabs.off[L] + i], 0u, col + 1u) != 0u) i = (i + 1) & mask;
        }
      }
      __syncthreads();
    } else {
      // one global copy, generation tagged, then everyone waits for it
      const uint64_t gt = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
      const uint64_t gn = static_cast<uint64_t>(gridDim.x) * blockDim.x;
      for (uint32_t L = 2; L < r; ++L)
        for (uint64_t j = gt; j < n[L]; j += gn) {
          const uint32_t col = __ldcg(P.hot_cols + L * cols + j);
          table_insert(P.table + (L - 2) * P.table_stride, P.table_bits, gen,
                       col & P.g.overlap_mask, col);
        }
      grid_barrier(P.bar);
    }
    phase_reconstruct(P, &S->cnt, n, tabs, &S->abort, cta_stage, q_s, &q_n);
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x < 256) S->arrive_ns[blockIdx.x] = globaltimer();
  stamp_phase(S, 3);
  grid_barrier(P.bar);
  stamp_phase(S, 4);

  // ---- phase C: USLE weights of every candidate (skipped on overflow, whose
  // report carries no candidates)
  const bool aborted = __ldcg(&S->abort) != 0;
  if (!empty && !cap_overflow && !aborted) phase_usle(P, __ldcg(&S->cnt.n_cand), red, off_s);
  stamp_phase(S, 5);

  // ---- the last CTA to finish publishes the record and resets the scratch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&S->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  WinResult* R = P.out;
  const uint64_t nc = __ldcg(&S->cnt.n_cand);
  if (threadIdx.x == 0) {
    S->phase_ns[6] = globaltimer();
    for (uint32_t i = 0; i < r; ++i) R->hot_counts[i] = n[i];
    for (uint32_t i = 0; i < P.le.r; ++i) R->row_weights[i] = __ldcg(&S->row_weights[i]);
    R->seed_work = seed_work;
    for (uint32_t i = 0; i <= kMaxRows; ++i) R->stage_count[i] = __ldcg(&S->cnt.stage[i]);
    R->n_candidates = nc;
    R->empty = empty;
    // overflow exactly as the reference's caps decide it, from the counts
    bool ov = cap_overflow || aborted;
    if (!empty && !ov) {
      uint64_t checked = seed_work;
      for (uint32_t row = 3; row <= r && !ov; ++row) {
        const uint64_t cnt = R->stage_count[row];
        if (cnt > P.tuple_cap) ov = true;
        else if (row < r) {
          const uint64_t work = cnt * n[row];
          if (checked + work > P.work_cap) ov = true;
          checked += work;
        }
      }
    }
    R->overflow = ov;
    R->cand_truncated = __ldcg(&S->cnt.truncated) != 0;
  }
  __syncthreads();
  const uint64_t pre = (R->overflow || empty) ? 0 : min(min(nc, P.cand_cap), P.host_prefix);
  for (uint64_t i = threadIdx.x; i < pre; i += blockDim.x) P.host_cands[i] = P.cands[i];
  // reset for the next launch (nothing reads the scratch any more)
  for (uint32_t i = threadIdx.x; i < kMaxRows; i += blockDim.x) {
    S->hot_counts[i] = 0;
    S->row_weights[i] = 0;
  }
  for (uint32_t i = threadIdx.x; i <= kMaxRows; i += blockDim.x) S->cnt.stage[i] = 0;
  if (threadIdx.x == 0) {
    S->cnt.n_cand = 0;
    S->cnt.truncated = 0;
    S->abort = 0;
    S->done = 0;
    S->gen = gen;
  }
  __threadfence_system();
}

}  // namespace

int detect_grid(int device) {
  int per_sm = 0, sms = 0;
  cudaFuncSetAttribute(k_detect, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(kDynSmem));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_detect, kThreads, kDynSmem);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return std::max(1, std::min(per_sm, 1)) * sms;
}

cudaError_t detect(const DetectParams& P, int grid, cudaStream_t st) {
  DetectParams p = P;
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_detect), dim3(grid), dim3(kThreads),
                                     args, kDynSmem, st);
}

}  // namespace dev
}  // namespace srlg
