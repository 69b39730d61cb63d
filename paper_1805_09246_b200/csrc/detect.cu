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

#include "scan_device.cuh"
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
// A1: RSRA hot columns. Thread per SRE; a warp covers 32 consecutive SREs of
// one row when 2^q >= 32, so one aggregated atomic appends its hot columns.
__device__ void phase_rsra(const DetectParams& P, DetectScratch* S, uint32_t rs_lo) {
  const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t gsize = static_cast<uint64_t>(gridDim.x) * blockDim.x;
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
        w = count_gt4(ld4(p), rs_lo) + count_gt4(ld4(p + 4), rs_lo);
      } else if ((rs.eta & 3) == 0) {
        for (uint32_t z = 0; z < rs.eta; z += 4) w += count_gt4(ld4(p + z), rs_lo);
      } else {
        for (uint32_t z = 0; z < rs.eta; ++z) w += p[z] > rs_lo;
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
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// A2: SLEA inside counts per row, run by `nw` warps (warp index `wid`), 4 x
// uint4 in flight per lane; counts accumulate per CTA in `row_cnt` (shared).
// When rows are 16 B aligned (row_len % 4 == 0, the paper geometry) the same
// pass writes a 1-bit-per-cell "inside" bitmap that phase C reads instead of
// the stamps (32x fewer bytes per candidate).
__device__ void phase_slea(const DetectParams& P, uint64_t wid, uint64_t nw, unsigned* row_cnt,
                           uint32_t le_lo) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t gtid = wid * 32 + lane;
  const uint64_t gsize = nw * 32;
  const SleaDev& le = P.le;
  if (P.le_bits) {
    const uint64_t nv = le.row_len / 4;             // uint4 per row
    const uint64_t nwv = (nv + 31) & ~uint64_t(31);  // warp-uniform trip count
    for (uint32_t row = 0; row < le.r; ++row) {
      const uint32_t* vb = le.cells + row * le.row_len;
      uint32_t* bits = P.le_bits + row * P.le_bits_row_words;
      uint32_t cnt = 0;
      for (uint64_t v = gtid; v < nwv; v += 4 * gsize) {
        uint4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t vu = v + u * gsize;
          x[u] = vu < nv ? ld4(vb + 4 * vu) : make_uint4(0, 0, 0, 0);  // 0 is never inside
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint64_t vu = v + u * gsize;
          if (vu >= nwv) break;  // warp-uniform
          const uint32_t nib = (x[u].x > le_lo) | (x[u].y > le_lo) << 1 |
                               (x[u].z > le_lo) << 2 | (x[u].w > le_lo) << 3;
          cnt += __popc(nib);
          uint32_t word = nib << (4 * (lane & 7));  // 8 lanes x 4 cells = one word
          word |= __shfl_xor_sync(0xFFFFFFFFu, word, 1);
          word |= __shfl_xor_sync(0xFFFFFFFFu, word, 2);
          word |= __shfl_xor_sync(0xFFFFFFFFu, word, 4);
          if ((lane & 7) == 0) bits[vu / 8] = word;
        }
      }
      cnt = warp_sum(cnt);
      if (lane == 0 && cnt) atomicAdd(&row_cnt[row], cnt);
    }
    return;
  }
  for (uint32_t row = 0; row < le.r; ++row) {
    const uint32_t* base = le.cells + row * le.row_len;
    uint32_t cnt = 0;
    uint64_t head = 0;
    if (((row * le.row_len) & 3) != 0) {  // misaligned row start: scalar head
      head = 4 - ((row * le.row_len) & 3);
      if (head > le.row_len) head = le.row_len;
      if (gtid < head) cnt += base[gtid] > le_lo;
    }
    const uint64_t nv = (le.row_len - head) / 4;
    const uint32_t* vb = base + head;
    uint64_t v = gtid;
    for (; v + 3 * gsize < nv; v += 4 * gsize) {
      const uint4 a = ld4(vb + 4 * v), b = ld4(vb + 4 * (v + gsize));
      const uint4 c = ld4(vb + 4 * (v + 2 * gsize)), d = ld4(vb + 4 * (v + 3 * gsize));
      cnt += count_gt4(a, le_lo) + count_gt4(b, le_lo) + count_gt4(c, le_lo) +
             count_gt4(d, le_lo);
    }
    for (; v < nv; v += gsize) cnt += count_gt4(ld4(vb + 4 * v), le_lo);
    for (uint64_t x = head + 4 * nv + gtid; x < le.row_len; x += gsize) cnt += base[x] > le_lo;
    cnt = warp_sum(cnt);
    if (lane == 0 && cnt) atomicAdd(&row_cnt[row], cnt);
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
// 4096 u32 entries (16 KB): rows 2..r-1 of the paper geometry need ~768 at a
// typical slide; more hot columns fall back to the global tables. Kept small
// so the detect kernel and the scan share one L1/shared carveout (a carveout
// switch between the two launches costs several microseconds per slide).
constexpr uint32_t kSmemTable = 4096;
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

struct DfsCtx {
  const DetectParams* P;
  ReconCounters* C;
  const Tables* t;
  unsigned* abort;
  unsigned long long* cta_stage;
  uint32_t* q_s;
  unsigned* q_n;
  uint32_t m0;
};

// complete tuple: queue it for a warp-parallel inversion
template <int R>
__device__ __forceinline__ void emit_tuple(const DfsCtx& d, const uint32_t (&tup)[R]) {
  const unsigned qi = atomicAdd(d.q_n, 1u);
  if (qi < kQueue) {
#pragma unroll
    for (int x = 0; x < R; ++x) d.q_s[qi * kQueueWidth + x] = tup[x];
  } else {
    invert_tuple(*d.P, d.C, tup);
  }
}

// compile-time depth: the tuple stays in registers (a dynamically indexed
// array would live in local memory, which spills past the L1 left beside the
// shared-memory tables)
template <int L, int R>
__device__ __forceinline__ void dfs(const DfsCtx& d, uint32_t (&tup)[R]) {
  const GroupDev& g = d.P->g;
  const uint32_t key = ((tup[L - 1] ^ tup[0]) >> g.delta) ^ d.m0;
  uint32_t slot = table_slot(key, d.t->bits[L]);
  while (true) {
    const uint32_t e = table_next(*d.t, L, key, g.overlap_mask, &slot);
    if (e == 0) return;
    tup[L] = e - 1;
    // a CTA-local count above tuple_cap proves the global one is: the
    // reference overflows, so everyone may stop
    if (atomicAdd(&d.cta_stage[L + 1], 1ull) >= d.P->tuple_cap) atomicExch(d.abort, 1u);
    if constexpr (L + 1 == R) {
      emit_tuple<R>(d, tup);
    } else {
      dfs<L + 1, R>(d, tup);
    }
  }
}

template <int R>
__device__ void dfs_pairs(DfsCtx d, const uint64_t* n) {
  const DetectParams& P = *d.P;
  const uint64_t cols = 1ull << P.g.q;
  const uint64_t tid = static_cast<uint64_t>(threadIdx.x) * gridDim.x + blockIdx.x;
  const uint64_t nthreads = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n1 = n[1];
  const uint64_t pairs = n[0] * n1;
  for (uint64_t p = tid; p < pairs; p += nthreads) {
    if (*reinterpret_cast<volatile unsigned*>(d.abort)) break;
    const uint64_t a = (p | n1) >> 32 ? p / n1
                                      : static_cast<uint32_t>(p) / static_cast<uint32_t>(n1);
    uint32_t tup[R];
    tup[0] = __ldcg(P.hot_cols + a);
    tup[1] = __ldcg(P.hot_cols + cols + (p - a * n1));
    d.m0 = tup[0] & P.g.overlap_mask;
    dfs<2, R>(d, tup);
  }
}

__device__ void phase_reconstruct(const DetectParams& P, ReconCounters* C, const uint64_t* n,
                                  const Tables& t, unsigned* abort,
                                  unsigned long long* cta_stage, uint32_t* q_s, unsigned* q_n) {
  const GroupDev& g = P.g;
  const uint32_t r = g.r;
  const DfsCtx d{&P, C, &t, abort, cta_stage, q_s, q_n, 0};
  switch (r) {
    case 3: dfs_pairs<3>(d, n); break;
    case 4: dfs_pairs<4>(d, n); break;
    case 5: dfs_pairs<5>(d, n); break;
    case 6: dfs_pairs<6>(d, n); break;
    case 7: dfs_pairs<7>(d, n); break;
    case 8: dfs_pairs<8>(d, n); break;
    default: break;
  }
  if (r <= 8) return;
  // r > 8: iterative depth-first walk with the state in local memory
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
        invert_tuple(P, C, tup);
      } else {
        ++L;
        key[L] = ((tup[L - 1] ^ tup[0]) >> g.delta) ^ m0;
        slot[L] = table_slot(key[L], t.bits[L]);
      }
    }
  }
}

// after a __syncthreads: invert the CTA's queued tuples (a warp per tuple)
// and publish the CTA's stage counts
__device__ void finish_reconstruct(const DetectParams& P, ReconCounters* C,
                                   const unsigned long long* cta_stage, const uint32_t* q_s,
                                   unsigned q_n) {
  const unsigned nq = min(q_n, kQueue);
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (unsigned t2 = warp; t2 < nq; t2 += blockDim.x >> 5)
    invert_tuple(P, C, q_s + t2 * kQueueWidth, lane, 32);
  if (threadIdx.x >= 3 && threadIdx.x <= P.g.r && cta_stage[threadIdx.x])
    atomicAdd(&C->stage[threadIdx.x], cta_stage[threadIdx.x]);
}

// ---------------------------------------------------------------- phase C
constexpr uint32_t kUsleChunk = 4096;  // slots per work item

__device__ void phase_usle(const DetectParams& P, uint64_t n, uint32_t* red, uint64_t* off_s,
                           uint32_t le_lo) {
  const SleaDev& le = P.le;
  if (n > P.cand_cap) n = P.cand_cap;
  if (P.le_bits) {
    // bitmap form: a warp per candidate; output word w holds slots
    // [32w, 32w+32) = the AND over rows of the row bitmap at bit offset
    // col_i*delta' + 32w (funnel shift across the word boundary)
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t warp = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
    const uint32_t words = (le.eta + 31) / 32;
    const uint32_t chunks = (words + 31) / 32;  // a warp item = 32 output words of one candidate
    for (uint64_t item = warp; item < n * chunks; item += nwarps) {
      const uint64_t c = item / chunks;
      const uint32_t w0 = static_cast<uint32_t>(item - c * chunks) * 32;
      const uint32_t aip = __ldcg(&P.cands[c].aip);
      uint64_t off = 0;
      if (lane < le.r)
        off = static_cast<uint64_t>(static_cast<uint32_t>(seeded(P.lh[lane], aip)) & le.col_mask) *
              le.delta;
      uint32_t cnt = 0;
      {
        const uint32_t w = w0 + lane;
        uint32_t acc = 0xFFFFFFFFu;
        for (uint32_t i = 0; i < le.r; ++i) {
          const uint64_t bit = __shfl_sync(0xFFFFFFFFu, off, i) + 32ull * w;
          if (w >= words) continue;
          const uint32_t* row = P.le_bits + i * P.le_bits_row_words;
          const uint32_t lo = __ldcg(row + (bit >> 5));
          const uint32_t hi = (bit & 31) ? __ldcg(row + (bit >> 5) + 1) : 0u;
          acc &= __funnelshift_r(lo, hi, static_cast<uint32_t>(bit & 31));
        }
        if (w < words) {
          const uint32_t valid = le.eta - 32 * w;
          if (valid < 32) acc &= (1u << valid) - 1;
          cnt += __popc(acc);
        }
      }
      for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
      if (lane == 0 && cnt) atomicAdd(&P.cands[c].weight, cnt);
    }
    return;
  }
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
          m0 &= v.x > le_lo;
          m1 &= v.y > le_lo;
          m2 &= v.z > le_lo;
          m3 &= v.w > le_lo;
        }
        cnt += m0 + m1 + m2 + m3;
      }
    } else {
      for (uint32_t z = z0 + threadIdx.x; z < z1; z += blockDim.x) {
        uint32_t m = 1;
        for (uint32_t i = 0; i < le.r; ++i) m &= le.cells[off_s[i] + z] > le_lo;
        cnt += m;
      }
    }
    const uint32_t t = block_sum(cnt, red);
    if (threadIdx.x == 0 && t) atomicAdd(&P.cands[c].weight, t);
  }
}

// Shared memory of one detection (static part; the overlap tables are the
// dynamic part)
struct DetSmem {
  uint32_t red[32];
  uint64_t off_s[kMaxRows];
  uint64_t n[kMaxRows];
  Tables tabs;
  unsigned long long cta_stage[kMaxRows + 1];
  uint32_t q_s[kQueue * kQueueWidth];
  unsigned q_n;
  unsigned row_cnt[kMaxRows];
  bool last;
};

// Where one window's result goes.
struct WinArgs {
  uint32_t rs_lo, le_lo;
  WinResult* out;          // mapped pinned host memory
  Candidate* host_cands;   // mapped pinned host memory, P.host_prefix entries
  uint32_t* ready;         // mapped flag set after the record (or null)
  Candidate* arena;        // device: candidates beyond the prefix (or null)
  uint64_t arena_cap;
};

// One run_detection (src/window.cpp:36-78) by the whole cooperative grid:
// A1 -> barrier -> (B || A2) -> barrier -> C -> last CTA publishes. Callers
// guarantee every scan of the window's state has completed (kernel start, or
// a grid barrier); nothing after C touches the stamps, so a following scan
// may overlap C.
__device__ void detect_window(const DetectParams& P, const WinArgs& W, DetSmem& sm,
                              uint32_t* stab) {
  DetectScratch* S = P.scratch;
  const uint32_t r = P.g.r;
  if (threadIdx.x <= kMaxRows) sm.cta_stage[threadIdx.x] = 0;
  if (threadIdx.x < kMaxRows) sm.row_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) sm.q_n = 0;
  const uint32_t gen = __ldcg(&S->gen) + 1;  // overlap-table generation (never 0)
  __syncthreads();

  // ---- phase A1: RSRA hot columns (all the reconstruction needs)
  stamp_phase(S, 0);
  phase_rsra(P, S, W.rs_lo);
  stamp_phase(S, 1);
  grid_barrier(P.bar);
  stamp_phase(S, 2);

  // ---- phase B (reconstruction) overlapped with A2 (SLEA row counts and
  // bitmap): the warps that own seed pairs walk them, every other warp
  // streams the SLEA. Decisions are identical in every CTA.
  if (threadIdx.x < r) sm.n[threadIdx.x] = __ldcg(&S->hot_counts[threadIdx.x]);
  __syncthreads();
  const uint64_t* n = sm.n;
  bool empty = false;
  for (uint32_t i = 0; i < r; ++i) empty |= n[i] == 0;
  const uint64_t seed_work = empty ? 0 : n[0] * n[1] * n[2];
  const bool cap_overflow = !empty && seed_work > P.work_cap;
  const bool recon = !empty && !cap_overflow;
  // dfs_pairs maps pair p to thread p / grid of CTA p % grid
  const uint32_t warp = threadIdx.x >> 5;
  const uint32_t nwarps_cta = blockDim.x >> 5;
  uint32_t dfs_warps = 0;
  if (recon) {
    const uint64_t per_cta = (n[0] * n[1] + gridDim.x - 1) / gridDim.x;
    const uint64_t want = (per_cta + 31) / 32;
    dfs_warps = static_cast<uint32_t>(want < nwarps_cta ? want : nwarps_cta);
  }
  Tables& tabs = sm.tabs;
  if (recon) {
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
    if (warp < dfs_warps)
      phase_reconstruct(P, &S->cnt, n, tabs, &S->abort, sm.cta_stage, sm.q_s, &sm.q_n);
  }
  if (warp >= dfs_warps) {
    const uint32_t a2 = nwarps_cta - dfs_warps;
    phase_slea(P, static_cast<uint64_t>(blockIdx.x) * a2 + (warp - dfs_warps),
               static_cast<uint64_t>(gridDim.x) * a2, sm.row_cnt, W.le_lo);
  }
  __syncthreads();
  if (dfs_warps == nwarps_cta)  // no warp was free for the SLEA: stream it now
    phase_slea(P, static_cast<uint64_t>(blockIdx.x) * nwarps_cta + warp,
               static_cast<uint64_t>(gridDim.x) * nwarps_cta, sm.row_cnt, W.le_lo);
  if (recon) finish_reconstruct(P, &S->cnt, sm.cta_stage, sm.q_s, sm.q_n);
  __syncthreads();
  if (threadIdx.x < P.le.r && sm.row_cnt[threadIdx.x])
    atomicAdd(&S->row_weights[threadIdx.x],
              static_cast<unsigned long long>(sm.row_cnt[threadIdx.x]));
  stamp_phase(S, 3);
  grid_barrier(P.bar);
  stamp_phase(S, 4);

  // ---- phase C: USLE weights of every candidate (skipped on overflow, whose
  // report carries no candidates)
  const bool aborted = __ldcg(&S->abort) != 0;
  const uint64_t nc = __ldcg(&S->cnt.n_cand);
  if (recon && !aborted) phase_usle(P, nc, sm.red, sm.off_s, W.le_lo);
  stamp_phase(S, 5);

  // ---- the last CTA to finish publishes the record and resets the scratch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    sm.last = atomicAdd(&S->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!sm.last) return;
  __threadfence();
  WinResult* R = W.out;
  __shared__ uint64_t tail_off;
  __shared__ bool ov_s;
  if (threadIdx.x == 0) {
    S->phase_ns[6] = globaltimer();
    R->t_begin = __ldcg(&S->phase_ns[0]);
    R->t_end = S->phase_ns[6];
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
    ov_s = ov;
    bool trunc = __ldcg(&S->cnt.truncated) != 0;
    // candidates beyond the host prefix go to the device arena (engine runs)
    tail_off = ~0ull;
    const uint64_t kept = min(nc, P.cand_cap);
    if (!ov && !empty && W.arena && kept > P.host_prefix) {
      const uint64_t tail = kept - P.host_prefix;
      const unsigned long long off = atomicAdd(&S->arena_used, static_cast<unsigned long long>(tail));
      if (off + tail <= W.arena_cap) tail_off = off;
      else trunc = true;
    }
    R->tail_offset = tail_off;
    R->cand_truncated = trunc;
  }
  __syncthreads();
  const uint64_t kept = min(nc, P.cand_cap);
  const uint64_t pre = (ov_s || empty) ? 0 : min(kept, P.host_prefix);
  for (uint64_t i = threadIdx.x; i < pre; i += blockDim.x) W.host_cands[i] = P.cands[i];
  if (tail_off != ~0ull)
    for (uint64_t i = pre + threadIdx.x; i < kept; i += blockDim.x)
      W.arena[tail_off + i - pre] = P.cands[i];
  // reset for the next detection (nothing reads the scratch any more)
  for (uint32_t i = threadIdx.x; i < kMaxRows; i += blockDim.x) {
    S->hot_counts[i] = 0;
    S->row_weights[i] = 0;
  }
  for (uint32_t i = threadIdx.x; i <= kMaxRows; i += blockDim.x) S->cnt.stage[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    S->cnt.n_cand = 0;
    S->cnt.truncated = 0;
    S->abort = 0;
    S->done = 0;
    S->gen = gen;
    __threadfence_system();
    if (W.ready) *reinterpret_cast<volatile uint32_t*>(W.ready) = 1u;
  }
}

__global__ void __launch_bounds__(kThreads, 1) k_detect(DetectParams P) {
  __shared__ DetSmem sm;
  extern __shared__ uint32_t stab[];  // kSmemTable entries
  const WinArgs W{P.rs_lo, P.le_lo, P.out, P.host_cands, nullptr, nullptr, 0};
  detect_window(P, W, sm, stab);
}

// The persistent engine: a whole batch of slices in one cooperative launch.
// Scan ops stamp their packets (red.max: consecutive slices may overlap, the
// larger stamp wins); a detect op waits for every earlier scan at a grid
// barrier, runs detect_window and flags its ring slot; the next scan overlaps
// its phase C. The host computes every op's stamps and window lows exactly as
// WindowEngine would advance its clocks (capi.cu).
template <int ROWS>
__global__ void __launch_bounds__(kThreads, 1) k_engine(DetectParams P, const EngineOp* ops,
                                                        uint32_t n_ops, const srlg_pair* pairs,
                                                        EngineRing ring) {
  __shared__ DetSmem sm;
  extern __shared__ uint32_t stab[];
  const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t gsize = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  if (gtid == 0) P.scratch->arena_used = 0;  // read only after a grid barrier
  for (uint32_t o = 0; o < n_ops; ++o) {
    const EngineOp op = ops[o];
    if (op.kind == 0) {
      uint64_t i = op.begin + gtid;
      for (; i + gsize < op.end; i += 2 * gsize) {
        const uint2 a = ld_pair_stream(pairs + i), b = ld_pair_stream(pairs + i + gsize);
        rsra_update<kStoreRedMax>(P.rs, op.rs_now, a.x, a.y);
        slea_update<kStoreRedMax, ROWS>(P.le, P.lh, op.le_now, a.x, a.y);
        rsra_update<kStoreRedMax>(P.rs, op.rs_now, b.x, b.y);
        slea_update<kStoreRedMax, ROWS>(P.le, P.lh, op.le_now, b.x, b.y);
      }
      for (; i < op.end; i += gsize) {
        const uint2 a = ld_pair_stream(pairs + i);
        rsra_update<kStoreRedMax>(P.rs, op.rs_now, a.x, a.y);
        slea_update<kStoreRedMax, ROWS>(P.le, P.lh, op.le_now, a.x, a.y);
      }
    } else {
      grid_barrier(P.bar);
      const WinArgs W{op.rs_lo, op.le_lo, ring.out + op.window,
                      ring.cands + op.window * P.host_prefix, ring.ready + op.window,
                      ring.arena, ring.arena_cap};
      detect_window(P, W, sm, stab);
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

cudaError_t detect(const DetectParams& P, int grid, cudaStream_t st) {
  DetectParams p = P;
  void* args[] = {&p};
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
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, kDynSmem, st);
}

}  // namespace dev
}  // namespace srlg
