// detect.cu — the per-slide estimate as ONE persistent cooperative kernel.
//
// run_detection (src/window.cpp:36-78) needs, per completed slice:
//   A  hot SREs per row (Rsra::extract_hot, src/rsra.cpp:45-57) and the
//      inside-window count of every SLEA row (Slea::setting_factor,
//      src/slea.cpp:57-61)                       -> one pass over the state
//   B  candidate reconstruction (reconstruct_candidates,
//      src/reconstruct.cpp:32-151 + ReversibleHashGroup::invert,
//      src/hash.cpp:77-112)                      -> tiny, latency bound
//   C  the USLE weight of every candidate (Slea::estimate,
//      src/slea.cpp:103-114)                     -> r' x eta' reads each
// Issued as separate launches these stages are dominated by launch gaps and
// by single-CTA serial work, so they run here as phases of one kernel with a
// grid barrier between them (grid = one CTA per SM, cooperative launch, so
// every CTA is resident). Phase B runs inside CTA 0 when the hot lists are
// small (the common case: ~100 candidates) and spreads over the whole grid
// otherwise. The result record and the first candidates are written straight
// into mapped pinned host memory; the host forms the doubles.
#include <algorithm>

#include "srlg_internal.cuh"

namespace srlg {
namespace dev {
namespace {

constexpr int kThreads = 1024;
constexpr uint64_t kSmallSeedWork = uint64_t{1} << 21;  // single-CTA reconstruction limit
constexpr uint32_t kSmallHot = 8192;                    // hot entries cached in smem

__device__ __forceinline__ uint32_t ld_acquire(const unsigned* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Sense-free grid barrier: the last arriving CTA resets the count and bumps
// the generation. Valid because the launch is cooperative (all CTAs resident).
__device__ void grid_barrier(DetectScratch* s) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire(&s->bar_gen);
    __threadfence();
    if (atomicAdd(&s->bar_count, 1u) == gridDim.x - 1) {
      s->bar_count = 0;
      __threadfence();
      atomicAdd(&s->bar_gen, 1u);
    } else {
      while (ld_acquire(&s->bar_gen) == gen) __nanosleep(64);
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

__device__ __forceinline__ bool consistent(const GroupDev& g, uint32_t b_prev, uint32_t b_cur) {
  return (b_prev >> g.delta) == (b_cur & g.overlap_mask);  // hash.hpp:101-103
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
    if (cols >= 32) {
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, hot);
      if (m) {
        unsigned long long base = 0;
        if (lane == __ffs(m) - 1) base = atomicAdd(&S->hot_counts[row], (unsigned long long)__popc(m));
        base = __shfl_sync(0xFFFFFFFFu, base, __ffs(m) - 1);
        if (hot) {
          const uint32_t off = __popc(m & ((1u << lane) - 1));
          P.hot_cols[row * cols + base + off] = static_cast<uint32_t>(s & (cols - 1));
        }
      }
    } else if (hot) {
      const unsigned long long i = atomicAdd(&S->hot_counts[row], 1ull);
      P.hot_cols[row * cols + i] = static_cast<uint32_t>(s & (cols - 1));
    }
  }
  // SLEA: inside counts per row, 4 x uint4 in flight per thread
  const SleaDev& le = P.le;
  for (uint32_t row = 0; row < le.r; ++row) {
    const uint32_t* base = le.cells + row * le.row_len;
    uint32_t cnt = 0;
    uint64_t head = 0;
    if (((row * le.row_len) & 3) != 0) {
      // misaligned row start: scalar cells up to the next 16 B boundary
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
    if (threadIdx.x == 0 && t) atomicAdd(&S->row_weights[row], (unsigned long long)t);
  }
}

// ---------------------------------------------------------------- phase B
struct Workers {
  uint64_t tid, n;
  bool grid;
};

__device__ __forceinline__ void stage_sync(const Workers& w, DetectScratch* S) {
  if (w.grid) grid_barrier(S);
  else __syncthreads();
}

// reconstruct_candidates over lists h[i] (smem or global), counts n[i]
__device__ void phase_reconstruct(const DetectParams& P, DetectScratch* S, const Workers& w,
                                  const uint32_t* const* h, const uint64_t* n) {
  const GroupDev& g = P.g;
  const uint32_t r = g.r;
  // seed over rows 0..2 (reconstruct.cpp:53-92)
  {
    const uint64_t pairs = n[0] * n[1];
    for (uint64_t p = w.tid; p < pairs; p += w.n) {
      const uint64_t a = p / n[1], b = p - a * n[1];
      const uint32_t he0 = h[0][a], he1 = h[1][b];
      const uint32_t key = (he1 ^ he0) >> g.delta;
      const uint32_t m0 = he0 & g.overlap_mask;
      for (uint64_t c = 0; c < n[2]; ++c) {
        const uint32_t he2 = h[2][c];
        if (((he2 & g.overlap_mask) ^ m0) != key) continue;
        const unsigned long long idx = atomicAdd(&S->stage_count[3], 1ull);
        if (idx < P.tuple_cap) {
          uint32_t* t = P.tuples_a + idx * r;
          t[0] = he0;
          t[1] = he1;
          t[2] = he2;
        }
      }
    }
  }
  stage_sync(w, S);
  const uint32_t* in = P.tuples_a;
  uint32_t* out = P.tuples_b;
  uint64_t checked = n[0] * n[1] * n[2];
  for (uint32_t row = 3; row < r; ++row) {
    const uint64_t count = *reinterpret_cast<volatile unsigned long long*>(&S->stage_count[row]);
    if (count > P.tuple_cap) return;  // overflow: decided by the caller
    const uint64_t work = count * n[row];
    if (checked + work > P.work_cap) return;
    checked += work;
    for (uint64_t t = w.tid; t < count; t += w.n) {
      const uint32_t* tup = in + t * r;
      const uint32_t he0 = tup[0];
      const uint32_t key = (tup[row - 1] ^ he0) >> g.delta;
      const uint32_t m0 = he0 & g.overlap_mask;
      for (uint64_t j = 0; j < n[row]; ++j) {
        const uint32_t he = h[row][j];
        if (((he & g.overlap_mask) ^ m0) != key) continue;
        const unsigned long long idx = atomicAdd(&S->stage_count[row + 1], 1ull);
        if (idx < P.tuple_cap) {
          uint32_t* o = out + idx * r;
          for (uint32_t x = 0; x < row; ++x) o[x] = tup[x];
          o[row] = he;
        }
      }
    }
    stage_sync(w, S);
    const uint32_t* t = in;
    in = out;
    out = const_cast<uint32_t*>(t);
  }
  const uint64_t kept = *reinterpret_cast<volatile unsigned long long*>(&S->stage_count[r]);
  if (kept > P.tuple_cap) return;
  // invert each surviving tuple; thread per (tuple, free-bit assignment)
  const uint64_t total = kept << g.n_free;
  for (uint64_t x = w.tid; x < total; x += w.n) {
    const uint32_t* cols = in + (x >> g.n_free) * r;
    const uint32_t v = static_cast<uint32_t>(x & ((1ull << g.n_free) - 1));
    const uint32_t c0 = cols[0];
    uint32_t prev = (cols[1] ^ c0) & g.col_mask;
    uint64_t known = static_cast<uint64_t>(prev) << g.delta;
    bool ok = true;
    for (uint32_t i = 2; i < r; ++i) {
      const uint32_t wv = (cols[i] ^ c0) & g.col_mask;
      ok &= consistent(g, prev, wv);
      const uint32_t sh = i * g.delta;
      if (sh < 64) known |= static_cast<uint64_t>(wv) << sh;
      prev = wv;
    }
    if (!ok) continue;
    uint32_t cand = static_cast<uint32_t>(known) & ~g.uncovered;
    for (uint32_t b = 0; b < g.n_free; ++b)
      if (v & (1u << b)) cand |= 1u << g.free_bits[b];
    const uint32_t f0 = static_cast<uint32_t>(seeded(g.h0, cand)) & g.col_mask;
    if (f0 != c0) continue;
    bool match = true;
    for (uint32_t i = 1; i < r && match; ++i) {
      const uint32_t sh = i * g.delta;
      match = (((sh >= 32 ? 0u : cand >> sh) ^ f0) & g.col_mask) == cols[i];
    }
    if (!match) continue;
    const unsigned long long idx = atomicAdd(&S->n_cand, 1ull);
    if (idx < P.cand_cap) P.cands[idx] = Candidate{cand, 0};
    else S->cand_truncated = 1;
  }
}

// ---------------------------------------------------------------- phase C
constexpr uint32_t kUsleChunk = 4096;  // slots per work item

__device__ void phase_usle(const DetectParams& P, DetectScratch* S, uint32_t* red,
                           uint64_t* off_s) {
  const SleaDev& le = P.le;
  uint64_t n = S->n_cand;
  if (n > P.cand_cap) n = P.cand_cap;
  const uint32_t chunks = (le.eta + kUsleChunk - 1) / kUsleChunk;
  const uint64_t items = n * chunks;
  const bool vec = (le.eta & 3) == 0 && (le.delta & 3) == 0 && (le.row_len & 3) == 0;
  for (uint64_t it = blockIdx.x; it < items; it += gridDim.x) {
    const uint64_t c = it / chunks;
    const uint32_t z0 = static_cast<uint32_t>(it - c * chunks) * kUsleChunk;
    const uint32_t z1 = min(le.eta, z0 + kUsleChunk);
    const uint32_t aip = P.cands[c].aip;
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
  __shared__ uint32_t hot_s[kSmallHot];
  __shared__ uint64_t n[kMaxRows];
  __shared__ const uint32_t* h[kMaxRows];
  DetectScratch* S = P.scratch;

  phase_counts(P, S, red);
  grid_barrier(S);

  // ---- phase B: decide the reconstruction mode (identical in every CTA)
  const uint32_t r = P.g.r;
  if (threadIdx.x < r)
    n[threadIdx.x] = *reinterpret_cast<volatile unsigned long long*>(&S->hot_counts[threadIdx.x]);
  __syncthreads();
  bool empty = false;
  uint64_t total_hot = 0;
  for (uint32_t i = 0; i < r; ++i) {
    empty |= n[i] == 0;
    total_hot += n[i];
  }
  const uint64_t seed_work = empty ? 0 : n[0] * n[1] * n[2];
  const bool cap_overflow = !empty && seed_work > P.work_cap;
  int mode = 0;
  if (!empty && !cap_overflow)
    mode = (seed_work <= kSmallSeedWork && total_hot <= kSmallHot) ? 1 : 2;
  const uint64_t cols = 1ull << P.g.q;
  if (mode == 1) {
    if (blockIdx.x == 0) {
      // hot lists into shared memory, then every stage inside this CTA
      uint64_t off = 0;
      for (uint32_t i = 0; i < r; ++i) {
        for (uint64_t j = threadIdx.x; j < n[i]; j += blockDim.x)
          hot_s[off + j] = P.hot_cols[i * cols + j];
        if (threadIdx.x == 0) h[i] = hot_s + off;
        off += n[i];
      }
      __syncthreads();
      phase_reconstruct(P, S, Workers{threadIdx.x, blockDim.x, false}, h, n);
    }
  } else if (mode == 2) {
    if (threadIdx.x < r) h[threadIdx.x] = P.hot_cols + threadIdx.x * cols;
    __syncthreads();
    phase_reconstruct(P, S,
                      Workers{static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x,
                              static_cast<uint64_t>(gridDim.x) * blockDim.x, true},
                      h, n);
  }
  grid_barrier(S);

  // ---- phase C: USLE weights of every candidate
  phase_usle(P, S, red, off_s);

  // ---- the last CTA to finish publishes the record and resets the scratch
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&S->done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  WinResult* R = P.out;
  const uint64_t nc = S->n_cand;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < r; ++i) R->hot_counts[i] = n[i];
    for (uint32_t i = 0; i < P.le.r; ++i) R->row_weights[i] = S->row_weights[i];
    R->seed_work = seed_work;
    for (uint32_t i = 0; i <= kMaxRows; ++i) R->stage_count[i] = S->stage_count[i];
    R->n_candidates = nc;
    R->empty = empty;
    // overflow (reconstruct.cpp:60-63, 97-99, 110-113), recomputed from the
    // final stage counts exactly as the reference's caps decide it
    bool ov = cap_overflow;
    if (!empty && !ov) {
      uint64_t checked = seed_work;
      for (uint32_t row = 3; row <= r && !ov; ++row) {
        if (S->stage_count[row] > P.tuple_cap) ov = true;
        else if (row < r) {
          const uint64_t work = S->stage_count[row] * n[row];
          if (checked + work > P.work_cap) ov = true;
          checked += work;
        }
      }
    }
    R->overflow = ov;
    R->cand_truncated = S->cand_truncated;
  }
  const uint64_t pre = min(min(nc, P.cand_cap), P.host_prefix);
  for (uint64_t i = threadIdx.x; i < pre; i += blockDim.x) P.host_cands[i] = P.cands[i];
  // reset for the next detection (nothing reads the scratch any more)
  for (uint32_t i = threadIdx.x; i < kMaxRows; i += blockDim.x) {
    S->hot_counts[i] = 0;
    S->row_weights[i] = 0;
  }
  for (uint32_t i = threadIdx.x; i <= kMaxRows; i += blockDim.x) S->stage_count[i] = 0;
  if (threadIdx.x == 0) {
    S->n_cand = 0;
    S->cand_truncated = 0;
    S->done = 0;
  }
  __threadfence_system();
}

}  // namespace

int detect_grid(int device) {
  int per_sm = 0, sms = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_detect, kThreads, 0);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  return std::max(1, std::min(per_sm, 1)) * sms;
}

cudaError_t detect(const DetectParams& P, int grid, cudaStream_t st) {
  DetectParams p = P;
  void* args[] = {&p};
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_detect), dim3(grid), dim3(kThreads),
                                     args, 0, st);
}

}  // namespace dev
}  // namespace srlg
