// kernels.cu — sm_100a kernels of the sliding super-point path.
//
//   K1 k_scan           Rsra::update + Slea::update over a packet batch
//                       (src/rsra.cpp:25-33, src/slea.cpp:38-45)
//   K2 k_window_counts  per-SRE inside-window weights -> hot bitmap
//                       (Rsra::extract_hot, src/rsra.cpp:45-57) and per-row
//                       SLEA inside counts (Slea::setting_factor,
//                       src/slea.cpp:57-61)
//      k_hot_compact    ordered hot lists + row weights + seed work
//   K4 k_seed/k_grow/k_invert
//                       reconstruct_candidates (src/reconstruct.cpp:32-151)
//                       and ReversibleHashGroup::invert (src/hash.cpp:77-112)
//   K3 k_usle           fused union + weight of Slea::estimate
//                       (src/slea.cpp:103-114), one CTA per candidate
//   k_export/k_import/k_merge
//                       stamp <-> u16 distance conversion; Rsra/Slea::merge_min
//                       (src/rsra.cpp:77-81) as a stamp max
//
// State is u32 stamps (see srlg_internal.cuh). Within one scan launch every
// record writes the same stamp `now`, and no stored stamp exceeds `now`, so
// the reference's relaxed "store 0 distance" (rsra.cpp:30-32) becomes an
// idempotent store of `now`: a plain store and red.max give identical
// results, and packet order cannot matter.
#include <algorithm>

#include <cub/block/block_scan.cuh>

#include "scan_device.cuh"
#include "srlg_internal.cuh"

namespace srlg {
namespace dev {
namespace {

constexpr int kScanThreads = 256;

// K1. Each thread walks the batch with a grid stride, UNROLL independent
// packets per step so the pair loads of later packets overlap the hashing of
// earlier ones.
template <int MODE, bool DO_RS, bool DO_LE, int ROWS>
__global__ void __launch_bounds__(kScanThreads) k_scan(const srlg_pair* __restrict__ pairs,
                                                       uint64_t n, RsraDev rs, uint32_t rs_now,
                                                       SleaDev le, uint32_t le_now, AnetDev anet,
                                                       unsigned long long* raw_records) {
  __shared__ uint64_t lh_s[kMaxRows];
  if constexpr (DO_LE && ROWS == 0) {
    if (threadIdx.x < le.r) lh_s[threadIdx.x] = le.lh_dev[threadIdx.x];
    __syncthreads();
  }
  constexpr int UNROLL = 4;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (anet.n) {  // raw packets: classify (trace.cpp:111-116) fused into the scan
    if constexpr (!DO_RS) rs.cells = nullptr;
    if constexpr (!DO_LE) le.cells = nullptr;
    uint32_t records = 0;
    for (; i < n; i += stride)
      records += ingest<MODE, ROWS>(rs, le, lh_s, rs_now, le_now, anet, ld_pair_stream(pairs + i));
    if (raw_records) {
      records = __reduce_add_sync(0xFFFFFFFFu, records);
      if ((threadIdx.x & 31) == 0 && records) atomicAdd(raw_records, static_cast<unsigned long long>(records));
    }
    return;
  }
  for (; i + (UNROLL - 1) * stride < n; i += UNROLL * stride) {
    uint2 p[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) p[u] = ld_pair_stream(pairs + i + u * stride);
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      if constexpr (DO_RS) rsra_update<MODE>(rs, rs_now, p[u].x, p[u].y);
      if constexpr (DO_LE) slea_update<MODE, ROWS>(le, lh_s, le_now, p[u].x, p[u].y);
    }
  }
  for (; i < n; i += stride) {
    const uint2 p = ld_pair_stream(pairs + i);
    if constexpr (DO_RS) rsra_update<MODE>(rs, rs_now, p.x, p.y);
    if constexpr (DO_LE) slea_update<MODE, ROWS>(le, lh_s, le_now, p.x, p.y);
  }
}

template <int MODE, bool DO_RS, bool DO_LE>
cudaError_t launch_scan_rows(const srlg_pair* pairs, uint64_t n, const RsraDev& rs,
                             uint32_t rs_now, const SleaDev& le, uint32_t le_now, dim3 grid,
                             cudaStream_t st, const AnetDev& anet, unsigned long long* rr) {
  if (DO_LE && le.r == 5)
    k_scan<MODE, DO_RS, DO_LE, 5><<<grid, kScanThreads, 0, st>>>(pairs, n, rs, rs_now, le, le_now, anet, rr);
  else if (DO_LE && le.r == 3)
    k_scan<MODE, DO_RS, DO_LE, 3><<<grid, kScanThreads, 0, st>>>(pairs, n, rs, rs_now, le, le_now, anet, rr);
  else
    k_scan<MODE, DO_RS, DO_LE, 0><<<grid, kScanThreads, 0, st>>>(pairs, n, rs, rs_now, le, le_now, anet, rr);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_scan_mode(const srlg_pair* pairs, uint64_t n, const RsraDev& rs,
                             uint32_t rs_now, const SleaDev& le, uint32_t le_now, dim3 grid,
                             cudaStream_t st, const AnetDev& anet, unsigned long long* rr) {
  const bool r_on = rs.cells != nullptr, l_on = le.cells != nullptr;
  if (r_on && l_on) return launch_scan_rows<MODE, true, true>(pairs, n, rs, rs_now, le, le_now, grid, st, anet, rr);
  if (r_on) return launch_scan_rows<MODE, true, false>(pairs, n, rs, rs_now, le, le_now, grid, st, anet, rr);
  if (l_on) return launch_scan_rows<MODE, false, true>(pairs, n, rs, rs_now, le, le_now, grid, st, anet, rr);
  return cudaSuccess;
}

// ------------------------------------------------------------------- K2

__device__ __forceinline__ uint32_t count_gt4(uint4 v, uint32_t lo) {
  return (v.x > lo) + (v.y > lo) + (v.z > lo) + (v.w > lo);
}

__device__ __forceinline__ uint4 ld4(const uint32_t* p) {
  return *reinterpret_cast<const uint4*>(p);
}

__global__ void __launch_bounds__(256) k_window_counts(RsraDev rs, uint32_t rs_lo, uint32_t hot_min,
                                                       uint64_t rs_sres, uint32_t rs_blocks,
                                                       SleaDev le, uint32_t le_lo, uint32_t bpr,
                                                       uint64_t chunk, uint32_t* hot_bits,
                                                       uint32_t* partials) {
  if (blockIdx.x < rs_blocks) {
    // RSRA: one SRE (eta stamps) per thread; a warp covers 32 consecutive
    // SREs and ballots one word of the hot bitmap.
    const uint64_t words = (rs_sres + 31) / 32;
    const uint64_t stride = static_cast<uint64_t>(rs_blocks) * blockDim.x;
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
         s < words * 32; s += stride) {
      bool hot = false;
      if (s < rs_sres) {
        const uint32_t* p = rs.cells + s * rs.eta;
        uint32_t w = 0;
        if (rs.eta == 8) {
          w = count_gt4(ld4(p), rs_lo) + count_gt4(ld4(p + 4), rs_lo);
        } else if ((rs.eta & 3) == 0) {
          for (uint32_t z = 0; z < rs.eta; z += 4) w += count_gt4(ld4(p + z), rs_lo);
        } else {
          for (uint32_t z = 0; z < rs.eta; ++z) w += p[z] > rs_lo;
        }
        hot = w >= hot_min;
      }
      const uint32_t bits = __ballot_sync(0xFFFFFFFFu, hot);
      if (lane == 0) hot_bits[s >> 5] = bits;
    }
    return;
  }
  // SLEA: block b covers cells [j*chunk, (j+1)*chunk) of row b / bpr
  const uint32_t b = blockIdx.x - rs_blocks;
  const uint32_t row = b / bpr, j = b % bpr;
  const uint64_t start = j * chunk;
  const uint64_t end = min(start + chunk, le.row_len);
  const uint32_t* base = le.cells + row * le.row_len;
  uint32_t cnt = 0;
  if (start < end) {
    if (((row * le.row_len) & 3) == 0) {
      const uint64_t vend = start + ((end - start) & ~uint64_t(3));
      for (uint64_t x = start + 4ull * threadIdx.x; x < vend; x += 4ull * blockDim.x)
        cnt += count_gt4(ld4(base + x), le_lo);
      for (uint64_t x = vend + threadIdx.x; x < end; x += blockDim.x) cnt += base[x] > le_lo;
    } else {
      for (uint64_t x = start + threadIdx.x; x < end; x += blockDim.x) cnt += base[x] > le_lo;
    }
  }
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
  __shared__ uint32_t ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    partials[b] = t;
  }
}

// Ordered compaction of one row's hot bits with a 1024-thread CTA; lists come
// out ascending like Rsra::extract_hot (rsra.cpp:49-55).
constexpr int kCompactThreads = 1024;

__global__ void __launch_bounds__(kCompactThreads)
    k_hot_compact(const uint32_t* __restrict__ hot_bits, uint32_t q, uint32_t r,
                  const uint32_t* __restrict__ partials, uint32_t le_rows, uint32_t bpr,
                  uint32_t* hot_cols, WinResult* res, uint64_t work_cap) {
  using Scan = cub::BlockScan<uint32_t, kCompactThreads>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ uint32_t total_s;
  const uint64_t cols = 1ull << q;
  for (uint32_t row = 0; row < r; ++row) {
    const uint64_t b0 = static_cast<uint64_t>(row) << q, b1 = b0 + cols;
    const uint64_t w0 = b0 >> 5, w1 = (b1 + 31) >> 5;
    const uint64_t nw = w1 - w0;
    const uint64_t per = (nw + kCompactThreads - 1) / kCompactThreads;
    const uint64_t my0 = w0 + per * threadIdx.x;
    const uint64_t my1 = min(my0 + per, w1);
    auto word = [&](uint64_t w) {
      uint32_t v = hot_bits[w];
      const uint64_t lo = w * 32, hi = lo + 32;
      if (lo < b0) v &= ~0u << (b0 - lo);
      if (hi > b1) v &= (b1 - lo) >= 32 ? ~0u : ((1u << (b1 - lo)) - 1);
      return v;
    };
    uint32_t c = 0;
    for (uint64_t w = my0; w < my1; ++w) c += __popc(word(w));
    uint32_t off, total;
    Scan(scan_tmp).ExclusiveSum(c, off, total);
    if (threadIdx.x == 0) total_s = total;
    uint32_t* out = hot_cols + row * cols;
    for (uint64_t w = my0; w < my1; ++w) {
      uint32_t v = word(w);
      while (v) {
        const uint32_t bit = __ffs(v) - 1;
        v &= v - 1;
        out[off++] = static_cast<uint32_t>(w * 32 + bit - b0);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) res->hot_counts[row] = total_s;
    __syncthreads();
  }
  if (threadIdx.x < le_rows) {
    uint64_t s = 0;
    for (uint32_t j = 0; j < bpr; ++j) s += partials[threadIdx.x * bpr + j];
    res->row_weights[threadIdx.x] = s;
  }
  if (threadIdx.x == 0) {
    bool empty = false;
    for (uint32_t i = 0; i < r; ++i) empty |= res->hot_counts[i] == 0;
    const uint64_t sw = empty ? 0 : res->hot_counts[0] * res->hot_counts[1] * res->hot_counts[2];
    res->seed_work = sw;
    res->overflow = (!empty && sw > work_cap) ? 1u : 0u;
    for (uint32_t i = 0; i <= kMaxRows; ++i) res->stage_count[i] = 0;
    res->n_candidates = 0;
    res->cand_truncated = 0;
    res->checked = 0;
    res->empty = empty ? 1u : 0u;  // "some row empty": nothing to reconstruct
  }
}

// ------------------------------------------------------------------- K4

__device__ __forceinline__ bool windows_consistent(const GroupDev& g, uint32_t b_prev,
                                                   uint32_t b_cur) {
  return (b_prev >> g.delta) == (b_cur & g.overlap_mask);  // hash.hpp:101-103
}

// seed tuples over rows 0..2 (reconstruct.cpp:53-92)
__global__ void __launch_bounds__(256) k_seed(GroupDev g, const uint32_t* __restrict__ hot_cols,
                                              WinResult* res, uint32_t* tuples,
                                              uint64_t tuple_cap) {
  if (res->overflow || res->empty) return;
  const uint64_t cols = 1ull << g.q;
  const uint32_t* h0 = hot_cols;
  const uint32_t* h1 = hot_cols + cols;
  const uint32_t* h2 = hot_cols + 2 * cols;
  const uint64_t n0 = res->hot_counts[0], n1 = res->hot_counts[1], n2 = res->hot_counts[2];
  const uint64_t pairs = n0 * n1;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < pairs;
       p += stride) {
    const uint64_t a = p / n1, b = p - a * n1;
    const uint32_t he0 = h0[a], he1 = h1[b];
    const uint32_t b1 = he1 ^ he0;
    for (uint64_t c = 0; c < n2; ++c) {
      const uint32_t he2 = h2[c];
      if (!windows_consistent(g, b1, he2 ^ he0)) continue;
      const unsigned long long idx =
          atomicAdd(reinterpret_cast<unsigned long long*>(&res->stage_count[3]), 1ull);
      if (idx < tuple_cap) {
        uint32_t* t = tuples + idx * g.r;
        t[0] = he0;
        t[1] = he1;
        t[2] = he2;
      }
    }
  }
}

// overflow test at the start of growth stage `row` (reconstruct.cpp:97-99,
// 60-63 / 110-113): recomputed identically by every block
__device__ __forceinline__ bool stage_overflowed(const WinResult* res, uint32_t row,
                                                 uint64_t tuple_cap, uint64_t work_cap) {
  if (res->overflow || res->empty) return true;
  if (res->stage_count[row] > tuple_cap) return true;
  uint64_t checked = res->seed_work;
  for (uint32_t j = 3; j < row; ++j) checked += res->stage_count[j] * res->hot_counts[j];
  return checked + res->stage_count[row] * res->hot_counts[row] > work_cap;
}

// grow one row (reconstruct.cpp:94-130)
__global__ void __launch_bounds__(256) k_grow(GroupDev g, uint32_t row,
                                              const uint32_t* __restrict__ hot_cols,
                                              WinResult* res, const uint32_t* __restrict__ in,
                                              uint32_t* out, uint64_t tuple_cap,
                                              uint64_t work_cap) {
  if (stage_overflowed(res, row, tuple_cap, work_cap)) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && !res->empty) res->overflow = 1;
    return;
  }
  const uint64_t cols = 1ull << g.q;
  const uint32_t* hr = hot_cols + row * cols;
  const uint64_t count = res->stage_count[row], nr = res->hot_counts[row];
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t t = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < count;
       t += stride) {
    const uint32_t* tup = in + t * g.r;
    const uint32_t he0 = tup[0];
    const uint32_t b_prev = tup[row - 1] ^ he0;
    for (uint64_t j = 0; j < nr; ++j) {
      const uint32_t he = hr[j];
      if (!windows_consistent(g, b_prev, he ^ he0)) continue;
      const unsigned long long idx =
          atomicAdd(reinterpret_cast<unsigned long long*>(&res->stage_count[row + 1]), 1ull);
      if (idx < tuple_cap) {
        uint32_t* o = out + idx * g.r;
        for (uint32_t w = 0; w < row; ++w) o[w] = tup[w];
        o[row] = he;
      }
    }
  }
}

// invert every surviving tuple (reconstruct.cpp:132-150 ->
// ReversibleHashGroup::invert, hash.cpp:77-112); thread per (tuple, free-bit
// assignment)
__global__ void __launch_bounds__(256) k_invert(GroupDev g, WinResult* res,
                                                const uint32_t* __restrict__ tuples,
                                                uint64_t tuple_cap, Candidate* cands,
                                                uint64_t cand_cap) {
  if (res->overflow || res->empty) return;
  if (res->stage_count[g.r] > tuple_cap) {
    if (blockIdx.x == 0 && threadIdx.x == 0) res->overflow = 1;
    return;
  }
  const uint64_t count = res->stage_count[g.r];
  const uint64_t total = count << g.n_free;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t x = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; x < total;
       x += stride) {
    const uint32_t* cols = tuples + (x >> g.n_free) * g.r;
    const uint32_t v = static_cast<uint32_t>(x & ((1ull << g.n_free) - 1));
    const uint32_t c0 = cols[0];
    uint32_t prev = (cols[1] ^ c0) & g.col_mask;
    uint64_t known = static_cast<uint64_t>(prev) << g.delta;
    bool ok = true;
    for (uint32_t i = 2; i < g.r; ++i) {
      const uint32_t w = (cols[i] ^ c0) & g.col_mask;
      ok &= windows_consistent(g, prev, w);
      const uint32_t sh = i * g.delta;
      if (sh < 64) known |= static_cast<uint64_t>(w) << sh;
      prev = w;
    }
    if (!ok) continue;
    uint32_t cand = static_cast<uint32_t>(known) & ~g.uncovered;
    for (uint32_t b = 0; b < g.n_free; ++b)
      if (v & (1u << b)) cand |= 1u << g.free_bits[b];
    // forward(cand) == cols  (hash.cpp:63-69)
    const uint32_t f0 = static_cast<uint32_t>(seeded(g.h0, cand)) & g.col_mask;
    if (f0 != c0) continue;
    bool match = true;
    for (uint32_t i = 1; i < g.r && match; ++i) {
      const uint32_t sh = i * g.delta;
      const uint32_t shifted = sh >= 32 ? 0u : cand >> sh;
      match = ((shifted ^ f0) & g.col_mask) == cols[i];
    }
    if (!match) continue;
    const unsigned long long idx =
        atomicAdd(reinterpret_cast<unsigned long long*>(&res->n_candidates), 1ull);
    if (idx < cand_cap) cands[idx].aip = cand;
    else res->cand_truncated = 1;
  }
}

// ------------------------------------------------------------------- K3

constexpr int kUsleThreads = 256;

// USLE weight = #{z < eta' : every row's stamp at col_i*delta'+z is inside}
// (min over stamps == max over distances, slea.cpp:109-114)
__global__ void __launch_bounds__(kUsleThreads) k_usle(SleaDev le, const uint64_t* __restrict__ lh,
                                                      uint32_t lo, Candidate* cands,
                                                      const WinResult* res, uint64_t n_host,
                                                      uint64_t cand_cap) {
  __shared__ uint64_t off[kMaxRows];
  __shared__ uint32_t ws[kUsleThreads / 32];
  __shared__ uint32_t vec_ok;
  uint64_t n = res ? res->n_candidates : n_host;
  if (n > cand_cap) n = cand_cap;
  for (uint64_t c = blockIdx.x; c < n; c += gridDim.x) {
    const uint32_t aip = cands[c].aip;
    if (threadIdx.x == 0) vec_ok = (le.eta & 3) == 0;
    __syncthreads();
    if (threadIdx.x < le.r) {
      const uint32_t col = static_cast<uint32_t>(seeded(lh[threadIdx.x], aip)) & le.col_mask;
      off[threadIdx.x] = threadIdx.x * le.row_len + static_cast<uint64_t>(col) * le.delta;
      if (off[threadIdx.x] & 3) atomicAnd(&vec_ok, 0u);
    }
    __syncthreads();
    uint32_t cnt = 0;
    if (vec_ok) {
      for (uint32_t z = 4 * threadIdx.x; z < le.eta; z += 4 * blockDim.x) {
        uint32_t m0 = 1, m1 = 1, m2 = 1, m3 = 1;
        for (uint32_t i = 0; i < le.r; ++i) {
          const uint4 v = ld4(le.cells + off[i] + z);
          m0 &= v.x > lo;
          m1 &= v.y > lo;
          m2 &= v.z > lo;
          m3 &= v.w > lo;
        }
        cnt += m0 + m1 + m2 + m3;
      }
    } else {
      for (uint32_t z = threadIdx.x; z < le.eta; z += blockDim.x) {
        uint32_t m = 1;
        for (uint32_t i = 0; i < le.r; ++i) m &= le.cells[off[i] + z] > lo;
        cnt += m;
      }
    }
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xFFFFFFFFu, cnt, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t t = 0;
      for (int w = 0; w < kUsleThreads / 32; ++w) t += ws[w];
      cands[c].weight = t;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------ export / import

__global__ void k_export(const uint32_t* __restrict__ s, uint64_t n, uint32_t now, uint32_t floor,
                         uint16_t* __restrict__ out) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const uint32_t v = s[i];
    uint16_t d = 0xFFFF;
    if (v > floor) {
      const uint32_t age = now - v;
      d = age >= 0xFFFFu ? 0xFFFF : static_cast<uint16_t>(age);
    }
    out[i] = d;
  }
}

__global__ void k_import(const uint16_t* __restrict__ in, uint64_t n, uint32_t now,
                         uint32_t* __restrict__ s) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const uint16_t d = in[i];
    s[i] = d == 0xFFFF ? 0u : now - d;
  }
}

// merge_min on distances == max on stamps, with b rebased onto a's clock
__global__ void k_merge(uint32_t* __restrict__ a, const uint32_t* __restrict__ b, uint64_t n,
                        uint32_t now_a, uint32_t floor_a, uint32_t now_b, uint32_t floor_b) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    uint32_t va = a[i];
    if (va <= floor_a) va = 0;
    const uint32_t vb = b[i];
    uint32_t rb = 0;
    if (vb > floor_b) {
      const uint32_t age = now_b - vb;
      if (age < 0xFFFFu) rb = now_a - age;
    }
    a[i] = va > rb ? va : rb;
  }
}

// Multi-GPU merge, root side: after the NCCL max-reduce of every rank's u8
// dirty map, a cell marked by any rank in this slice gets the slice's stamp
// (exactly what a single node's scan would have stored), and the map is
// cleared for the next slice. Cells [0, n_rs) are RSRA, the rest SLEA.
__global__ void k_apply_marks(uint8_t* __restrict__ dirty, uint64_t n_rs, uint32_t* __restrict__ rs,
                              uint32_t rs_now, uint64_t n_le, uint32_t* __restrict__ le,
                              uint32_t le_now) {
  const uint64_t n = n_rs + n_le;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t v = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; v * 16 < n;
       v += stride) {
    uint4 m = v * 16 + 16 <= n ? reinterpret_cast<const uint4*>(dirty)[v] : make_uint4(0, 0, 0, 0);
    if (v * 16 + 16 > n)
      for (uint64_t i = v * 16; i < n; ++i)
        if (dirty[i]) reinterpret_cast<uint8_t*>(&m)[i - v * 16] = 1;
    if (!(m.x | m.y | m.z | m.w)) continue;
    const uint8_t* b = reinterpret_cast<const uint8_t*>(&m);
    for (int j = 0; j < 16; ++j) {
      if (!b[j]) continue;
      const uint64_t i = v * 16 + j;
      if (i < n_rs) rs[i] = rs_now;
      else if (i < n) le[i - n_rs] = le_now;
    }
    if (v * 16 + 16 <= n) reinterpret_cast<uint4*>(dirty)[v] = make_uint4(0, 0, 0, 0);
    else
      for (uint64_t i = v * 16; i < n; ++i) dirty[i] = 0;
  }
}

int grid_for(uint64_t n, int threads, int cap_blocks) {
  uint64_t b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > static_cast<uint64_t>(cap_blocks)) b = cap_blocks;
  return static_cast<int>(b);
}

}  // namespace

cudaError_t scan(const srlg_pair* pairs, uint64_t n, const RsraDev& rs, uint32_t rs_now,
                 const SleaDev& le, uint32_t le_now, int mode, cudaStream_t st,
                 const AnetDev* anet_p, unsigned long long* raw_records) {
  if (n == 0) return cudaSuccess;
  AnetDev anet{};
  if (anet_p) anet = *anet_p;
  // Occupancy first: one packet per thread while the batch is small (a C2
  // slice is 166k packets -> 651 CTAs); beyond 8 CTAs per SM the grid stops
  // growing and each thread walks UNROLL packets per step.
  const int dev_blocks = 148 * 8;
  const dim3 grid(grid_for(n, kScanThreads, dev_blocks));
  if (mode == kStoreMark)
    return launch_scan_mode<kStoreMark>(pairs, n, rs, rs_now, le, le_now, grid, st, anet, raw_records);
  if (mode == kStoreRedMax)
    return launch_scan_mode<kStoreRedMax>(pairs, n, rs, rs_now, le, le_now, grid, st, anet, raw_records);
  return launch_scan_mode<kStorePlain>(pairs, n, rs, rs_now, le, le_now, grid, st, anet, raw_records);
}

cudaError_t apply_marks(uint8_t* dirty, uint64_t n_rs, uint32_t* rs, uint32_t rs_now,
                        uint64_t n_le, uint32_t* le, uint32_t le_now, cudaStream_t st) {
  const uint64_t vec = (n_rs + n_le + 15) / 16;
  k_apply_marks<<<grid_for(vec, 256, 148 * 8), 256, 0, st>>>(dirty, n_rs, rs, rs_now, n_le, le,
                                                           le_now);
  return cudaGetLastError();
}

CountsLayout counts_layout(const RsraDev* rs, const SleaDev* le) {
  CountsLayout L{};
  if (rs) {
    L.rs_sres = static_cast<uint64_t>(rs->r) << rs->q;
    const uint64_t words = (L.rs_sres + 31) / 32;
    L.rs_blocks = static_cast<uint32_t>(std::min<uint64_t>((words * 32 + 255) / 256, 148 * 8));
  }
  if (le) {
    L.le_chunk = 16384;
    L.le_blocks_per_row = static_cast<uint32_t>((le->row_len + L.le_chunk - 1) / L.le_chunk);
  }
  return L;
}

cudaError_t window_counts(const RsraDev* rs, uint32_t rs_lo, uint32_t hot_min, const SleaDev* le,
                          uint32_t le_lo, const CountsLayout& L, uint32_t* hot_bits,
                          uint32_t* partials, cudaStream_t st) {
  RsraDev r0{};
  SleaDev l0{};
  const uint32_t rb = rs ? L.rs_blocks : 0;
  const uint32_t lb = le ? L.le_blocks_per_row * le->r : 0;
  if (rb + lb == 0) return cudaSuccess;
  k_window_counts<<<rb + lb, 256, 0, st>>>(rs ? *rs : r0, rs_lo, hot_min, rs ? L.rs_sres : 0, rb,
                                           le ? *le : l0, le_lo, L.le_blocks_per_row ? L.le_blocks_per_row : 1,
                                           L.le_chunk, hot_bits, partials);
  return cudaGetLastError();
}

cudaError_t hot_compact(const uint32_t* hot_bits, uint32_t q, uint32_t r, const uint32_t* partials,
                        uint32_t le_rows, uint32_t bpr, uint32_t* hot_cols, WinResult* res,
                        uint64_t work_cap, cudaStream_t st) {
  k_hot_compact<<<1, kCompactThreads, 0, st>>>(hot_bits, q, r, partials, le_rows, bpr, hot_cols,
                                              res, work_cap);
  return cudaGetLastError();
}

cudaError_t reconstruct(const GroupDev& g, const uint32_t* hot_cols, WinResult* res,
                        uint32_t* tuples_a, uint32_t* tuples_b, uint64_t tuple_cap,
                        uint64_t work_cap, Candidate* cands, uint64_t cand_cap, int n_sms,
                        cudaStream_t st) {
  const int grid = n_sms * 4;
  k_seed<<<grid, 256, 0, st>>>(g, hot_cols, res, tuples_a, tuple_cap);
  uint32_t* in = tuples_a;
  uint32_t* out = tuples_b;
  for (uint32_t row = 3; row < g.r; ++row) {
    k_grow<<<grid, 256, 0, st>>>(g, row, hot_cols, res, in, out, tuple_cap, work_cap);
    uint32_t* t = in;
    in = out;
    out = t;
  }
  k_invert<<<grid, 256, 0, st>>>(g, res, in, tuple_cap, cands, cand_cap);
  return cudaGetLastError();
}

cudaError_t usle_weights(const SleaDev& le, uint32_t le_lo, Candidate* cands, const WinResult* res,
                         uint64_t n_host, uint64_t cand_cap, int n_sms, cudaStream_t st) {
  const int grid = res ? n_sms * 2 : grid_for(n_host, 1, n_sms * 2);
  if (!res && n_host == 0) return cudaSuccess;
  k_usle<<<grid, kUsleThreads, 0, st>>>(le, le.lh_dev, le_lo, cands,
                                        res, n_host, cand_cap);
  return cudaGetLastError();
}

cudaError_t export_distances(const uint32_t* stamps, uint64_t n, uint32_t now, uint32_t floor,
                             uint16_t* out, cudaStream_t st) {
  if (!n) return cudaSuccess;
  k_export<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(stamps, n, now, floor, out);
  return cudaGetLastError();
}

cudaError_t import_distances(const uint16_t* in, uint64_t n, uint32_t now, uint32_t* stamps,
                             cudaStream_t st) {
  if (!n) return cudaSuccess;
  k_import<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(in, n, now, stamps);
  return cudaGetLastError();
}

cudaError_t merge_max(uint32_t* a, const uint32_t* b, uint64_t n, uint32_t now_a, uint32_t floor_a,
                      uint32_t now_b, uint32_t floor_b, cudaStream_t st) {
  if (!n) return cudaSuccess;
  k_merge<<<grid_for(n, 256, 148 * 16), 256, 0, st>>>(a, b, n, now_a, floor_a, now_b, floor_b);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace srlg

// ------------------------------------------------ roofline microbenchmark
// Random u32 updates into a buffer of the sketch-state footprint, addresses
// from a counter hash (no input stream): the L2 / HBM random-update rate R
// that SURVEY.md §8d uses as the scan's roofline denominator.
namespace srlg {
namespace dev {
namespace {
template <int MODE>
__global__ void __launch_bounds__(256) k_random_updates(uint32_t* buf, uint64_t n_cells,
                                                        uint64_t n_updates, uint64_t seed,
                                                        uint32_t v) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n_updates;
       i += stride) {
    const uint64_t h = mix64(seed + i * kGolden64);
    const uint64_t idx = __umul64hi(h, n_cells);
    put_stamp<MODE>(buf + idx, v);
  }
}
}  // namespace

namespace {
// The cell-index stream of a trace in one flat index space (RSRA cell i as i,
// SLEA cell j as rs_n + j): r' SLEA entries per packet in packet order, then
// the gated packets' RSRA entries (compacted, order across warps unspecified)
__global__ void __launch_bounds__(256) k_trace_indices(const srlg_pair* pairs, uint64_t n,
                                                       RsraDev rs, SleaDev le, uint32_t rs_n,
                                                       uint32_t* le_idx, uint32_t* rs_idx,
                                                       unsigned long long* rs_cnt) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const srlg_pair p = pairs[i];
    uint32_t k = 0;
    slea_cells<0>(le, le.lh_dev, p.aip, p.bip, [&](uint64_t idx) {
      le_idx[i * le.r + k++] = rs_n + static_cast<uint32_t>(idx);
    });
    rsra_cells(rs, p.aip, p.bip, [&](uint64_t idx) {
      rs_idx[atomicAdd(rs_cnt, 1ull)] = static_cast<uint32_t>(idx);
    });
  }
}

// replay of an index stream as red.max updates (the random-update roofline on
// the trace's own address distribution)
__global__ void __launch_bounds__(256) k_replay_updates(const uint32_t* idx, uint64_t n,
                                                        uint32_t* buf, uint32_t v) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t pol = policy_evict_first();
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    uint32_t e;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(e)
                 : "l"(idx + i), "l"(pol));
    put_stamp<kStoreRedMax>(buf + e, v);
  }
}
}  // namespace

cudaError_t trace_indices(const srlg_pair* pairs, uint64_t n, const RsraDev& rs, const SleaDev& le,
                          uint32_t* le_idx, uint32_t* rs_idx, unsigned long long* rs_cnt,
                          int n_sms, cudaStream_t st) {
  const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(n_sms) * 8);
  k_trace_indices<<<static_cast<unsigned>(std::max<uint64_t>(blocks, 1)), 256, 0, st>>>(
      pairs, n, rs, le, static_cast<uint32_t>(uint64_t{rs.r} << rs.q) * rs.eta, le_idx, rs_idx,
      rs_cnt);
  return cudaGetLastError();
}

cudaError_t replay_updates(const uint32_t* idx, uint64_t n, uint32_t* buf, uint32_t v, int n_sms,
                           cudaStream_t st) {
  k_replay_updates<<<n_sms * 8, 256, 0, st>>>(idx, n, buf, v);
  return cudaGetLastError();
}

cudaError_t random_updates(uint32_t* buf, uint64_t n_cells, uint64_t n_updates, int mode,
                           uint64_t seed, uint32_t v, int n_sms, cudaStream_t st) {
  const int grid = n_sms * 8;
  if (mode == kStoreRedMax)
    k_random_updates<kStoreRedMax><<<grid, 256, 0, st>>>(buf, n_cells, n_updates, seed, v);
  else
    k_random_updates<kStorePlain><<<grid, 256, 0, st>>>(buf, n_cells, n_updates, seed, v);
  return cudaGetLastError();
}
}  // namespace dev
}  // namespace srlg
