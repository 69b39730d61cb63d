// scan_device.cuh — per-packet device functions shared by the scan kernel
// (kernels.cu) and the persistent engine kernel (detect.cu).
#pragma once

#include "srlg_internal.cuh"

namespace srlg {
namespace dev {

// L2 residency: the sketch state (63 MB at paper geometry) is touched every
// slice and must stay in the 126 MB L2, while the packet trace is read once.
// State accesses carry an evict_last policy, trace loads evict_first.
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ uint2 ld_pair_stream(const srlg_pair* p) {
  uint2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y)
               : "l"(p), "l"(policy_evict_first()));
  return v;
}

// stamp load that stays in L2 (phase A of the detection)
__device__ __forceinline__ uint32_t ld_state(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(policy_evict_last()));
  return v;
}

template <int MODE>
__device__ __forceinline__ void put_stamp(uint32_t* p, uint32_t v) {
  if constexpr (MODE == kStoreRedMax) {
    asm volatile("red.relaxed.gpu.global.max.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v),
                 "l"(policy_evict_last())
                 : "memory");
  } else {
    asm volatile("st.global.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v),
                 "l"(policy_evict_last())
                 : "memory");
  }
}

// One record's effect on cell idx. kStoreMark is the multi-GPU scan: `base`
// is then a u8 dirty map and the cell is only marked touched in this slice
// (the root turns marks into stamps after the per-slide NCCL max-reduce).
template <int MODE>
__device__ __forceinline__ void put(uint32_t* base, uint64_t idx, uint32_t v) {
  if constexpr (MODE == kStoreMark) {
    asm volatile("st.global.u8 [%0], %1;" ::"l"(reinterpret_cast<uint8_t*>(base) + idx),
                 "r"(1u)
                 : "memory");
  } else {
    put_stamp<MODE>(base + idx, v);
  }
}

__device__ __forceinline__ uint32_t mod_eta(uint64_t h, uint32_t eta, uint32_t pow2) {
  return pow2 ? static_cast<uint32_t>(h) & (eta - 1) : static_cast<uint32_t>(h % eta);
}

// Rsra::update (src/rsra.cpp:25-33) with sample_gate (src/hash.cpp:29-33) and
// ReversibleHashGroup::forward (src/hash.cpp:63-69): f(idx) for each of the
// record's r cells when the gate passes
template <class F>
__device__ __forceinline__ void rsra_cells(const RsraDev& rs, uint32_t aip, uint32_t bip, F&& f) {
  // lsb(low32(H1(bip))) >= tau  <=>  the low tau bits are zero (lsb(0) = 32)
  const uint32_t g = static_cast<uint32_t>(seeded(rs.h1, bip));
  if (rs.gate_never || (g & rs.gate_mask) != 0) return;
  const uint32_t slot = mod_eta(seeded(rs.h2, bip), rs.eta, rs.eta_pow2);
  const uint32_t c0 = static_cast<uint32_t>(seeded(rs.h0, aip)) & rs.col_mask;
  for (uint32_t i = 0; i < rs.r; ++i) {
    const uint32_t sh = i * rs.delta;
    const uint32_t shifted = sh >= 32 ? 0u : aip >> sh;
    const uint32_t col = i == 0 ? c0 : ((shifted ^ c0) & rs.col_mask);
    f(((static_cast<uint64_t>(i) << rs.q) + col) * rs.eta + slot);
  }
}

// Slea::update (src/slea.cpp:38-45) with le_index (src/hash.cpp:35-37) and
// lh_column (src/slea.cpp:34-36): f(idx) for each of the r' cells. ROWS > 0:
// compile-time row count.
template <int ROWS, class F>
__device__ __forceinline__ void slea_cells(const SleaDev& le, const uint64_t* lh, uint32_t aip,
                                           uint32_t bip, F&& f) {
  const uint32_t slot = mod_eta(seeded(le.h3, bip), le.eta, le.eta_pow2);
  if constexpr (ROWS > 0) {
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      const uint32_t col = static_cast<uint32_t>(seeded(le.lh[i], aip)) & le.col_mask;
      f(i * le.row_len + static_cast<uint64_t>(col) * le.delta + slot);
    }
  } else {
    for (uint32_t i = 0; i < le.r; ++i) {
      const uint32_t col = static_cast<uint32_t>(seeded(lh[i], aip)) & le.col_mask;
      f(i * le.row_len + static_cast<uint64_t>(col) * le.delta + slot);
    }
  }
}

template <int MODE>
__device__ __forceinline__ void rsra_update(const RsraDev& rs, uint32_t now, uint32_t aip,
                                            uint32_t bip) {
  rsra_cells(rs, aip, bip, [&](uint64_t idx) { put<MODE>(rs.cells, idx, now); });
}

template <int MODE, int ROWS>
__device__ __forceinline__ void slea_update(const SleaDev& le, const uint64_t* lh, uint32_t now,
                                            uint32_t aip, uint32_t bip) {
  slea_cells<ROWS>(le, lh, aip, bip, [&](uint64_t idx) { put<MODE>(le.cells, idx, now); });
}

// ------------------------------------------------ tracked updates (engine)
// The same stamp updates as rsra_update / slea_update, plus the marks of the
// incremental detection (IncDev, srlg_internal.cuh): a marked block is
// re-examined by the next detection.
//  * RSRA: every gated update marks its block (a plain store next to the
//    red; 1/2^tau of the records pass the gate).
//  * SLEA with kOpLe: a cell whose bit of the live inside bitmap (exact for
//    the last detection; it only changes in phase A) is clear enters the
//    window, and its block is marked. (An atom.max returning the old stamp
//    and this L2 read cost alike: each doubles the scan's L2 operations.)
// A block may be marked more than once (idempotent); never less.
__device__ __forceinline__ uint32_t ld_live(const uint32_t* bits, uint64_t idx) {
  uint32_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(bits + (idx >> 5)), "l"(policy_evict_last()));
  return v;
}

__device__ __forceinline__ void mark_block(uint32_t* smin, uint64_t idx) {
  asm volatile("st.global.u32 [%0], %1;" ::"l"(smin + (idx >> kIncBlockLog)), "r"(0u) : "memory");
}

// RSRA cell: stamp and mark
__device__ __forceinline__ void track_rs_cell(uint32_t* cells, uint32_t* smin, uint64_t idx,
                                              uint32_t now) {
  put_stamp<kStoreRedMax>(cells + idx, now);
  mark_block(smin, idx);
}

// SLEA cell, one at a time (merge apply, dynamic row counts)
__device__ __forceinline__ void track_le_cell(const SleaDev& le, const IncDev& inc, uint64_t idx,
                                              uint32_t now) {
  put_stamp<kStoreRedMax>(le.cells + idx, now);
  if (!((ld_live(inc.live_bits, idx) >> (idx & 31)) & 1u)) mark_block(inc.le_smin, idx);
}

// The first n <= N records' SLEA cells: every red and every bitmap read of
// the records is issued before any bit is examined (one round trip per call;
// cell indices fit 32 bits: the reference caps a sketch at 2^31 cells)
template <int ROWS, int N>
__device__ __forceinline__ void track_le_rows(const SleaDev& le, const IncDev& inc, uint32_t now,
                                              const uint2 (&p)[N], uint32_t n) {
  uint32_t idx[N][ROWS];
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const uint32_t slot = mod_eta(seeded(le.h3, p[k].y), le.eta, le.eta_pow2);
#pragma unroll
    for (int i = 0; i < ROWS; ++i)
      idx[k][i] = static_cast<uint32_t>(i * le.row_len) +
                  (static_cast<uint32_t>(seeded(le.lh[i], p[k].x)) & le.col_mask) * le.delta + slot;
  }
  uint32_t w[N][ROWS];
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int i = 0; i < ROWS; ++i) {
      w[k][i] = 0xFFFFFFFFu;
      if (k < n) {
        put_stamp<kStoreRedMax>(le.cells + idx[k][i], now);
        w[k][i] = ld_live(inc.live_bits, idx[k][i]);
      }
    }
#pragma unroll
  for (int k = 0; k < N; ++k)
#pragma unroll
    for (int i = 0; i < ROWS; ++i)
      if (!((w[k][i] >> (idx[k][i] & 31)) & 1u)) mark_block(inc.le_smin, idx[k][i]);
}

// the first n <= N records (aip, bip) = p[k], RSRA and SLEA tracked (kOpLe)
template <int ROWS, int N>
__device__ __forceinline__ void track_records(const RsraDev& rs, const SleaDev& le, const uint64_t* lh,
                                              const IncDev& inc, uint32_t rs_now, uint32_t le_now,
                                              const uint2 (&p)[N], uint32_t n) {
#pragma unroll
  for (int k = 0; k < N; ++k)
    if (k < n)
      rsra_cells(rs, p[k].x, p[k].y,
                 [&](uint64_t idx) { track_rs_cell(rs.cells, inc.rs_smin, idx, rs_now); });
  if constexpr (ROWS > 0) {
    track_le_rows<ROWS, N>(le, inc, le_now, p, n);
  } else {
#pragma unroll
    for (int k = 0; k < N; ++k)
      if (k < n)
        slea_cells<0>(le, lh, p[k].x, p[k].y,
                      [&](uint64_t idx) { track_le_cell(le, inc, idx, le_now); });
  }
}

// one record, RSRA tracked, SLEA stamped only
template <int ROWS>
__device__ __forceinline__ void track_rs_record(const RsraDev& rs, const SleaDev& le, const uint64_t* lh,
                                                const IncDev& inc, uint32_t rs_now, uint32_t le_now,
                                                uint32_t aip, uint32_t bip) {
  rsra_cells(rs, aip, bip, [&](uint64_t idx) { track_rs_cell(rs.cells, inc.rs_smin, idx, rs_now); });
  slea_update<kStoreRedMax, ROWS>(le, lh, le_now, aip, bip);
}

// CidrPrefix::contains / AnetSpec::contains (trace.hpp:38-42, 53-57)
__device__ __forceinline__ bool anet_contains(const AnetDev& a, uint32_t ip) {
  bool in = false;
  for (uint32_t i = 0; i < a.n; ++i) in |= (ip & a.mask[i]) == a.addr[i];
  return in;
}

// One packet's effect: a classified record (aip, bip) when anet.n == 0, else
// classify (trace.cpp:111-116): a record per endpoint inside the network.
// rec(aip, bip) applies one record. Returns the number of records.
template <class Rec>
__device__ __forceinline__ uint32_t ingest_with(const AnetDev& anet, uint2 p, Rec&& rec) {
  if (anet.n == 0) {
    rec(p.x, p.y);
    return 1;
  }
  uint32_t k = 0;
  if (anet_contains(anet, p.x)) {
    rec(p.x, p.y);
    ++k;
  }
  if (anet_contains(anet, p.y)) {
    rec(p.y, p.x);
    ++k;
  }
  return k;
}

template <int MODE, int ROWS>
__device__ __forceinline__ uint32_t ingest(const RsraDev& rs, const SleaDev& le,
                                           const uint64_t* lh, uint32_t rs_now, uint32_t le_now,
                                           const AnetDev& anet, uint2 p) {
  return ingest_with(anet, p, [&](uint32_t aip, uint32_t bip) {
    if (rs.cells) rsra_update<MODE>(rs, rs_now, aip, bip);
    if (le.cells) slea_update<MODE, ROWS>(le, lh, le_now, aip, bip);
  });
}

}  // namespace dev
}  // namespace srlg
