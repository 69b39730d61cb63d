// exact.cu — the exact sliding-window super-point oracle on the GPU
// (SURVEY.md §8f-4): ExactSlidingOracle (exact_oracle.hpp:25-62,
// exact_oracle.cpp:22-101) for scoring detection accuracy at 10^8–10^9
// packets, where the reference's unordered_map oracle is slow and capped by
// max_pairs.
//
// Representation, as for the sketches: a pair's "last seen slice" is a u32
// stamp (the slice's clock value) in an open-addressing table keyed by
// aip<<32|bip — one slot per distinct pair ever seen, like the reference's
// last_seen_ map, which never shrinks (max_pairs budget, ResourceError).
// Recording is idempotent (atomicMax of the slice stamp), so packet order
// inside a slice cannot matter. A window's exact per-host distinct-peer
// counts are the live pairs (stamp > lo) grouped by aip: one sweep over the
// pair table into an aip-keyed count table, then a sweep collecting the hosts
// with count >= theta. The host sorts them (cardinality desc, aip asc,
// exact_oracle.cpp:85-89).
#include <cuda_runtime.h>
#include <stdint.h>

#include "srlg.h"

namespace srlg {
namespace exact {

constexpr unsigned long long kEmptyPair = ~0ull;  // the pair (0xFFFFFFFF, 0xFFFFFFFF) has its own slot
constexpr uint32_t kEmptyAip = 0xFFFFFFFFu;       // so does the host 0xFFFFFFFF

__device__ __forceinline__ uint64_t mix(uint64_t x) {  // splitmix64 finalizer (slot hash)
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

// record one pair in the slice stamped `now`; the table has `mask + 1` slots
// plus one spare (index mask + 1) for the all-ones key
__global__ void k_insert(const srlg_pair* __restrict__ pairs, uint64_t n, uint32_t now,
                         unsigned long long* keys, uint32_t* stamps, uint64_t mask,
                         unsigned long long* n_pairs) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const srlg_pair p = pairs[i];
    const unsigned long long key = (static_cast<unsigned long long>(p.aip) << 32) | p.bip;
    uint64_t s;
    if (key == kEmptyPair) {  // the spare slot: a first stamp marks the pair seen
      s = mask + 1;
      if (atomicMax(stamps + s, now) == 0) atomicAdd(n_pairs, 1ull);
      continue;
    } else {
      s = mix(key) & mask;
      while (true) {
        const unsigned long long cur = keys[s];
        if (cur == key) break;
        if (cur == kEmptyPair) {
          const unsigned long long old = atomicCAS(keys + s, kEmptyPair, key);
          if (old == kEmptyPair) {
            atomicAdd(n_pairs, 1ull);
            break;
          }
          if (old == key) break;
        }
        s = (s + 1) & mask;
      }
    }
    atomicMax(stamps + s, now);
  }
}

__device__ __forceinline__ void count_host(uint32_t aip, uint32_t* akeys, uint32_t* counts,
                                           uint64_t amask) {
  uint64_t s;
  if (aip == kEmptyAip) {
    s = amask + 1;
  } else {
    s = mix(aip) & amask;
    while (true) {
      const uint32_t cur = akeys[s];
      if (cur == aip) break;
      if (cur == kEmptyAip) {
        const uint32_t old = atomicCAS(akeys + s, kEmptyAip, aip);
        if (old == kEmptyAip || old == aip) break;
      }
      s = (s + 1) & amask;
    }
  }
  atomicAdd(counts + s, 1u);
}

// live pairs of the window (stamp > lo) counted per host
__global__ void k_count(const unsigned long long* keys, const uint32_t* stamps, uint64_t slots,
                        uint32_t lo, uint32_t* akeys, uint32_t* counts, uint64_t amask) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < slots;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    if (stamps[i] <= lo) continue;  // never seen (0) or outside the window
    count_host(i == slots - 1 ? kEmptyAip : static_cast<uint32_t>(keys[i] >> 32), akeys, counts,
               amask);
  }
}

// hosts with count >= theta -> out (aip, count); the count table is cleared
// on the way (ready for the next window)
__global__ void k_collect(uint32_t* akeys, uint32_t* counts, uint64_t aslots, uint64_t theta,
                          uint64_t* out, unsigned long long* n_out, uint64_t cap) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < aslots;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t c = counts[i];
    if (c == 0) continue;
    const uint32_t aip = i == aslots - 1 ? kEmptyAip : akeys[i];
    if (c >= theta) {
      const unsigned long long k = atomicAdd(n_out, 1ull);
      if (k < cap) out[k] = (static_cast<uint64_t>(aip) << 32) | c;
    }
    counts[i] = 0;
    akeys[i] = kEmptyAip;
  }
}

}  // namespace exact

namespace dev {

cudaError_t exact_insert(const srlg_pair* pairs, uint64_t n, uint32_t now, unsigned long long* keys,
                         uint32_t* stamps, uint64_t mask, unsigned long long* n_pairs,
                         cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint64_t blocks = (n + 255) / 256;
  exact::k_insert<<<static_cast<unsigned>(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>(
      pairs, n, now, keys, stamps, mask, n_pairs);
  return cudaGetLastError();
}

cudaError_t exact_window(const unsigned long long* keys, const uint32_t* stamps, uint64_t slots,
                         uint32_t lo, uint32_t* akeys, uint32_t* counts, uint64_t amask,
                         uint64_t theta, uint64_t* out, unsigned long long* n_out, uint64_t cap,
                         cudaStream_t st) {
  exact::k_count<<<148 * 8, 256, 0, st>>>(keys, stamps, slots, lo, akeys, counts, amask);
  exact::k_collect<<<148 * 8, 256, 0, st>>>(akeys, counts, amask + 2, theta, out, n_out, cap);
  return cudaGetLastError();
}

}  // namespace dev
}  // namespace srlg
