// slidecard/trace.hpp — B200 drop-in of the reference's trace types
// (proj/core/include/slidecard/trace.hpp:14-73). TraceRecord lives in
// slidecard/window.hpp; RawPacket, CidrPrefix, AnetSpec and classify keep the
// reference's names and semantics. Text parsing (parse_ipv4, CidrPrefix::
// parse, AnetSpec::parse, parse_trace_line, TraceReader) is CLI-side and out
// of scope; on the device, classify is fused into the scan
// (srlg_update_raw, srlg_engine_set_anet) and binary traces are read by
// srlg_engine_process_file.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

#include "slidecard/window.hpp"
#include "srlg.h"

namespace slidecard {

// raw packet endpoint pair, before direction classification
struct RawPacket {
  uint64_t ts_us = 0;
  uint32_t src = 0;
  uint32_t dst = 0;

  bool operator==(const RawPacket&) const = default;
};

struct CidrPrefix {
  uint32_t addr = 0;
  uint32_t bits = 0;

  bool contains(uint32_t ip) const {
    if (bits == 0) return true;
    const uint32_t mask = bits >= 32 ? 0xFFFFFFFFu : ~((uint32_t{1} << (32 - bits)) - 1);
    return (ip & mask) == (addr & mask);
  }
};

// the monitored network; a packet is measured from the perspective of every
// endpoint inside it
struct AnetSpec {
  std::vector<CidrPrefix> prefixes;

  bool contains(uint32_t ip) const {
    for (const auto& p : prefixes)
      if (p.contains(ip)) return true;
    return false;
  }

  // the C ABI form (at most SRLG_MAX_PREFIXES prefixes; ConfigError beyond)
  srlg_anet to_c() const;
};

// zero, one or two measurement records depending on which endpoints are
// inside the monitored network; returns how many were written
inline int classify(const RawPacket& p, const AnetSpec& anet, std::array<TraceRecord, 2>& out) {
  int n = 0;
  if (anet.contains(p.src)) out[n++] = TraceRecord{p.ts_us, p.src, p.dst};
  if (anet.contains(p.dst)) out[n++] = TraceRecord{p.ts_us, p.dst, p.src};
  return n;
}

}  // namespace slidecard
