// slidecard/window.hpp — B200 drop-in of proj/core/include/slidecard/window.hpp
// plus the record / report types it uses (trace.hpp, report.hpp) and the
// reconstruction entry point (reconstruct.hpp).
#pragma once

#include <cstdint>
#include <functional>
#include <iosfwd>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "slidecard/rsra.hpp"
#include "slidecard/slea.hpp"

namespace slidecard {

// ---- trace.hpp:23-29
struct TraceRecord {
  uint64_t ts_us = 0;
  uint32_t aip = 0;
  uint32_t bip = 0;
  bool operator==(const TraceRecord&) const = default;
};

std::string format_ipv4(uint32_t addr);

// ---- report.hpp:10-27
struct ReportEntry {
  uint32_t aip = 0;
  double estimate = 0.0;
  bool saturated = false;
};

struct DetectionReport {
  uint64_t window_end_slice = 0;
  std::vector<ReportEntry> entries;
  uint64_t candidate_count = 0;
  std::vector<uint64_t> hot_per_row;
  double sf_product = 0.0;
  bool overflow = false;
  bool slea_saturated = false;
  bool partial = false;
};

void write_report_header(std::ostream& out);
void write_report(const DetectionReport& report, std::ostream& out);
std::string report_to_csv(const std::vector<DetectionReport>& reports);

// parses report blobs of the C ABI (srlg_report_header) into reports
std::vector<DetectionReport> parse_report_blobs(std::span<const uint8_t> blob);

// ---- reconstruct.hpp:10-33
struct ReconstructOptions {
  uint64_t tuple_cap = uint64_t{1} << 22;
  uint64_t work_cap = uint64_t{1} << 32;
  uint32_t workers = 1;  // accepted; the device grid replaces worker threads
  int device = 0;
};

struct ReconstructResult {
  std::vector<uint32_t> addresses;
  bool overflow = false;
  uint64_t tuples_checked = 0;
  uint64_t tuples_kept = 0;
};

ReconstructResult reconstruct_candidates(const std::vector<std::vector<uint32_t>>& hot_columns,
                                         const ReversibleHashGroup& group,
                                         const ReconstructOptions& opt = {});

// ---- window.hpp:15-98
struct WindowConfig {
  std::optional<uint64_t> t0_us;
  uint64_t slice_us = 1'000'000;
  uint32_t k = 300;
  uint64_t theta = 1024;
  bool reinit_per_window = false;
  uint64_t regression_tolerance_us = 0;
  bool keep_below_threshold = false;
  uint32_t workers = 1;
  uint64_t tuple_cap = uint64_t{1} << 22;

  void validate() const;
  srlg_window_config to_c() const;
};

uint64_t slice_index(uint64_t ts_us, uint64_t t0_us, uint64_t slice_us);

class SliceClock {
 public:
  SliceClock(std::optional<uint64_t> t0_us, uint64_t slice_us, uint64_t tolerance_us)
      : t0_(t0_us), slice_us_(slice_us), tolerance_us_(tolerance_us) {}
  uint64_t place(uint64_t ts_us);
  bool started() const { return max_ts_.has_value(); }
  uint64_t t0() const { return *t0_; }
  uint64_t clamped() const { return clamped_; }

 private:
  std::optional<uint64_t> t0_;
  uint64_t slice_us_;
  uint64_t tolerance_us_;
  std::optional<uint64_t> max_ts_;
  uint64_t clamped_ = 0;
};

// run_detection (src/window.cpp:36-78) on the device sketches
DetectionReport run_detection(const Rsra& rsra, const Slea& slea, uint64_t window_end_slice,
                              bool partial, const WindowConfig& cfg);

// WindowEngine (window.hpp:64-98) over the device engine (srlg_engine).
// Detection runs asynchronously on the GPU; reports reach the sink in order,
// at the latest when the call that completed their slice returns.
class WindowEngine {
 public:
  using ReportSink = std::function<void(const DetectionReport&)>;

  WindowEngine(const WindowConfig& cfg, Rsra rsra, Slea slea, ReportSink sink);
  // value semantics like the reference's: a deep copy (device sketches
  // copied device to device, clock, open slice, sink)
  WindowEngine(const WindowEngine& other);
  WindowEngine& operator=(const WindowEngine& other);
  ~WindowEngine();

  void process(const TraceRecord& rec);
  void process_batch(std::span<const TraceRecord> recs);
  // pre-sliced fast path: slice first+i holds pairs[offsets[i], offsets[i+1])
  void process_slices(std::span<const srlg_pair> pairs, std::span<const uint64_t> offsets,
                      uint64_t first_slice);
  void advance_to_slice(uint64_t slice);
  // raw-packet ingest: later process_slices / process take {src, dst} packets
  // classified on the device (srlg_engine_set_anet); NULL: records again
  void set_anet(const srlg_anet* anet);
  void finish();

  const Rsra& rsra() const;
  const Slea& slea() const;
  uint64_t current_slice() const;
  uint64_t records() const;
  uint64_t clamped() const;
  srlg_engine* handle() const { return e_; }

 private:
  void deliver();

  WindowConfig cfg_;
  ReportSink sink_;
  srlg_engine* e_ = nullptr;
  int device_ = 0;
  mutable std::unique_ptr<Rsra> rsra_view_;
  mutable std::unique_ptr<Slea> slea_view_;
};

}  // namespace slidecard
