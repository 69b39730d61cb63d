// slidecard/exact_oracle.hpp — B200 drop-in of the reference's exact sliding
// oracle (proj/core/include/slidecard/exact_oracle.hpp:14-94). TruthEntry,
// TruthWindow, AccuracyResult and score() keep the reference's names and
// semantics; the oracle itself runs on the device (srlg_exact_*, exact.cu)
// over pre-sliced pairs, the layout WindowEngine::process_slices takes.
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "srlg.h"

namespace slidecard {

struct TruthEntry {
  uint32_t aip = 0;
  uint64_t cardinality = 0;
};

struct TruthWindow {
  uint64_t window_end_slice = 0;
  bool partial = false;
  std::vector<TruthEntry> supers;  // cardinality >= theta; card desc, aip asc
};

struct ExactOptions {
  uint64_t theta = 1024;
  uint32_t k = 300;
  uint64_t max_pairs = 100'000'000;  // explicit budget; ResourceError beyond
  int device = 0;
};

// exact_detect (exact_oracle.cpp:92-101) over pre-sliced pairs: one window
// per completed slice from k-1 on plus the partial one at stream end
std::vector<TruthWindow> exact_detect_slices(std::span<const srlg_pair> pairs,
                                             std::span<const uint64_t> offsets,
                                             const ExactOptions& opt);

// detection-accuracy ratios, all normalized by the true super-point count
struct AccuracyResult {
  uint64_t window_end_slice = 0;
  uint64_t n_true = 0;
  uint64_t n_detected = 0;
  uint64_t n_false_pos = 0;
  uint64_t n_false_neg = 0;
  double fpr = 0.0;
  double fnr = 0.0;
  double tfr = 0.0;
  bool defined = false;  // false when no true super points exist
};

AccuracyResult score(uint64_t window_end_slice, std::span<const uint32_t> detected,
                     std::span<const TruthEntry> truth);

}  // namespace slidecard
