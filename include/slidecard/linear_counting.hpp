// slidecard/linear_counting.hpp — B200 drop-in of
// proj/core/include/slidecard/linear_counting.hpp (host double math, the
// reference's exact expressions).
#pragma once

#include <cstdint>

namespace slidecard {

inline constexpr double kSaturationEps = 1e-9;

struct LinearEstimate {
  double value = 0.0;
  bool saturated = false;
};

LinearEstimate le_estimate(double weight, uint32_t eta_prime);
double corrected_weight(double usle_weight, double sf_product, uint32_t eta_prime);

}  // namespace slidecard
