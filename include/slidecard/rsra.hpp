// slidecard/rsra.hpp — B200 drop-in of proj/core/include/slidecard/rsra.hpp.
//
// Same class, same methods, same value semantics; the counters live on the
// GPU as u32 slice stamps behind the C ABI (include/srlg.h). Differences a
// caller can observe are limited to performance:
//  - update() is staged on the host (thread-safe, any order within a slice,
//    exactly as rsra.hpp:38-39 allows) and applied as one batched scan on the
//    next non-update call; update_batch() hands a whole slice over at once;
//  - slide() / reinitialize() are O(1) (the stamp clock moves);
//  - cells() materialises a host mirror of the u16 distances on demand;
//    writes through cells_mut() are pushed back before the next device call.
#pragma once

#include <cstdint>
#include <memory>
#include <mutex>
#include <span>
#include <string>
#include <vector>

#include "slidecard/hash.hpp"
#include "slidecard/sliding_counters.hpp"
#include "srlg.h"

namespace slidecard {

struct RsraConfig {
  uint32_t q = 17;
  uint32_t r = 5;
  uint32_t delta = 5;
  uint32_t eta = 8;
  uint32_t tau = 7;
  uint64_t seed_h1 = 0;
  uint64_t seed_h2 = 0;
  uint64_t seed_rhfg0 = 0;

  bool operator==(const RsraConfig&) const = default;
};

class Rsra {
 public:
  explicit Rsra(const RsraConfig& cfg, int device = 0);
  Rsra(const Rsra& other);
  Rsra& operator=(const Rsra& other);
  Rsra(Rsra&& other) noexcept;
  Rsra& operator=(Rsra&& other) noexcept;
  ~Rsra();

  const RsraConfig& config() const { return cfg_; }
  const ReversibleHashGroup& hash_group() const { return group_; }
  uint64_t slides() const;
  void set_slides(uint64_t s);

  void update(uint32_t aip, uint32_t bip);
  void update_batch(std::span<const srlg_pair> pairs);
  void slide();
  void reinitialize();

  std::vector<std::vector<uint32_t>> extract_hot(uint32_t k) const;
  std::span<const uint16_t> sre(uint32_t row, uint32_t col) const;

  void merge_min(const Rsra& other);
  std::string compatibility_mismatch(const Rsra& other) const;

  std::span<const uint16_t> cells() const;
  std::span<uint16_t> cells_mut();
  uint64_t columns() const { return uint64_t{1} << cfg_.q; }

  // the device handle, with staged updates and host edits applied
  srlg_rsra* handle() const;
  int device() const { return device_; }
  // wraps a handle owned elsewhere (WindowEngine::rsra())
  static Rsra view(srlg_rsra* h, int device);
  // takes ownership of a handle created elsewhere (deserialize_sketch)
  static Rsra adopt(srlg_rsra* h, int device);
  srlg_rsra* release();

 private:
  Rsra() = default;
  void sync() const;
  void mutated() const;

  RsraConfig cfg_;
  ReversibleHashGroup group_{2, 2, 1, 0};
  int device_ = 0;
  srlg_rsra* h_ = nullptr;
  bool owned_ = true;
  mutable std::unique_ptr<std::mutex> mu_ = std::make_unique<std::mutex>();
  mutable std::vector<srlg_pair> staged_;
  mutable std::vector<uint16_t> mirror_;
  mutable bool mirror_valid_ = false;
  bool host_dirty_ = false;
};

Rsra merge(const Rsra& a, const Rsra& b);

}  // namespace slidecard
