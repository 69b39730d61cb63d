// dropin.cpp — the C++ drop-in of the reference estimator API
// (include/slidecard/*.hpp) over the C ABI of include/srlg.h.
//
// A caller of the reference (proj/core, namespace slidecard) recompiles
// against include/ and links libslidecard_b200.so + libsrlg.so; Rsra, Slea,
// run_detection, WindowEngine, reconstruct_candidates and run_distributed
// then execute on the GPU. Host-only helpers (hashing, parameters, report
// formatting) follow the reference's definitions.
#include <algorithm>
#include <iterator>
#include <unistd.h>
#include <atomic>
#include <cmath>
#include <cstring>
#include <fstream>
#include <ostream>
#include <sstream>
#include <stdexcept>

#include "slidecard/config.hpp"
#include "slidecard/distributed.hpp"
#include "slidecard/sketch_io.hpp"
#include "slidecard/errors.hpp"
#include "slidecard/hash.hpp"
#include "slidecard/linear_counting.hpp"
#include "slidecard/rng.hpp"
#include "slidecard/rsra.hpp"
#include "slidecard/slea.hpp"
#include "slidecard/sliding_counters.hpp"
#include "slidecard/window.hpp"
#include "srlg.h"

namespace slidecard {

// ------------------------------------------------------------------ errors

void throw_status(int st) {
  if (st == SRLG_OK) return;
  const std::string msg = srlg_last_error();
  switch (st) {
    case SRLG_ERR_CONFIG: throw ConfigError(msg);
    case SRLG_ERR_PARSE: throw ParseError(msg);
    case SRLG_ERR_ORDERING: throw OrderingError(msg);
    case SRLG_ERR_FORMAT: throw FormatError(msg);
    case SRLG_ERR_RESOURCE: throw ResourceError(msg);
    case SRLG_ERR_INCOMPATIBLE: throw IncompatibleSketchError(msg);
    case SRLG_ERR_SATURATION: throw SaturationError(msg);
    case SRLG_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
    case SRLG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw DeviceError(msg);
  }
}

namespace {
void ok(int st) { throw_status(st); }
constexpr size_t kStageFlush = size_t{1} << 22;  // staged pairs before an eager flush
}  // namespace

// ----------------------------------------------------------------- hashing

uint32_t sampling_threshold(uint64_t theta, uint64_t eta) {
  if (eta == 0) throw ConfigError("sampling threshold: eta must be positive");
  uint32_t t = 0;
  while (t < 64 && eta <= (UINT64_MAX >> t) && (eta << t) < theta) ++t;
  return t;
}

HashSeeds HashSeeds::derive(uint64_t m, uint32_t lh_count) {
  HashSeeds s;
  s.h1 = hash64(1, m);
  s.h2 = hash64(2, m);
  s.h3 = hash64(3, m);
  s.rhfg0 = hash64(4, m);
  for (uint32_t i = 0; i < lh_count; ++i) s.lh.push_back(hash64(100 + i, m));
  return s;
}

std::optional<uint32_t> sample_gate(uint32_t bip, uint32_t tau, uint32_t eta,
                                    const SeededHash& h1, const SeededHash& h2) {
  if (lsb(static_cast<uint32_t>(h1(bip))) < tau) return std::nullopt;
  return static_cast<uint32_t>(h2(bip) % eta);
}

uint32_t le_index(uint32_t bip, uint32_t eta_prime, const SeededHash& h3) {
  return static_cast<uint32_t>(h3(bip) % eta_prime);
}

ReversibleHashGroup::ReversibleHashGroup(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed)
    : q_(q), r_(r), delta_(delta), seed_(seed), h0_(seed) {
  if (q == 0 || q > 31) throw ConfigError("hash group: q must be in [1, 31]");
  if (r < 2) throw ConfigError("hash group: need at least 2 rows");
  if (delta == 0 || delta >= q) throw ConfigError("hash group: delta must satisfy 1 <= delta < q");
  col_mask_ = (uint32_t{1} << q) - 1;
  overlap_mask_ = (uint32_t{1} << (q - delta)) - 1;
  uint64_t covered = 0;
  for (uint32_t i = 1; i < r; ++i) {
    const uint32_t lo = i * delta;
    if (lo >= kAddressBits) break;
    const uint32_t hi = std::min<uint32_t>(kAddressBits, lo + q);
    covered |= ((uint64_t{1} << (hi - lo)) - 1) << lo;
  }
  uncovered_mask_ = static_cast<uint32_t>(~covered & 0xFFFFFFFFull);
}

void ReversibleHashGroup::forward(uint32_t aip, std::span<uint32_t> out) const {
  out[0] = base(aip);
  for (uint32_t i = 1; i < r_; ++i) {
    const uint32_t sh = i * delta_;
    out[i] = ((sh >= kAddressBits ? 0u : aip >> sh) ^ out[0]) & col_mask_;
  }
}

std::vector<uint32_t> ReversibleHashGroup::forward(uint32_t aip) const {
  std::vector<uint32_t> v(r_);
  forward(aip, v);
  return v;
}

// invert = reconstruction over one-element hot lists, on the device
std::vector<uint32_t> ReversibleHashGroup::invert(std::span<const uint32_t> columns) const {
  if (columns.size() != r_)
    throw std::invalid_argument("invert: expected one column index per row");
  if (r_ < 3) {
    // reconstruct_candidates needs 3 rows; 2-row groups invert on the host
    std::vector<uint32_t> out;
    const uint32_t w1 = (columns[1] ^ columns[0]) & col_mask_;
    const uint32_t assembled = static_cast<uint32_t>(static_cast<uint64_t>(w1) << delta_);
    std::vector<uint32_t> free_bits;
    for (uint32_t b = 0; b < kAddressBits; ++b)
      if (uncovered_mask_ & (1u << b)) free_bits.push_back(b);
    if (free_bits.size() > 26) throw ResourceError("invert: too many unconstrained bits");
    for (uint64_t v = 0; v < (uint64_t{1} << free_bits.size()); ++v) {
      uint32_t c = assembled & ~uncovered_mask_;
      for (size_t b = 0; b < free_bits.size(); ++b)
        if (v & (uint64_t{1} << b)) c |= 1u << free_bits[b];
      if (forward(c) == std::vector<uint32_t>(columns.begin(), columns.end())) out.push_back(c);
    }
    return out;
  }
  std::vector<std::vector<uint32_t>> hot(r_);
  for (uint32_t i = 0; i < r_; ++i) {
    if (columns[i] > col_mask_) return {};
    hot[i] = {columns[i]};
  }
  return reconstruct_candidates(hot, *this).addresses;
}

// -------------------------------------------------------- sliding counters

namespace counter_ops {
void record(std::span<uint16_t> c, size_t idx) {
  if (idx >= c.size()) throw std::out_of_range("record: slot index out of range");
  std::atomic_ref<uint16_t>(c[idx]).store(0, std::memory_order_relaxed);
}
void slide(std::span<uint16_t> c) {
  for (uint16_t& v : c)
    if (v != kNeverSet) ++v;
}
size_t weight(std::span<const uint16_t> c, uint32_t k) {
  if (k > kNeverSet) k = kNeverSet;
  size_t n = 0;
  for (uint16_t v : c) n += v < k;
  return n;
}
void min_into(std::span<uint16_t> acc, std::span<const uint16_t> other) {
  if (acc.size() != other.size()) throw std::invalid_argument("min_into: length mismatch");
  for (size_t i = 0; i < acc.size(); ++i) acc[i] = std::min(acc[i], other[i]);
}
void max_into(std::span<uint16_t> acc, std::span<const uint16_t> other) {
  if (acc.size() != other.size()) throw std::invalid_argument("max_into: length mismatch");
  for (size_t i = 0; i < acc.size(); ++i) acc[i] = std::max(acc[i], other[i]);
}
}  // namespace counter_ops

double detection_rho() { return 0.99 * (1.0 - std::exp(-1.0 / 3.0)); }

void SlidingCounterVector::record(size_t idx) { counter_ops::record(c_, idx); }

SlidingCounterVector combine_min(const SlidingCounterVector& a, const SlidingCounterVector& b) {
  SlidingCounterVector r(a);
  counter_ops::min_into(r.span(), b.span());
  return r;
}

SlidingCounterVector combine_max(const SlidingCounterVector& a, const SlidingCounterVector& b) {
  SlidingCounterVector r(a);
  counter_ops::max_into(r.span(), b.span());
  return r;
}

// ------------------------------------------------------- linear counting

LinearEstimate le_estimate(double weight, uint32_t eta_prime) {
  const double eta = static_cast<double>(eta_prime);
  if (weight <= 0.0) return {0.0, false};
  if (weight >= eta) return {eta * std::log(eta), true};
  return {-eta * std::log((eta - weight) / eta), false};
}

double corrected_weight(double usle_weight, double sf_product, uint32_t eta_prime) {
  if (sf_product >= 1.0)
    throw SaturationError("corrected weight: setting-factor product is 1, estimate unusable");
  if (sf_product < 0.0) sf_product = 0.0;
  const double eta = static_cast<double>(eta_prime);
  return std::clamp((usle_weight - eta * sf_product) / (1.0 - sf_product), 0.0, eta);
}

// ------------------------------------------------------------------- Rsra

namespace {
srlg_rsra_config to_c(const RsraConfig& c) {
  srlg_rsra_config o{};
  o.q = c.q;
  o.r = c.r;
  o.delta = c.delta;
  o.eta = c.eta;
  o.tau = c.tau;
  o.seed_h1 = c.seed_h1;
  o.seed_h2 = c.seed_h2;
  o.seed_rhfg0 = c.seed_rhfg0;
  return o;
}

RsraConfig from_c(const srlg_rsra_config& c) {
  RsraConfig o;
  o.q = c.q;
  o.r = c.r;
  o.delta = c.delta;
  o.eta = c.eta;
  o.tau = c.tau;
  o.seed_h1 = c.seed_h1;
  o.seed_h2 = c.seed_h2;
  o.seed_rhfg0 = c.seed_rhfg0;
  return o;
}

srlg_slea_config to_c(const SleaConfig& c) {
  srlg_slea_config o{};
  o.q = c.q;
  o.r = c.r;
  o.delta = c.delta;
  o.eta = c.eta;
  o.seed_h3 = c.seed_h3;
  if (c.seeds_lh.size() > SRLG_MAX_ROWS) throw ConfigError("slea: at most 64 rows supported");
  if (c.seeds_lh.size() != c.r) throw ConfigError("slea: need exactly one row hash seed per row");
  for (size_t i = 0; i < c.seeds_lh.size(); ++i) o.seeds_lh[i] = c.seeds_lh[i];
  return o;
}

SleaConfig from_c(const srlg_slea_config& c) {
  SleaConfig o;
  o.q = c.q;
  o.r = c.r;
  o.delta = c.delta;
  o.eta = c.eta;
  o.seed_h3 = c.seed_h3;
  o.seeds_lh.assign(c.seeds_lh, c.seeds_lh + c.r);
  return o;
}
}  // namespace

Rsra::Rsra(const RsraConfig& cfg, int device)
    : cfg_(cfg), group_(cfg.q, cfg.r, cfg.delta, cfg.seed_rhfg0), device_(device) {
  const srlg_rsra_config c = to_c(cfg);
  ok(srlg_rsra_create(&c, device, &h_));
}

Rsra::Rsra(const Rsra& o) : cfg_(o.cfg_), group_(o.group_), device_(o.device_) {
  ok(srlg_rsra_clone(o.handle(), &h_));
}

Rsra& Rsra::operator=(const Rsra& o) {
  if (this != &o) {
    Rsra tmp(o);
    *this = std::move(tmp);
  }
  return *this;
}

Rsra::Rsra(Rsra&& o) noexcept
    : cfg_(o.cfg_),
      group_(o.group_),
      device_(o.device_),
      h_(o.h_),
      owned_(o.owned_),
      mu_(std::move(o.mu_)),
      staged_(std::move(o.staged_)),
      mirror_(std::move(o.mirror_)),
      mirror_valid_(o.mirror_valid_),
      host_dirty_(o.host_dirty_) {
  o.h_ = nullptr;
  o.mu_ = std::make_unique<std::mutex>();
}

Rsra& Rsra::operator=(Rsra&& o) noexcept {
  if (this != &o) {
    if (h_ && owned_) srlg_rsra_destroy(h_);
    cfg_ = o.cfg_;
    group_ = o.group_;
    device_ = o.device_;
    h_ = o.h_;
    owned_ = o.owned_;
    mu_ = std::move(o.mu_);
    staged_ = std::move(o.staged_);
    mirror_ = std::move(o.mirror_);
    mirror_valid_ = o.mirror_valid_;
    host_dirty_ = o.host_dirty_;
    o.h_ = nullptr;
    o.mu_ = std::make_unique<std::mutex>();
  }
  return *this;
}

Rsra::~Rsra() {
  if (h_ && owned_) srlg_rsra_destroy(h_);
}

Rsra Rsra::view(srlg_rsra* h, int device) {
  Rsra r;
  srlg_rsra_config c{};
  srlg_rsra_config_get(h, &c);
  r.cfg_ = from_c(c);
  r.group_ = ReversibleHashGroup(c.q, c.r, c.delta, c.seed_rhfg0);
  r.device_ = device;
  r.h_ = h;
  r.owned_ = false;
  return r;
}

Rsra Rsra::adopt(srlg_rsra* h, int device) {
  Rsra r = view(h, device);
  r.owned_ = true;
  return r;
}

srlg_rsra* Rsra::release() {
  sync();
  srlg_rsra* h = h_;
  h_ = nullptr;
  return h;
}

// host edits first (they were made against the state before the staged
// updates), then the staged updates as one batched scan
void Rsra::sync() const {
  auto* self = const_cast<Rsra*>(this);
  if (host_dirty_) {
    ok(srlg_rsra_import_cells(h_, mirror_.data(), mirror_.size()));
    (void)self;  // sticky: a handed-out cells_mut() span stays authoritative
  }
  std::vector<srlg_pair> batch;
  {
    std::lock_guard<std::mutex> lk(*mu_);
    batch.swap(staged_);
  }
  if (!batch.empty()) {
    ok(srlg_update_pairs(h_, nullptr, batch.data(), batch.size(), 0, nullptr));
    mutated();
  }
}

// device state changed: drop the mirror, or — once a cells_mut() span has
// been handed out — refresh it in place so the span keeps showing the live
// state (the reference's span aliases its storage)
void Rsra::mutated() const {
  mirror_valid_ = false;
  if (host_dirty_) {
    ok(srlg_rsra_export_cells(h_, mirror_.data(), mirror_.size()));
    mirror_valid_ = true;
  }
}

srlg_rsra* Rsra::handle() const {
  sync();
  return h_;
}

uint64_t Rsra::slides() const { return srlg_rsra_slides(h_); }
void Rsra::set_slides(uint64_t s) { ok(srlg_rsra_set_slides(h_, s)); }

void Rsra::update(uint32_t aip, uint32_t bip) {
  bool flush = false;
  {
    std::lock_guard<std::mutex> lk(*mu_);
    staged_.push_back(srlg_pair{aip, bip});
    flush = staged_.size() >= kStageFlush && !host_dirty_;
  }
  if (flush) sync();
}

void Rsra::update_batch(std::span<const srlg_pair> pairs) {
  sync();
  ok(srlg_update_pairs(h_, nullptr, pairs.data(), pairs.size(), 0, nullptr));
  mutated();
}

void Rsra::slide() {
  sync();
  ok(srlg_rsra_slide(h_));
  mutated();
}

void Rsra::reinitialize() {
  sync();
  ok(srlg_rsra_reinitialize(h_));
  mutated();
}

std::vector<std::vector<uint32_t>> Rsra::extract_hot(uint32_t k) const {
  sync();
  std::vector<uint32_t> cols(std::max<uint64_t>(1, static_cast<uint64_t>(cfg_.r) << cfg_.q));
  std::vector<uint64_t> counts(cfg_.r);
  ok(srlg_rsra_extract_hot(h_, k, cols.data(), cols.size(), counts.data()));
  std::vector<std::vector<uint32_t>> out(cfg_.r);
  size_t off = 0;
  for (uint32_t i = 0; i < cfg_.r; ++i) {
    out[i].assign(cols.begin() + off, cols.begin() + off + counts[i]);
    off += counts[i];
  }
  return out;
}

std::span<const uint16_t> Rsra::cells() const {
  sync();
  if (!mirror_valid_) {
    mirror_.resize(srlg_rsra_num_cells(h_));
    ok(srlg_rsra_export_cells(h_, mirror_.data(), mirror_.size()));
    mirror_valid_ = true;
  }
  return mirror_;
}

std::span<uint16_t> Rsra::cells_mut() {
  cells();
  host_dirty_ = true;
  return mirror_;
}

std::span<const uint16_t> Rsra::sre(uint32_t row, uint32_t col) const {
  if (row >= cfg_.r || col >= columns()) throw std::out_of_range("rsra: row/column out of range");
  return cells().subspan(((static_cast<size_t>(row) << cfg_.q) + col) * cfg_.eta, cfg_.eta);
}

std::string Rsra::compatibility_mismatch(const Rsra& o) const {
  char buf[64];
  ok(srlg_rsra_compatibility_mismatch(h_, o.h_, buf, sizeof buf));
  return buf;
}

void Rsra::merge_min(const Rsra& o) {
  sync();
  ok(srlg_rsra_merge_min(h_, o.handle()));
  mutated();
}

Rsra merge(const Rsra& a, const Rsra& b) {
  Rsra out = a;
  out.merge_min(b);
  return out;
}

// ------------------------------------------------------------------- Slea

Slea::Slea(const SleaConfig& cfg, int device) : cfg_(cfg), device_(device) {
  if (cfg.r == 0) throw ConfigError("slea: need at least one row");
  if (cfg.r > 64) throw ConfigError("slea: at most 64 rows supported");
  const srlg_slea_config c = to_c(cfg);
  ok(srlg_slea_create(&c, device, &h_));
  row_len_ = srlg_slea_row_length(h_);
}

Slea::Slea(const Slea& o) : cfg_(o.cfg_), row_len_(o.row_len_), device_(o.device_) {
  ok(srlg_slea_clone(o.handle(), &h_));
}

Slea& Slea::operator=(const Slea& o) {
  if (this != &o) {
    Slea tmp(o);
    *this = std::move(tmp);
  }
  return *this;
}

Slea::Slea(Slea&& o) noexcept
    : cfg_(std::move(o.cfg_)),
      row_len_(o.row_len_),
      device_(o.device_),
      h_(o.h_),
      owned_(o.owned_),
      mu_(std::move(o.mu_)),
      staged_(std::move(o.staged_)),
      mirror_(std::move(o.mirror_)),
      mirror_valid_(o.mirror_valid_),
      host_dirty_(o.host_dirty_) {
  o.h_ = nullptr;
  o.mu_ = std::make_unique<std::mutex>();
}

Slea& Slea::operator=(Slea&& o) noexcept {
  if (this != &o) {
    if (h_ && owned_) srlg_slea_destroy(h_);
    cfg_ = std::move(o.cfg_);
    row_len_ = o.row_len_;
    device_ = o.device_;
    h_ = o.h_;
    owned_ = o.owned_;
    mu_ = std::move(o.mu_);
    staged_ = std::move(o.staged_);
    mirror_ = std::move(o.mirror_);
    mirror_valid_ = o.mirror_valid_;
    host_dirty_ = o.host_dirty_;
    o.h_ = nullptr;
    o.mu_ = std::make_unique<std::mutex>();
  }
  return *this;
}

Slea::~Slea() {
  if (h_ && owned_) srlg_slea_destroy(h_);
}

Slea Slea::view(srlg_slea* h, int device) {
  Slea s;
  srlg_slea_config c{};
  srlg_slea_config_get(h, &c);
  s.cfg_ = from_c(c);
  s.row_len_ = srlg_slea_row_length(h);
  s.device_ = device;
  s.h_ = h;
  s.owned_ = false;
  return s;
}

Slea Slea::adopt(srlg_slea* h, int device) {
  Slea s = view(h, device);
  s.owned_ = true;
  return s;
}

srlg_slea* Slea::release() {
  sync();
  srlg_slea* h = h_;
  h_ = nullptr;
  return h;
}

void Slea::sync() const {
  auto* self = const_cast<Slea*>(this);
  if (host_dirty_) {
    ok(srlg_slea_import_cells(h_, mirror_.data(), mirror_.size()));
    (void)self;  // sticky: a handed-out cells_mut() span stays authoritative
  }
  std::vector<srlg_pair> batch;
  {
    std::lock_guard<std::mutex> lk(*mu_);
    batch.swap(staged_);
  }
  if (!batch.empty()) {
    ok(srlg_update_pairs(nullptr, h_, batch.data(), batch.size(), 0, nullptr));
    mutated();
  }
}

void Slea::mutated() const {
  mirror_valid_ = false;
  if (host_dirty_) {
    ok(srlg_slea_export_cells(h_, mirror_.data(), mirror_.size()));
    mirror_valid_ = true;
  }
}

srlg_slea* Slea::handle() const {
  sync();
  return h_;
}

uint64_t Slea::slides() const { return srlg_slea_slides(h_); }
void Slea::set_slides(uint64_t s) { ok(srlg_slea_set_slides(h_, s)); }

double Slea::memory_reduction_ratio() const {
  const double full = static_cast<double>(cfg_.eta) * static_cast<double>(uint64_t{1} << cfg_.q);
  return 1.0 - static_cast<double>(row_len_) / full;
}

void Slea::update(uint32_t aip, uint32_t bip) {
  bool flush = false;
  {
    std::lock_guard<std::mutex> lk(*mu_);
    staged_.push_back(srlg_pair{aip, bip});
    flush = staged_.size() >= kStageFlush && !host_dirty_;
  }
  if (flush) sync();
}

void Slea::update_batch(std::span<const srlg_pair> pairs) {
  sync();
  ok(srlg_update_pairs(nullptr, h_, pairs.data(), pairs.size(), 0, nullptr));
  mutated();
}

void Slea::slide() {
  sync();
  ok(srlg_slea_slide(h_));
  mutated();
}

void Slea::reinitialize() {
  sync();
  ok(srlg_slea_reinitialize(h_));
  mutated();
}

double Slea::setting_factor(uint32_t row, uint32_t k) const {
  if (row >= cfg_.r) throw std::out_of_range("slea: row out of range");
  return make_estimate_context(k).setting_factors[row];
}

uint32_t Slea::lh_column(uint32_t row, uint32_t aip) const {
  uint32_t c = 0;
  ok(srlg_slea_lh_column(h_, row, aip, &c));
  return c;
}

Slea::EstimateContext Slea::make_estimate_context(uint32_t k) const {
  sync();
  EstimateContext ctx;
  ctx.k = k;
  ctx.setting_factors.resize(cfg_.r);
  ok(srlg_slea_estimate_context(h_, k, ctx.setting_factors.data(), &ctx.sf_product));
  return ctx;
}

std::vector<Slea::Estimate> Slea::estimate_many(std::span<const uint32_t> aips,
                                                const EstimateContext& ctx) const {
  if (ctx.sf_product >= 1.0 - kSaturationEps)
    throw SaturationError("slea estimate: array saturated, setting-factor product ~ 1");
  sync();
  std::vector<uint64_t> w(aips.size());
  if (!aips.empty()) ok(srlg_slea_usle_weights(h_, ctx.k, aips.data(), aips.size(), w.data()));
  std::vector<Estimate> out(aips.size());
  for (size_t i = 0; i < aips.size(); ++i) {
    Estimate& e = out[i];
    e.usle_weight = w[i];
    e.sf_product = ctx.sf_product;
    e.corrected_weight = corrected_weight(static_cast<double>(w[i]), ctx.sf_product, cfg_.eta);
    const LinearEstimate le = le_estimate(e.corrected_weight, cfg_.eta);
    e.value = le.value;
    e.saturated = le.saturated;
  }
  return out;
}

Slea::Estimate Slea::estimate(uint32_t aip, const EstimateContext& ctx) const {
  return estimate_many(std::span<const uint32_t>(&aip, 1), ctx)[0];
}

Slea::Estimate Slea::estimate(uint32_t aip, uint32_t k) const {
  return estimate(aip, make_estimate_context(k));
}

std::span<const uint16_t> Slea::cells() const {
  sync();
  if (!mirror_valid_) {
    mirror_.resize(srlg_slea_num_cells(h_));
    ok(srlg_slea_export_cells(h_, mirror_.data(), mirror_.size()));
    mirror_valid_ = true;
  }
  return mirror_;
}

std::span<uint16_t> Slea::cells_mut() {
  cells();
  host_dirty_ = true;
  return mirror_;
}

std::span<const uint16_t> Slea::row(uint32_t i) const {
  if (i >= cfg_.r) throw std::out_of_range("slea: row out of range");
  return cells().subspan(static_cast<size_t>(i) * row_len_, row_len_);
}

std::span<const uint16_t> Slea::sle(uint32_t r, uint32_t j) const {
  if (r >= cfg_.r || j >= (uint64_t{1} << cfg_.q))
    throw std::out_of_range("slea: estimator out of range");
  return cells().subspan(static_cast<size_t>(r) * row_len_ + static_cast<size_t>(j) * cfg_.delta,
                         cfg_.eta);
}

std::string Slea::compatibility_mismatch(const Slea& o) const {
  char buf[64];
  ok(srlg_slea_compatibility_mismatch(h_, o.h_, buf, sizeof buf));
  return buf;
}

void Slea::merge_min(const Slea& o) {
  sync();
  ok(srlg_slea_merge_min(h_, o.handle()));
  mutated();
}

Slea merge(const Slea& a, const Slea& b) {
  Slea out = a;
  out.merge_min(b);
  return out;
}

// ----------------------------------------------------------------- config

srlg_params SketchParams::to_c() const {
  srlg_params p{};
  p.q = q;
  p.r = r;
  p.delta = delta;
  p.eta = eta;
  p.q_prime = q_prime;
  p.r_prime = r_prime;
  p.delta_prime = delta_prime;
  p.eta_prime = eta_prime;
  p.theta = theta;
  p.seed = seed;
  return p;
}

void SketchParams::validate() const {
  const srlg_params p = to_c();
  ok(srlg_params_validate(&p));
}

uint32_t SketchParams::tau() const { return sampling_threshold(theta, eta); }
HashSeeds SketchParams::seeds() const { return HashSeeds::derive(seed, r_prime); }

RsraConfig SketchParams::rsra_config() const {
  const srlg_params p = to_c();
  srlg_rsra_config c{};
  ok(srlg_params_rsra_config(&p, &c));
  return from_c(c);
}

SleaConfig SketchParams::slea_config() const {
  const srlg_params p = to_c();
  srlg_slea_config c{};
  ok(srlg_params_slea_config(&p, &c));
  return from_c(c);
}

namespace {
std::string trim(std::string s) {
  const char* ws = " \t\r";
  s.erase(0, s.find_first_not_of(ws));
  const size_t e = s.find_last_not_of(ws);
  s.erase(e == std::string::npos ? 0 : e + 1);
  return s;
}
}  // namespace

// key = value lines, '#' comments (src/config.cpp:74-112)
SketchParams SketchParams::parse(const std::string& text) {
  SketchParams p;
  std::istringstream in(text);
  std::string line;
  uint64_t lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    line = trim(line);
    if (line.empty() || line[0] == '#') continue;
    const size_t eq = line.find('=');
    if (eq == std::string::npos)
      throw ConfigError("parameter file line " + std::to_string(lineno) + ": expected key = value");
    const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
    try {
      uint64_t* u64 = nullptr;
      uint32_t* u32 = nullptr;
      if (key == "q") u32 = &p.q;
      else if (key == "r") u32 = &p.r;
      else if (key == "delta") u32 = &p.delta;
      else if (key == "eta") u32 = &p.eta;
      else if (key == "q_prime") u32 = &p.q_prime;
      else if (key == "r_prime") u32 = &p.r_prime;
      else if (key == "delta_prime") u32 = &p.delta_prime;
      else if (key == "eta_prime") u32 = &p.eta_prime;
      else if (key == "theta") u64 = &p.theta;
      else if (key == "seed") u64 = &p.seed;
      else throw ConfigError("parameter file: unknown key '" + key + "'");
      if (u32) *u32 = static_cast<uint32_t>(std::stoul(value));
      else *u64 = std::stoull(value);
    } catch (const ConfigError&) {
      throw;
    } catch (const std::exception&) {
      throw ConfigError("parameter file line " + std::to_string(lineno) + ": bad value for '" +
                        key + "'");
    }
  }
  return p;
}

SketchParams SketchParams::load_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ParseError("cannot open parameter file: " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return parse(ss.str());
}

// ---------------------------------------------------------- trace / report

std::string format_ipv4(uint32_t a) {
  return std::to_string(a >> 24) + '.' + std::to_string((a >> 16) & 255) + '.' +
         std::to_string((a >> 8) & 255) + '.' + std::to_string(a & 255);
}

void write_report_header(std::ostream& out) { out << "window_end_slice,aip,estimate,flags\n"; }

void write_report(const DetectionReport& r, std::ostream& out) {
  std::vector<ReportEntry> rows = r.entries;
  std::sort(rows.begin(), rows.end(), [](const ReportEntry& a, const ReportEntry& b) {
    if (a.estimate != b.estimate) return a.estimate > b.estimate;
    return a.aip < b.aip;
  });
  char est[32];
  for (const auto& e : rows) {
    std::snprintf(est, sizeof est, "%.2f", e.estimate);
    std::string flags;
    auto add = [&flags](const char* f) {
      if (!flags.empty()) flags += '|';
      flags += f;
    };
    if (r.partial) add("partial");
    if (e.saturated) add("saturated");
    if (r.overflow) add("overflow");
    out << r.window_end_slice << ',' << format_ipv4(e.aip) << ',' << est << ',' << flags << '\n';
  }
}

std::string report_to_csv(const std::vector<DetectionReport>& reports) {
  std::ostringstream out;
  write_report_header(out);
  for (const auto& r : reports) write_report(r, out);
  return out.str();
}

std::vector<DetectionReport> parse_report_blobs(std::span<const uint8_t> blob) {
  std::vector<DetectionReport> out;
  size_t off = 0;
  while (off + sizeof(srlg_report_header) <= blob.size()) {
    srlg_report_header h;
    std::memcpy(&h, blob.data() + off, sizeof h);
    off += sizeof h;
    DetectionReport r;
    r.window_end_slice = h.window_end_slice;
    r.candidate_count = h.candidate_count;
    r.sf_product = h.sf_product;
    r.partial = h.partial;
    r.overflow = h.overflow;
    r.slea_saturated = h.slea_saturated;
    r.hot_per_row.resize(h.n_rows);
    std::memcpy(r.hot_per_row.data(), blob.data() + off, 8 * h.n_rows);
    off += 8 * h.n_rows;
    for (uint32_t i = 0; i < h.n_entries; ++i) {
      srlg_entry e;
      std::memcpy(&e, blob.data() + off, sizeof e);
      off += sizeof e;
      r.entries.push_back(ReportEntry{e.aip, e.estimate, e.saturated != 0});
    }
    out.push_back(std::move(r));
  }
  return out;
}

// ---------------------------------------------------------- reconstruction

ReconstructResult reconstruct_candidates(const std::vector<std::vector<uint32_t>>& hot,
                                         const ReversibleHashGroup& g,
                                         const ReconstructOptions& opt) {
  if (hot.size() != g.r()) throw std::invalid_argument("reconstruct: expected one hot list per row");
  if (g.r() < 3) throw std::invalid_argument("reconstruct: need at least 3 rows");
  std::vector<uint32_t> flat;
  std::vector<uint64_t> counts;
  for (const auto& row : hot) {
    flat.insert(flat.end(), row.begin(), row.end());
    counts.push_back(row.size());
  }
  if (flat.empty()) flat.push_back(0);
  ReconstructResult res;
  uint64_t n = 0;
  int overflow = 0;
  std::vector<uint32_t> out(1 << 16);
  while (true) {
    ok(srlg_reconstruct_group(g.q(), g.r(), g.delta(), g.seed(), opt.device, flat.data(),
                              counts.data(), opt.tuple_cap, opt.work_cap, out.data(), out.size(),
                              &n, &overflow, &res.tuples_checked, &res.tuples_kept));
    if (n <= out.size()) break;
    out.resize(n);
  }
  out.resize(n);
  res.addresses = std::move(out);
  res.overflow = overflow != 0;
  return res;
}

// ------------------------------------------------------------------ window

srlg_window_config WindowConfig::to_c() const {
  srlg_window_config c;
  srlg_window_config_default(&c);
  c.has_t0 = t0_us.has_value();
  c.t0_us = t0_us.value_or(0);
  c.slice_us = slice_us;
  c.k = k;
  c.theta = theta;
  c.reinit_per_window = reinit_per_window;
  c.regression_tolerance_us = regression_tolerance_us;
  c.keep_below_threshold = keep_below_threshold;
  c.workers = workers;
  c.tuple_cap = tuple_cap;
  return c;
}

void WindowConfig::validate() const {
  const srlg_window_config c = to_c();
  ok(srlg_window_config_validate(&c));
}

uint64_t slice_index(uint64_t ts_us, uint64_t t0_us, uint64_t slice_us) {
  if (ts_us < t0_us) throw OrderingError("timestamp precedes the stream start");
  return (ts_us - t0_us) / slice_us;
}

uint64_t SliceClock::place(uint64_t ts_us) {
  if (!t0_) t0_ = ts_us;
  if (max_ts_ && ts_us < *max_ts_) {
    if (*max_ts_ - ts_us > tolerance_us_)
      throw OrderingError("timestamp regression beyond tolerance");
    ++clamped_;
    return slice_index(*max_ts_, *t0_, slice_us_);
  }
  if (!max_ts_ || ts_us > *max_ts_) max_ts_ = ts_us;
  return slice_index(ts_us, *t0_, slice_us_);
}

DetectionReport run_detection(const Rsra& rsra, const Slea& slea, uint64_t window_end_slice,
                              bool partial, const WindowConfig& cfg) {
  const srlg_window_config c = cfg.to_c();
  std::vector<uint8_t> blob(1 << 16);
  uint64_t n = 0;
  while (true) {
    ok(srlg_detect(rsra.handle(), slea.handle(), &c, window_end_slice, partial, blob.data(),
                   blob.size(), &n));
    if (n <= blob.size()) break;
    blob.resize(n);
  }
  blob.resize(n);
  return parse_report_blobs(blob).at(0);
}

WindowEngine::WindowEngine(const WindowConfig& cfg, Rsra rsra, Slea slea, ReportSink sink)
    : cfg_(cfg), sink_(std::move(sink)), device_(rsra.device()) {
  cfg_.validate();
  const srlg_window_config c = cfg_.to_c();
  srlg_rsra* r = rsra.release();
  srlg_slea* s = slea.release();
  const int st = srlg_engine_create(&c, r, s, &e_);
  if (st != SRLG_OK) {
    srlg_rsra_destroy(r);
    srlg_slea_destroy(s);
    throw_status(st);
  }
}

WindowEngine::WindowEngine(const WindowEngine& other)
    : cfg_(other.cfg_), sink_(other.sink_), device_(other.device_) {
  // the reference delivers a slice's report before the copy can be taken:
  // hand the source's finished reports to its own sink first
  const_cast<WindowEngine&>(other).deliver();
  ok(srlg_engine_clone(other.e_, &e_));
}

WindowEngine& WindowEngine::operator=(const WindowEngine& other) {
  if (this == &other) return *this;
  const_cast<WindowEngine&>(other).deliver();
  srlg_engine* copy = nullptr;
  ok(srlg_engine_clone(other.e_, &copy));
  rsra_view_.reset();
  slea_view_.reset();
  srlg_engine_destroy(e_);
  e_ = copy;
  cfg_ = other.cfg_;
  sink_ = other.sink_;
  device_ = other.device_;
  return *this;
}

WindowEngine::~WindowEngine() {
  rsra_view_.reset();
  slea_view_.reset();
  srlg_engine_destroy(e_);
}

// hands finished reports to the sink, in order
void WindowEngine::deliver() {
  uint64_t need = 0, n = 0;
  ok(srlg_engine_take_reports(e_, nullptr, 0, &need, &n));
  if (!need) return;
  std::vector<uint8_t> blob(need);
  ok(srlg_engine_take_reports(e_, blob.data(), blob.size(), &need, &n));
  if (!sink_) return;
  for (const auto& r : parse_report_blobs(blob)) sink_(r);
}

void WindowEngine::process(const TraceRecord& rec) {
  const uint64_t before = srlg_engine_current_slice(e_);
  const srlg_record r{rec.ts_us, rec.aip, rec.bip};
  ok(srlg_engine_process(e_, &r, 1));
  if (srlg_engine_current_slice(e_) != before) deliver();
}

void WindowEngine::process_batch(std::span<const TraceRecord> recs) {
  static_assert(sizeof(TraceRecord) == sizeof(srlg_record));
  ok(srlg_engine_process(e_, reinterpret_cast<const srlg_record*>(recs.data()), recs.size()));
  deliver();
}

void WindowEngine::process_slices(std::span<const srlg_pair> pairs,
                                  std::span<const uint64_t> offsets, uint64_t first_slice) {
  ok(srlg_engine_process_slices(e_, pairs.data(), offsets.data(), offsets.size() - 1, first_slice,
                                0));
  deliver();
}

void WindowEngine::advance_to_slice(uint64_t slice) {
  ok(srlg_engine_advance_to_slice(e_, slice));
  deliver();
}

void WindowEngine::finish() {
  ok(srlg_engine_finish(e_));
  deliver();
}

const Rsra& WindowEngine::rsra() const {
  ok(srlg_engine_sync(e_));
  rsra_view_ = std::make_unique<Rsra>(Rsra::view(srlg_engine_rsra(e_), device_));
  return *rsra_view_;
}

const Slea& WindowEngine::slea() const {
  ok(srlg_engine_sync(e_));
  slea_view_ = std::make_unique<Slea>(Slea::view(srlg_engine_slea(e_), device_));
  return *slea_view_;
}

uint64_t WindowEngine::current_slice() const { return srlg_engine_current_slice(e_); }
uint64_t WindowEngine::records() const { return srlg_engine_records(e_); }
uint64_t WindowEngine::clamped() const { return srlg_engine_clamped(e_); }

// ------------------------------------------------------------- distributed

PartitionPolicy parse_partition_policy(std::string_view name) {
  if (name == "hash-pair") return PartitionPolicy::hash_pair;
  if (name == "round-robin") return PartitionPolicy::round_robin;
  if (name == "by-source-prefix") return PartitionPolicy::by_source_prefix;
  throw ConfigError("unknown partition policy: " + std::string(name));
}

namespace {
uint32_t route(const TraceRecord& rec, uint64_t index, PartitionPolicy policy, uint32_t nodes) {
  switch (policy) {
    case PartitionPolicy::hash_pair:
      return static_cast<uint32_t>(
          hash64((static_cast<uint64_t>(rec.aip) << 32) | rec.bip, 0x70617274) % nodes);
    case PartitionPolicy::round_robin:
      return static_cast<uint32_t>(index % nodes);
    case PartitionPolicy::by_source_prefix:
      return (rec.aip >> 24) % nodes;
  }
  return 0;
}
}  // namespace

// run_distributed (src/distributed.cpp:35-117) with device sketches. The
// records are first placed on the slice clock (SliceClock::place, the same
// sequential rule: t0 = first record, clamped regressions) and bucketed per
// slice and node; the slices are then replayed in order: every node's batch
// of the slice is one fused scan, a completed slice from k-1 on is detected
// on the merged global (a device copy of node 0, max-merged in stamp space
// with the other nodes), then every node slides (or reinitialises). The
// stream's last slice is reported partial.
std::vector<DetectionReport> run_distributed(std::span<const TraceRecord> records,
                                             const WindowConfig& cfg, const RsraConfig& rsra_cfg,
                                             const SleaConfig& slea_cfg,
                                             const DistributedOptions& opt,
                                             DistributedStats* stats) {
  cfg.validate();
  if (opt.nodes == 0) throw ConfigError("distributed run needs at least one node");
  std::vector<DetectionReport> reports;
  if (records.empty()) return reports;
  const uint32_t n_nodes = opt.nodes;

  // slice of every record, then (slice, node) buckets in record order
  SliceClock clock(cfg.t0_us, cfg.slice_us, cfg.regression_tolerance_us);
  std::vector<uint64_t> slice_of(records.size());
  for (size_t i = 0; i < records.size(); ++i) slice_of[i] = clock.place(records[i].ts_us);
  const uint64_t last = slice_of.back();
  std::vector<std::vector<std::vector<srlg_pair>>> batch(n_nodes);
  for (auto& per_node : batch) per_node.resize(last + 1);
  for (size_t i = 0; i < records.size(); ++i)
    batch[route(records[i], i, opt.policy, n_nodes)][slice_of[i]].push_back(
        srlg_pair{records[i].aip, records[i].bip});

  std::vector<Rsra> rs;
  std::vector<Slea> le;
  for (uint32_t n = 0; n < n_nodes; ++n) {
    const int dev = static_cast<int>(n % std::max<uint32_t>(1, opt.devices));
    rs.emplace_back(rsra_cfg, dev);
    le.emplace_back(slea_cfg, dev);
  }
  const uint64_t exchanged = n_nodes * (serialized_size(rs[0]) + serialized_size(le[0]));
  for (uint64_t s = 0; s <= last; ++s) {
    for (uint32_t n = 0; n < n_nodes; ++n) {
      const auto& b = batch[n][s];
      if (!b.empty())
        ok(srlg_update_pairs(rs[n].handle(), le[n].handle(), b.data(), b.size(), 0, nullptr));
    }
    const bool partial = s == last;
    if (partial || s + 1 >= cfg.k) {  // the transient global of this slice
      Rsra global_rs = rs[0];
      Slea global_le = le[0];
      for (uint32_t n = 1; n < n_nodes; ++n) {
        global_rs.merge_min(rs[n]);
        global_le.merge_min(le[n]);
      }
      if (stats) {
        ++stats->slice_merges;
        stats->bytes_exchanged += exchanged;
      }
      reports.push_back(run_detection(global_rs, global_le, s, partial, cfg));
    }
    if (partial) break;
    for (uint32_t n = 0; n < n_nodes; ++n) {
      if (cfg.reinit_per_window) {
        rs[n].reinitialize();
        le[n].reinitialize();
      } else {
        rs[n].slide();
        le[n].slide();
      }
    }
  }
  return reports;
}

}  // namespace slidecard

// ====================================================== sketch streams
// sketch_io.cpp:106-180 over the C ABI (srlg_*_serialize and create +
// import_cells), reading exactly one stream from `in` like the reference.
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <istream>
#include <ostream>

#include "slidecard/sketch_io.hpp"

namespace slidecard {

namespace {

void read_exact(std::istream& in, void* p, size_t n, const char* what) {
  if (!in.read(static_cast<char*>(p), static_cast<std::streamsize>(n))) throw FormatError(what);
}

template <class T>
T get_le(std::istream& in) {
  T v{};
  read_exact(in, &v, sizeof(T), "sketch stream truncated");  // little-endian host (srlg.h)
  return v;
}

template <class H, class Ser>
void write_stream(const H* h, uint64_t n, Ser ser, std::ostream& out) {
  std::vector<uint8_t> buf(n);
  uint64_t w = 0;
  ok(ser(h, buf.data(), n, &w));
  out.write(reinterpret_cast<const char*>(buf.data()), static_cast<std::streamsize>(w));
  if (!out) throw FormatError("sketch write failed");
}

}  // namespace

uint64_t serialized_size(const Rsra& s) { return srlg_rsra_serialized_size(s.handle()); }
uint64_t serialized_size(const Slea& s) { return srlg_slea_serialized_size(s.handle()); }

void serialize_sketch(const Rsra& s, std::ostream& out) {
  write_stream(s.handle(), serialized_size(s), srlg_rsra_serialize, out);
}

void serialize_sketch(const Slea& s, std::ostream& out) {
  write_stream(s.handle(), serialized_size(s), srlg_slea_serialize, out);
}

void serialize_sketch(const AnySketch& s, std::ostream& out) {
  std::visit([&out](const auto& v) { serialize_sketch(v, out); }, s);
}

AnySketch deserialize_sketch(std::istream& in, int device) {
  char magic[4];
  read_exact(in, magic, 4, "sketch stream truncated");
  if (!std::equal(magic, magic + 4, kSketchMagic)) throw FormatError("bad sketch magic");
  const uint16_t version = get_le<uint16_t>(in);
  if (version != kSketchVersion)
    throw FormatError("unsupported sketch format version " + std::to_string(version));
  const int t = in.get();
  if (t != static_cast<int>(SketchType::rsra) && t != static_cast<int>(SketchType::slea))
    throw FormatError("unknown sketch type tag");
  if (t == static_cast<int>(SketchType::rsra)) {
    RsraConfig cfg;
    cfg.q = get_le<uint32_t>(in);
    cfg.r = get_le<uint32_t>(in);
    cfg.delta = get_le<uint32_t>(in);
    cfg.eta = get_le<uint32_t>(in);
    cfg.tau = get_le<uint32_t>(in);
    cfg.seed_h1 = get_le<uint64_t>(in);
    cfg.seed_h2 = get_le<uint64_t>(in);
    cfg.seed_rhfg0 = get_le<uint64_t>(in);
    const uint64_t slides = get_le<uint64_t>(in);
    Rsra s(cfg, device);  // ConfigError as the reference's constructor
    const uint64_t n = srlg_rsra_num_cells(s.handle());
    std::vector<uint16_t> cells(n);
    read_exact(in, cells.data(), 2 * n, "sketch stream truncated in counter block");
    ok(srlg_rsra_import_cells(s.handle(), cells.data(), n));
    ok(srlg_rsra_set_slides(s.handle(), slides));
    return Rsra::adopt(s.release(), device);
  }
  SleaConfig cfg;
  cfg.q = get_le<uint32_t>(in);
  cfg.r = get_le<uint32_t>(in);
  cfg.delta = get_le<uint32_t>(in);
  cfg.eta = get_le<uint32_t>(in);
  if (cfg.r > 64) throw FormatError("sketch stream declares too many rows");
  cfg.seeds_lh.resize(cfg.r);
  cfg.seed_h3 = get_le<uint64_t>(in);
  for (auto& seed : cfg.seeds_lh) seed = get_le<uint64_t>(in);
  const uint64_t slides = get_le<uint64_t>(in);
  Slea s(cfg, device);
  const uint64_t n = srlg_slea_num_cells(s.handle());
  std::vector<uint16_t> cells(n);
  read_exact(in, cells.data(), 2 * n, "sketch stream truncated in counter block");
  ok(srlg_slea_import_cells(s.handle(), cells.data(), n));
  ok(srlg_slea_set_slides(s.handle(), slides));
  return Slea::adopt(s.release(), device);
}

AnySketch load_sketch_file(const std::string& path, int device) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw ParseError("cannot open sketch file: " + path);
  try {
    return deserialize_sketch(in, device);
  } catch (const FormatError& e) {
    throw FormatError(path + ": " + e.what());
  }
}

// Replace `path` atomically (io_util.cpp write_file_atomic's contract): the
// stream is serialised in memory first, written to a sibling file named after
// the process, flushed to disk, then renamed over `path`; a failure removes
// the sibling and raises ResourceError.
void save_sketch_file(const AnySketch& s, const std::string& path) {
  std::ostringstream buf(std::ios::binary);
  serialize_sketch(s, buf);
  const std::string bytes = buf.str();
  const std::string side = path + ".part-" + std::to_string(::getpid());
  std::FILE* f = std::fopen(side.c_str(), "wb");
  if (!f) throw ResourceError("cannot open output file: " + side);
  const bool written = std::fwrite(bytes.data(), 1, bytes.size(), f) == bytes.size() &&
                       std::fflush(f) == 0 && ::fsync(::fileno(f)) == 0;
  const bool closed = std::fclose(f) == 0;
  std::error_code ec;
  if (written && closed) std::filesystem::rename(side, path, ec);
  if (!written || !closed || ec) {
    std::filesystem::remove(side);
    throw ResourceError("cannot write " + path + (ec ? ": " + ec.message() : std::string()));
  }
}

}  // namespace slidecard

// ============================================================ ingest
#include "slidecard/trace.hpp"

namespace slidecard {

void WindowEngine::set_anet(const srlg_anet* anet) { ok(srlg_engine_set_anet(e_, anet)); }

srlg_anet AnetSpec::to_c() const {
  if (prefixes.size() > SRLG_MAX_PREFIXES)
    throw ConfigError("monitored network: at most " + std::to_string(SRLG_MAX_PREFIXES) +
                      " prefixes on the device path");
  srlg_anet a{};
  a.n = static_cast<uint32_t>(prefixes.size());
  for (size_t i = 0; i < prefixes.size(); ++i) {
    a.addr[i] = prefixes[i].addr;
    a.bits[i] = prefixes[i].bits;
  }
  return a;
}

}  // namespace slidecard

// ========================================================= exact oracle
#include "slidecard/exact_oracle.hpp"

namespace slidecard {

std::vector<TruthWindow> exact_detect_slices(std::span<const srlg_pair> pairs,
                                             std::span<const uint64_t> offsets,
                                             const ExactOptions& opt) {
  srlg_exact* e = nullptr;
  ok(srlg_exact_create(opt.theta, opt.k, opt.max_pairs, opt.device, &e));
  std::unique_ptr<srlg_exact, void (*)(srlg_exact*)> guard(e, srlg_exact_destroy);
  ok(srlg_exact_process_slices(e, pairs.data(), offsets.data(), offsets.size() - 1, 0, 0));
  ok(srlg_exact_finish(e));
  uint64_t bytes = 0, n = 0;
  ok(srlg_exact_take_windows(e, nullptr, 0, &bytes, &n));
  std::vector<uint8_t> blob(bytes);
  ok(srlg_exact_take_windows(e, blob.data(), bytes, &bytes, &n));
  std::vector<TruthWindow> out;
  size_t off = 0;
  while (off < blob.size()) {
    TruthWindow w;
    uint32_t partial = 0, cnt = 0;
    std::memcpy(&w.window_end_slice, blob.data() + off, 8);
    std::memcpy(&partial, blob.data() + off + 8, 4);
    std::memcpy(&cnt, blob.data() + off + 12, 4);
    off += 16;
    w.partial = partial != 0;
    for (uint32_t i = 0; i < cnt; ++i, off += 16) {
      TruthEntry t;
      std::memcpy(&t.aip, blob.data() + off, 4);
      std::memcpy(&t.cardinality, blob.data() + off + 8, 8);
      w.supers.push_back(t);
    }
    out.push_back(std::move(w));
  }
  return out;
}

// score (exact_oracle.cpp:105-132): false positives are detected hosts
// outside the truth, false negatives true hosts never detected; the rates
// are relative to the number of true hosts (the reference's definitions)
AccuracyResult score(uint64_t window_end_slice, std::span<const uint32_t> detected,
                     std::span<const TruthEntry> truth) {
  std::vector<uint32_t> got(detected.begin(), detected.end());
  std::sort(got.begin(), got.end());
  got.erase(std::unique(got.begin(), got.end()), got.end());
  std::vector<uint32_t> want;
  want.reserve(truth.size());
  std::transform(truth.begin(), truth.end(), std::back_inserter(want),
                 [](const TruthEntry& t) { return t.aip; });
  std::sort(want.begin(), want.end());
  std::vector<uint32_t> only_got, only_want;
  std::set_difference(got.begin(), got.end(), want.begin(), want.end(),
                      std::back_inserter(only_got));
  std::set_difference(want.begin(), want.end(), got.begin(), got.end(),
                      std::back_inserter(only_want));
  AccuracyResult r;
  r.window_end_slice = window_end_slice;
  r.n_true = truth.size();
  r.n_detected = detected.size();
  r.n_false_pos = only_got.size();
  r.n_false_neg = only_want.size();
  if (r.n_true) {
    const double t = static_cast<double>(r.n_true);
    r.defined = true;
    r.fpr = static_cast<double>(r.n_false_pos) / t;
    r.fnr = static_cast<double>(r.n_false_neg) / t;
    r.tfr = r.fpr + r.fnr;
  }
  return r;
}

}  // namespace slidecard
