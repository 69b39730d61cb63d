// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// An extern "C" face over the UNMODIFIED reference library (slidecard,
// /root/reference/proj/core/src/*.cpp compiled in place by oracle/Makefile into
// oracle/_ref/libslidecard_ref.so). Every function forwards to the reference's
// own public C++ API; nothing here re-implements reference behaviour except
// the report-blob serialisation shared with include/srlg.h.
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / the
// --impl reference arm) may load this library.

#include <algorithm>
#include <array>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <sstream>
#include <string>
#include <thread>
#include <variant>
#include <vector>

#include "slidecard/config.hpp"
#include "slidecard/exact_oracle.hpp"
#include "slidecard/distributed.hpp"
#include "slidecard/errors.hpp"
#include "slidecard/hash.hpp"
#include "slidecard/linear_counting.hpp"
#include "slidecard/parallel.hpp"
#include "slidecard/reconstruct.hpp"
#include "slidecard/report.hpp"
#include "slidecard/rng.hpp"
#include "slidecard/rsra.hpp"
#include "slidecard/sketch_io.hpp"
#include "slidecard/trace.hpp"
#include "slidecard/slea.hpp"
#include "slidecard/window.hpp"

#include "srlg.h"

using namespace slidecard;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SRLG_OK;
  } catch (const ConfigError& e) {
    return fail(SRLG_ERR_CONFIG, e.what());
  } catch (const OrderingError& e) {
    return fail(SRLG_ERR_ORDERING, e.what());
  } catch (const FormatError& e) {
    return fail(SRLG_ERR_FORMAT, e.what());
  } catch (const ParseError& e) {
    return fail(SRLG_ERR_PARSE, e.what());
  } catch (const ResourceError& e) {
    return fail(SRLG_ERR_RESOURCE, e.what());
  } catch (const IncompatibleSketchError& e) {
    return fail(SRLG_ERR_INCOMPATIBLE, e.what());
  } catch (const SaturationError& e) {
    return fail(SRLG_ERR_SATURATION, e.what());
  } catch (const std::out_of_range& e) {
    return fail(SRLG_ERR_OUT_OF_RANGE, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(SRLG_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::exception& e) {
    return fail(SRLG_ERR_RESOURCE, e.what());
  }
}

SketchParams to_params(const srlg_params* p) {
  SketchParams s;
  s.q = p->q;
  s.r = p->r;
  s.delta = p->delta;
  s.eta = p->eta;
  s.q_prime = p->q_prime;
  s.r_prime = p->r_prime;
  s.delta_prime = p->delta_prime;
  s.eta_prime = p->eta_prime;
  s.theta = p->theta;
  s.seed = p->seed;
  return s;
}

WindowConfig to_window(const srlg_window_config* c) {
  WindowConfig w;
  if (c->has_t0) w.t0_us = c->t0_us;
  w.slice_us = c->slice_us;
  w.k = c->k;
  w.theta = c->theta;
  w.reinit_per_window = c->reinit_per_window != 0;
  w.regression_tolerance_us = c->regression_tolerance_us;
  w.keep_below_threshold = c->keep_below_threshold != 0;
  w.workers = c->workers;
  w.tuple_cap = c->tuple_cap;
  return w;
}

void append_blob(std::vector<uint8_t>& out, const DetectionReport& r) {
  srlg_report_header h{};
  h.window_end_slice = r.window_end_slice;
  h.candidate_count = r.candidate_count;
  h.sf_product = r.sf_product;
  h.n_rows = static_cast<uint32_t>(r.hot_per_row.size());
  h.n_entries = static_cast<uint32_t>(r.entries.size());
  h.partial = r.partial;
  h.overflow = r.overflow;
  h.slea_saturated = r.slea_saturated;
  const size_t base = out.size();
  out.resize(base + sizeof(h) + 8 * r.hot_per_row.size() + sizeof(srlg_entry) * r.entries.size());
  uint8_t* p = out.data() + base;
  std::memcpy(p, &h, sizeof(h));
  p += sizeof(h);
  for (uint64_t v : r.hot_per_row) {
    std::memcpy(p, &v, 8);
    p += 8;
  }
  for (const auto& e : r.entries) {
    srlg_entry x{};
    x.aip = e.aip;
    x.saturated = e.saturated;
    x.estimate = e.estimate;
    std::memcpy(p, &x, sizeof(x));
    p += sizeof(x);
  }
}

uint64_t emit_blobs(const std::vector<DetectionReport>& reps, uint8_t* blob, uint64_t cap,
                    uint64_t* n_reports) {
  std::vector<uint8_t> buf;
  for (const auto& r : reps) append_blob(buf, r);
  if (n_reports) *n_reports = reps.size();
  if (blob && buf.size() <= cap) std::memcpy(blob, buf.data(), buf.size());
  return buf.size();
}

struct Sketch {
  Rsra rsra;
  Slea slea;
};

struct Engine {
  WindowConfig cfg;
  std::vector<DetectionReport> reports;
  std::unique_ptr<WindowEngine> engine;
};

// The engine's sink appends to whichever Engine the current API call drives;
// this keeps copies (ref_engine_clone) reporting into their own list.
thread_local Engine* g_current = nullptr;

void sink_to_current(const DetectionReport& r) { g_current->reports.push_back(r); }

ReversibleHashGroup group_of(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed) {
  return ReversibleHashGroup(q, r, delta, seed);
}

}  // namespace

#pragma GCC visibility push(default)
extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix64(uint64_t x) { return mix64(x); }
uint64_t ref_hash64(uint64_t key, uint64_t seed) { return hash64(key, seed); }
uint32_t ref_sampling_threshold(uint64_t theta, uint64_t eta) {
  return sampling_threshold(theta, eta);
}
uint32_t ref_lsb(uint32_t x) { return lsb(x); }
double ref_detection_rho() { return detection_rho(); }

int ref_le_estimate(double weight, uint32_t eta_prime, double* value, int* saturated) {
  return guarded([&] {
    const auto le = le_estimate(weight, eta_prime);
    *value = le.value;
    *saturated = le.saturated;
  });
}

int ref_corrected_weight(double w, double sfp, uint32_t eta_prime, double* out) {
  return guarded([&] { *out = corrected_weight(w, sfp, eta_prime); });
}

int ref_params_configs(const srlg_params* p, srlg_rsra_config* rc, srlg_slea_config* sc) {
  return guarded([&] {
    const SketchParams s = to_params(p);
    s.validate();
    const RsraConfig r = s.rsra_config();
    const SleaConfig l = s.slea_config();
    *rc = srlg_rsra_config{};
    rc->q = r.q;
    rc->r = r.r;
    rc->delta = r.delta;
    rc->eta = r.eta;
    rc->tau = r.tau;
    rc->seed_h1 = r.seed_h1;
    rc->seed_h2 = r.seed_h2;
    rc->seed_rhfg0 = r.seed_rhfg0;
    *sc = srlg_slea_config{};
    sc->q = l.q;
    sc->r = l.r;
    sc->delta = l.delta;
    sc->eta = l.eta;
    sc->seed_h3 = l.seed_h3;
    for (size_t i = 0; i < l.seeds_lh.size(); ++i) sc->seeds_lh[i] = l.seeds_lh[i];
  });
}

int ref_params_validate(const srlg_params* p) {
  return guarded([&] { to_params(p).validate(); });
}

// ------------------------------------------------------------------ sketches

void* ref_sketch_create(const srlg_params* p) {
  Sketch* out = nullptr;
  const int rc = guarded([&] {
    const SketchParams s = to_params(p);
    s.validate();
    out = new Sketch{Rsra(s.rsra_config()), Slea(s.slea_config())};
  });
  return rc == SRLG_OK ? out : nullptr;
}

void* ref_sketch_clone(const void* h) { return new Sketch(*static_cast<const Sketch*>(h)); }
void ref_sketch_destroy(void* h) { delete static_cast<Sketch*>(h); }

// the WindowEngine::flush_pending body (src/window.cpp:89-98)
int ref_update(void* h, const srlg_pair* pairs, uint64_t n, uint32_t workers) {
  auto* s = static_cast<Sketch*>(h);
  return guarded([&] {
    parallel_chunks(n, workers, [&](size_t, size_t begin, size_t end) {
      for (size_t i = begin; i < end; ++i) {
        s->rsra.update(pairs[i].aip, pairs[i].bip);
        s->slea.update(pairs[i].aip, pairs[i].bip);
      }
    });
  });
}

int ref_update_rsra_only(void* h, const srlg_pair* pairs, uint64_t n) {
  auto* s = static_cast<Sketch*>(h);
  return guarded([&] {
    for (uint64_t i = 0; i < n; ++i) s->rsra.update(pairs[i].aip, pairs[i].bip);
  });
}

int ref_update_slea_only(void* h, const srlg_pair* pairs, uint64_t n) {
  auto* s = static_cast<Sketch*>(h);
  return guarded([&] {
    for (uint64_t i = 0; i < n; ++i) s->slea.update(pairs[i].aip, pairs[i].bip);
  });
}

void ref_slide(void* h) {
  auto* s = static_cast<Sketch*>(h);
  s->rsra.slide();
  s->slea.slide();
}

void ref_reinit(void* h) {
  auto* s = static_cast<Sketch*>(h);
  s->rsra.reinitialize();
  s->slea.reinitialize();
}

uint64_t ref_slides(const void* h) { return static_cast<const Sketch*>(h)->rsra.slides(); }
void ref_set_slides(void* h, uint64_t v) {
  auto* s = static_cast<Sketch*>(h);
  s->rsra.set_slides(v);
  s->slea.set_slides(v);
}
uint64_t ref_rsra_ncells(const void* h) { return static_cast<const Sketch*>(h)->rsra.cells().size(); }
uint64_t ref_slea_ncells(const void* h) { return static_cast<const Sketch*>(h)->slea.cells().size(); }
uint64_t ref_slea_row_length(const void* h) {
  return static_cast<const Sketch*>(h)->slea.row_length();
}

void ref_export(const void* h, uint16_t* rsra, uint16_t* slea) {
  const auto* s = static_cast<const Sketch*>(h);
  if (rsra) std::copy(s->rsra.cells().begin(), s->rsra.cells().end(), rsra);
  if (slea) std::copy(s->slea.cells().begin(), s->slea.cells().end(), slea);
}

void ref_import(void* h, const uint16_t* rsra, const uint16_t* slea) {
  auto* s = static_cast<Sketch*>(h);
  if (rsra) std::copy(rsra, rsra + s->rsra.cells().size(), s->rsra.cells_mut().begin());
  if (slea) std::copy(slea, slea + s->slea.cells().size(), s->slea.cells_mut().begin());
}

// deserialize_sketch (sketch_io.cpp:144-175): type, slides and the u16
// counters of one stream
int ref_deserialize(const uint8_t* in, uint64_t n, int* type, uint16_t* cells, uint64_t cap,
                    uint64_t* ncells, uint64_t* slides) {
  return guarded([&] {
    std::istringstream is(std::string(reinterpret_cast<const char*>(in), n));
    const AnySketch a = deserialize_sketch(is);
    *type = static_cast<int>(a.index()) + 1;
    std::visit(
        [&](const auto& s) {
          const auto c = s.cells();
          *ncells = c.size();
          *slides = s.slides();
          if (cells && cap >= c.size()) std::memcpy(cells, c.data(), c.size() * sizeof(uint16_t));
        },
        a);
  });
}

// classify (trace.cpp:111-116) with the reference's AnetSpec / CidrPrefix:
// raw packets {src, dst} -> records {aip, bip}; *n_out records written
int ref_classify(const srlg_pair* raw, uint64_t n, const srlg_anet* a, srlg_pair* out,
                 uint64_t* n_out) {
  return guarded([&] {
    AnetSpec spec;
    for (uint32_t i = 0; i < a->n; ++i) spec.prefixes.push_back(CidrPrefix{a->addr[i], a->bits[i]});
    uint64_t k = 0;
    std::array<TraceRecord, 2> recs;
    for (uint64_t i = 0; i < n; ++i) {
      const int m = classify(RawPacket{0, raw[i].aip, raw[i].bip}, spec, recs);
      for (int j = 0; j < m; ++j) out[k++] = srlg_pair{recs[j].aip, recs[j].bip};
    }
    *n_out = k;
  });
}

// exact_detect (exact_oracle.cpp:92-101) over pre-sliced pairs (slice j at
// ts = t0 + j * 1 s): windows in the srlg_exact_take_windows blob layout
int ref_exact_detect(const srlg_pair* pairs, const uint64_t* offsets, uint64_t n_slices,
                     uint64_t theta, uint32_t k, uint8_t* blob, uint64_t cap, uint64_t* bytes) {
  return guarded([&] {
    ExactSlidingOracle::Options opt;
    opt.theta = theta;
    opt.k = k;
    opt.t0_us = 0;
    opt.slice_us = 1'000'000;
    std::vector<TraceRecord> recs;
    recs.reserve(offsets[n_slices]);
    for (uint64_t j = 0; j < n_slices; ++j)
      for (uint64_t i = offsets[j]; i < offsets[j + 1]; ++i)
        recs.push_back(TraceRecord{j * 1'000'000, pairs[i].aip, pairs[i].bip});
    const auto wins = exact_detect(recs, opt);
    std::vector<uint8_t> out;
    auto put = [&out](const void* p, size_t n) {
      const auto* b = static_cast<const uint8_t*>(p);
      out.insert(out.end(), b, b + n);
    };
    for (const auto& w : wins) {
      const uint64_t end = w.window_end_slice;
      const uint32_t part = w.partial ? 1u : 0u, n = static_cast<uint32_t>(w.supers.size()), z = 0;
      put(&end, 8);
      put(&part, 4);
      put(&n, 4);
      for (const auto& t : w.supers) {
        put(&t.aip, 4);
        put(&z, 4);
        put(&t.cardinality, 8);
      }
    }
    *bytes = out.size();
    if (blob && cap >= out.size()) std::memcpy(blob, out.data(), out.size());
  });
}

int ref_merge_min(void* a, const void* b) {
  auto* x = static_cast<Sketch*>(a);
  const auto* y = static_cast<const Sketch*>(b);
  return guarded([&] {
    x->rsra.merge_min(y->rsra);
    x->slea.merge_min(y->slea);
  });
}

int ref_extract_hot(const void* h, uint32_t k, uint32_t* cols, uint64_t cap,
                    uint64_t* row_counts) {
  const auto* s = static_cast<const Sketch*>(h);
  return guarded([&] {
    const auto hot = s->rsra.extract_hot(k);
    uint64_t off = 0;
    for (size_t i = 0; i < hot.size(); ++i) {
      row_counts[i] = hot[i].size();
      for (uint32_t c : hot[i]) {
        if (off < cap) cols[off] = c;
        ++off;
      }
    }
    if (off > cap) throw ResourceError("hot list buffer too small");
  });
}

int ref_estimate_context(const void* h, uint32_t k, double* factors, double* sfp) {
  const auto* s = static_cast<const Sketch*>(h);
  return guarded([&] {
    const auto ctx = s->slea.make_estimate_context(k);
    for (size_t i = 0; i < ctx.setting_factors.size(); ++i) factors[i] = ctx.setting_factors[i];
    *sfp = ctx.sf_product;
  });
}

int ref_estimate(const void* h, uint32_t aip, uint32_t k, srlg_estimate* out) {
  const auto* s = static_cast<const Sketch*>(h);
  return guarded([&] {
    const auto est = s->slea.estimate(aip, k);
    *out = srlg_estimate{};
    out->value = est.value;
    out->corrected_weight = est.corrected_weight;
    out->usle_weight = est.usle_weight;
    out->sf_product = est.sf_product;
    out->saturated = est.saturated;
  });
}

uint32_t ref_lh_column(const void* h, uint32_t row, uint32_t aip) {
  return static_cast<const Sketch*>(h)->slea.lh_column(row, aip);
}

int ref_forward(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t aip,
                uint32_t* cols) {
  return guarded([&] { group_of(q, r, delta, seed).forward(aip, {cols, r}); });
}

int ref_group_info(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t* uncovered,
                   int* covers) {
  return guarded([&] {
    const auto g = group_of(q, r, delta, seed);
    *uncovered = g.uncovered_mask();
    *covers = g.covers_address();
  });
}

int ref_invert(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, const uint32_t* cols,
               uint32_t* out, uint64_t cap, uint64_t* n) {
  return guarded([&] {
    const auto v = group_of(q, r, delta, seed).invert({cols, r});
    *n = v.size();
    for (size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
  });
}

int ref_reconstruct(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed,
                    const uint32_t* hot_cols, const uint64_t* row_counts, uint64_t tuple_cap,
                    uint64_t work_cap, uint32_t workers, uint32_t* out, uint64_t cap,
                    uint64_t* n, int* overflow, uint64_t* checked, uint64_t* kept) {
  return guarded([&] {
    const auto g = group_of(q, r, delta, seed);
    std::vector<std::vector<uint32_t>> hot(r);
    uint64_t off = 0;
    for (uint32_t i = 0; i < r; ++i) {
      hot[i].assign(hot_cols + off, hot_cols + off + row_counts[i]);
      off += row_counts[i];
    }
    ReconstructOptions opt;
    opt.tuple_cap = tuple_cap;
    opt.work_cap = work_cap;
    opt.workers = workers;
    const auto res = reconstruct_candidates(hot, g, opt);
    *n = res.addresses.size();
    for (size_t i = 0; i < res.addresses.size() && i < cap; ++i) out[i] = res.addresses[i];
    *overflow = res.overflow;
    *checked = res.tuples_checked;
    *kept = res.tuples_kept;
  });
}

// run_detection (src/window.cpp:36-78) on the sketch's current state
int ref_detect(const void* h, const srlg_window_config* wc, uint64_t window_end, int partial,
               uint8_t* blob, uint64_t cap, uint64_t* bytes) {
  const auto* s = static_cast<const Sketch*>(h);
  return guarded([&] {
    const auto rep = run_detection(s->rsra, s->slea, window_end, partial != 0, to_window(wc));
    *bytes = emit_blobs({rep}, blob, cap, nullptr);
  });
}

// -------------------------------------------------------------------- engine

void* ref_engine_create(const srlg_params* p, const srlg_window_config* wc) {
  Engine* e = nullptr;
  const int rc = guarded([&] {
    const SketchParams s = to_params(p);
    s.validate();
    auto owned = std::make_unique<Engine>();
    owned->cfg = to_window(wc);
    owned->engine = std::make_unique<WindowEngine>(owned->cfg, Rsra(s.rsra_config()),
                                                   Slea(s.slea_config()), sink_to_current);
    e = owned.release();
  });
  return rc == SRLG_OK ? e : nullptr;
}

void ref_engine_destroy(void* h) { delete static_cast<Engine*>(h); }

// copy of the whole engine state (sketches, clock, pending batch); the sink of
// the copy appends to the copy's own report list
void* ref_engine_clone(const void* h) {
  const auto* src = static_cast<const Engine*>(h);
  auto out = std::make_unique<Engine>();
  out->cfg = src->cfg;
  out->reports = src->reports;
  out->engine = std::make_unique<WindowEngine>(*src->engine);
  return out.release();
}

int ref_engine_process(void* h, const srlg_record* recs, uint64_t n) {
  auto* e = static_cast<Engine*>(h);
  g_current = e;
  return guarded([&] {
    for (uint64_t i = 0; i < n; ++i)
      e->engine->process(TraceRecord{recs[i].ts_us, recs[i].aip, recs[i].bip});
  });
}

// records of slice s carry ts = t0 + s * slice_us (t0 must be configured)
int ref_engine_process_slices(void* h, const srlg_pair* pairs, const uint64_t* offsets,
                              uint64_t n_slices, uint64_t first_slice) {
  auto* e = static_cast<Engine*>(h);
  g_current = e;
  return guarded([&] {
    if (!e->cfg.t0_us) throw ConfigError("process_slices needs a configured t0");
    const uint64_t t0 = *e->cfg.t0_us;
    for (uint64_t s = 0; s < n_slices; ++s) {
      const uint64_t ts = t0 + (first_slice + s) * e->cfg.slice_us;
      for (uint64_t i = offsets[s]; i < offsets[s + 1]; ++i)
        e->engine->process(TraceRecord{ts, pairs[i].aip, pairs[i].bip});
    }
  });
}

int ref_engine_advance(void* h, uint64_t slice) {
  auto* e = static_cast<Engine*>(h);
  g_current = e;
  return guarded([&] { e->engine->advance_to_slice(slice); });
}

int ref_engine_finish(void* h) {
  auto* e = static_cast<Engine*>(h);
  g_current = e;
  return guarded([&] { e->engine->finish(); });
}

uint64_t ref_engine_take_reports(void* h, uint8_t* blob, uint64_t cap, uint64_t* n_reports) {
  auto* e = static_cast<Engine*>(h);
  const uint64_t need = emit_blobs(e->reports, blob, cap, n_reports);
  if (blob && need <= cap) e->reports.clear();
  return need;
}

uint64_t ref_engine_current_slice(const void* h) {
  return static_cast<const Engine*>(h)->engine->current_slice();
}

void ref_engine_export(const void* h, uint16_t* rsra, uint16_t* slea) {
  const auto* e = static_cast<const Engine*>(h);
  if (rsra) std::copy(e->engine->rsra().cells().begin(), e->engine->rsra().cells().end(), rsra);
  if (slea) std::copy(e->engine->slea().cells().begin(), e->engine->slea().cells().end(), slea);
}

// ---------------------------------------------------------------- distributed

int ref_run_distributed(const srlg_record* recs, uint64_t n, const srlg_params* p,
                        const srlg_window_config* wc, uint32_t nodes, uint32_t policy,
                        uint8_t* blob, uint64_t cap, uint64_t* bytes, uint64_t* n_reports,
                        uint64_t* slice_merges, uint64_t* bytes_exchanged) {
  return guarded([&] {
    const SketchParams s = to_params(p);
    s.validate();
    std::vector<TraceRecord> v(n);
    for (uint64_t i = 0; i < n; ++i) v[i] = TraceRecord{recs[i].ts_us, recs[i].aip, recs[i].bip};
    DistributedOptions opt;
    opt.nodes = nodes;
    opt.policy = static_cast<PartitionPolicy>(policy);
    DistributedStats st;
    const auto reps = run_distributed(v, to_window(wc), s.rsra_config(), s.slea_config(), opt, &st);
    *bytes = emit_blobs(reps, blob, cap, n_reports);
    *slice_merges = st.slice_merges;
    *bytes_exchanged = st.bytes_exchanged;
  });
}

// report_to_csv (src/report.cpp) over a blob sequence
uint64_t ref_blobs_to_csv(const uint8_t* blob, uint64_t bytes, char* out, uint64_t cap) {
  std::vector<DetectionReport> reps;
  uint64_t off = 0;
  while (off + sizeof(srlg_report_header) <= bytes) {
    srlg_report_header h;
    std::memcpy(&h, blob + off, sizeof(h));
    off += sizeof(h);
    DetectionReport r;
    r.window_end_slice = h.window_end_slice;
    r.candidate_count = h.candidate_count;
    r.sf_product = h.sf_product;
    r.partial = h.partial;
    r.overflow = h.overflow;
    r.slea_saturated = h.slea_saturated;
    for (uint32_t i = 0; i < h.n_rows; ++i) {
      uint64_t v;
      std::memcpy(&v, blob + off, 8);
      off += 8;
      r.hot_per_row.push_back(v);
    }
    for (uint32_t i = 0; i < h.n_entries; ++i) {
      srlg_entry x;
      std::memcpy(&x, blob + off, sizeof(x));
      off += sizeof(x);
      r.entries.push_back(ReportEntry{x.aip, x.estimate, x.saturated != 0});
    }
    reps.push_back(std::move(r));
  }
  const std::string csv = report_to_csv(reps);
  if (out && csv.size() + 1 <= cap) std::memcpy(out, csv.c_str(), csv.size() + 1);
  return csv.size() + 1;
}

// Rng (include/slidecard/rng.hpp:11-32): pair i = (next_u32(), next_u32())
void ref_rng_pairs(uint64_t seed, uint64_t n, srlg_pair* out) {
  Rng rng(seed);
  for (uint64_t i = 0; i < n; ++i) {
    out[i].aip = rng.next_u32();
    out[i].bip = rng.next_u32();
  }
}

// sketch_io (src/sketch_io.cpp:106-180): serialised "SRLG" v1 bytes
uint64_t ref_serialize(const void* h, int which, uint8_t* out, uint64_t cap) {
  const auto* s = static_cast<const Sketch*>(h);
  std::ostringstream os;
  if (which == 1) serialize_sketch(s->rsra, os);
  else serialize_sketch(s->slea, os);
  const std::string b = os.str();
  if (out && b.size() <= cap) std::memcpy(out, b.data(), b.size());
  return b.size();
}

unsigned ref_hardware_threads() { return std::max(1u, std::thread::hardware_concurrency()); }

}  // extern "C"
#pragma GCC visibility pop
