// dropin_check.cpp — exercises the C++ drop-in (include/slidecard/) the way
// a reference caller does: the same class names, calls and exception types
// as proj/core (tests/test_rsra.cpp, test_slea.cpp, test_window.cpp,
// test_distributed.cpp). Self-checks fail the exit code; the traces and the
// report CSVs are written to <outdir> so tests/test_dropin.py can replay the
// traces through the CPU oracle and compare byte for byte.
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "slidecard/config.hpp"
#include "slidecard/distributed.hpp"
#include "slidecard/errors.hpp"
#include "slidecard/rng.hpp"
#include "slidecard/sketch_io.hpp"
#include "slidecard/trace.hpp"
#include "slidecard/window.hpp"

using namespace slidecard;

static int failures = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                        \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, T)       \
  do {                                 \
    bool thrown = false;               \
    try {                              \
      (void)(expr);                    \
    } catch (const T&) {               \
      thrown = true;                   \
    } catch (...) {                    \
    }                                  \
    CHECK(thrown && #T);               \
  } while (0)

static SketchParams small_params(uint64_t seed) {
  SketchParams p;
  p.q = 12;
  p.r = 5;
  p.delta = 7;
  p.eta = 8;
  p.q_prime = 8;
  p.r_prime = 3;
  p.delta_prime = 8;
  p.eta_prime = 256;
  p.theta = 64;
  p.seed = seed;
  p.validate();
  return p;
}

static std::vector<TraceRecord> trace(uint64_t seed, size_t n, uint64_t slices, uint32_t hosts) {
  Rng rng(seed);
  std::vector<TraceRecord> recs;
  for (size_t i = 0; i < n; ++i)
    recs.push_back({1'000'000 + rng.below(slices * 1'000'000),
                    static_cast<uint32_t>(0x0A000000 + rng.below(hosts)), rng.next_u32()});
  std::set<uint32_t> peers;
  while (peers.size() < 150) peers.insert(rng.next_u32());
  for (uint32_t b : peers) recs.push_back({1'000'000 + 1'000'000 * (slices / 2) + 7, 0x0A0000AA, b});
  std::stable_sort(recs.begin(), recs.end(),
                   [](const TraceRecord& a, const TraceRecord& b) { return a.ts_us < b.ts_us; });
  return recs;
}

static void save(const std::string& path, const void* p, size_t n) {
  std::ofstream f(path, std::ios::binary);
  f.write(static_cast<const char*>(p), static_cast<std::streamsize>(n));
}

static std::vector<DetectionReport> engine_run(const WindowConfig& cfg, const SketchParams& p,
                                               const std::vector<TraceRecord>& recs) {
  std::vector<DetectionReport> out;
  WindowEngine e(cfg, Rsra(p.rsra_config()), Slea(p.slea_config()),
                 [&](const DetectionReport& r) { out.push_back(r); });
  for (const auto& r : recs) e.process(r);
  e.finish();
  return out;
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";

  // ---- configuration errors map to the reference's exception types
  {
    SketchParams bad = small_params(1);
    bad.delta = 3;
    CHECK_THROWS_AS(bad.validate(), ConfigError);
    RsraConfig rc = small_params(1).rsra_config();
    rc.r = 2;
    CHECK_THROWS_AS(Rsra{rc}, ConfigError);
    WindowConfig wc;
    wc.k = 0;
    CHECK_THROWS_AS(wc.validate(), ConfigError);
  }

  // ---- WindowEngine value semantics (window.hpp:64-98): a copy taken
  // mid-stream continues exactly like the original (reports and state)
  {
    const SketchParams p = small_params(21);
    WindowConfig cfg;
    cfg.k = 3;
    cfg.theta = 64;
    cfg.t0_us = 1'000'000;
    const auto recs = trace(23, 60000, 12, 30);
    std::vector<DetectionReport> A, B;
    std::vector<DetectionReport>* target = &A;
    WindowEngine a(cfg, Rsra(p.rsra_config()), Slea(p.slea_config()),
                   [&](const DetectionReport& r) { target->push_back(r); });
    const size_t half = recs.size() / 2;
    for (size_t i = 0; i < half; ++i) a.process(recs[i]);
    WindowEngine b = a;
    const size_t common = A.size();
    for (size_t i = half; i < recs.size(); ++i) a.process(recs[i]);
    a.finish();
    target = &B;
    for (size_t i = half; i < recs.size(); ++i) b.process(recs[i]);
    b.finish();
    CHECK(A.size() > common + 3);
    CHECK(report_to_csv(std::vector<DetectionReport>(A.begin() + common, A.end())) ==
          report_to_csv(B));
    CHECK(std::equal(a.rsra().cells().begin(), a.rsra().cells().end(), b.rsra().cells().begin()));
    CHECK(std::equal(a.slea().cells().begin(), a.slea().cells().end(), b.slea().cells().begin()));
    WindowEngine c = a;  // copy assignment target
    c = b;
    CHECK(c.current_slice() == b.current_slice() && c.records() == b.records());
  }

  // ---- Rsra / Slea value semantics and per-pair updates (test_rsra.cpp:58-86)
  {
    const SketchParams p = small_params(3);
    Rsra a(p.rsra_config());
    Slea s(p.slea_config());
    Rng rng(5);
    for (int i = 0; i < 20000; ++i) {
      const uint32_t aip = 0x0A000000 + static_cast<uint32_t>(rng.below(40));
      const uint32_t bip = rng.next_u32();
      a.update(aip, bip);
      s.update(aip, bip);
    }
    Rsra before = a;  // deep copy (src/rsra.cpp:83-87)
    CHECK(std::equal(before.cells().begin(), before.cells().end(), a.cells().begin()));
    a.slide();
    s.slide();
    CHECK(a.slides() == 1 && s.slides() == 1);
    CHECK(!std::equal(before.cells().begin(), before.cells().end(), a.cells().begin()));
    CHECK(a.compatibility_mismatch(before) == "slice position");
    CHECK_THROWS_AS(a.merge_min(before), IncompatibleSketchError);
    before.slide();
    a.merge_min(before);  // same content: idempotent
    CHECK(std::equal(before.cells().begin(), before.cells().end(), a.cells().begin()));
    save(dir + "/state_rsra.bin", a.cells().data(), a.cells().size() * 2);
    save(dir + "/state_slea.bin", s.cells().data(), s.cells().size() * 2);
    // cells_mut write-back (test_slea.cpp:95-116 toy row)
    SleaConfig tiny;
    tiny.q = 1;
    tiny.r = 1;
    tiny.delta = 2;
    tiny.eta = 6;
    tiny.seed_h3 = 1;
    tiny.seeds_lh = {2};
    Slea t(tiny);
    CHECK(t.row_length() == 8);
    auto cells = t.cells_mut();
    const uint16_t values[8] = {0, 1, 2, 3, kNeverSet, kNeverSet, kNeverSet, kNeverSet};
    std::copy(values, values + 8, cells.begin());
    CHECK(t.setting_factor(0, 3) == 3.0 / 8.0);
    std::fill(cells.begin(), cells.end(), uint16_t{0});
    CHECK(t.setting_factor(0, 1) == 1.0);
    CHECK_THROWS_AS(t.estimate(0x0A000001, 1), SaturationError);
    // hot extraction of a planted host (test_rsra.cpp:104-127)
    Rsra h(small_params(9).rsra_config());
    std::set<uint32_t> peers;
    while (peers.size() < 128) peers.insert(rng.next_u32());
    for (uint32_t b : peers) h.update(0x0A111213, b);
    const auto hot = h.extract_hot(1);
    const auto cols = h.hash_group().forward(0x0A111213);
    for (uint32_t i = 0; i < 5; ++i) {
      CHECK(std::is_sorted(hot[i].begin(), hot[i].end()));
      CHECK(std::binary_search(hot[i].begin(), hot[i].end(), cols[i]));
    }
    const auto inv = h.hash_group().invert(cols);
    CHECK(std::find(inv.begin(), inv.end(), 0x0A111213u) != inv.end());
    const auto rec = reconstruct_candidates(hot, h.hash_group());
    CHECK(std::find(rec.addresses.begin(), rec.addresses.end(), 0x0A111213u) !=
          rec.addresses.end());
  }

  // ---- sketch streams (test_sketch_io.cpp:52-131): round trips through a
  // stream and a file, identical bytes, FormatError on truncation
  {
    const SketchParams p = small_params(5);
    Rsra a(p.rsra_config());
    Slea s(p.slea_config());
    Rng rng(11);
    for (int i = 0; i < 5000; ++i) {
      const uint32_t aip = 0x0A000000 + static_cast<uint32_t>(rng.below(40));
      const uint32_t bip = rng.next_u32();
      a.update(aip, bip);
      s.update(aip, bip);
    }
    a.slide();
    s.slide();
    std::ostringstream out;
    serialize_sketch(a, out);
    CHECK(out.str().size() == serialized_size(a));
    std::istringstream in(out.str());
    const AnySketch back = deserialize_sketch(in);
    CHECK(std::holds_alternative<Rsra>(back));
    const Rsra& b = std::get<Rsra>(back);
    CHECK(b.slides() == a.slides());
    CHECK(std::equal(b.cells().begin(), b.cells().end(), a.cells().begin()));
    const std::string path = dir + "/sketch_slea.srlg";
    save_sketch_file(AnySketch(s), path);
    const AnySketch sb = load_sketch_file(path);
    CHECK(std::holds_alternative<Slea>(sb));
    std::ostringstream o1, o2;
    serialize_sketch(s, o1);
    serialize_sketch(std::get<Slea>(sb), o2);
    CHECK(o1.str() == o2.str());
    const std::string cut = out.str().substr(0, out.str().size() - 3);
    std::istringstream tin(cut);
    CHECK_THROWS_AS((void)deserialize_sketch(tin), FormatError);
    std::istringstream bad(std::string("SRLX") + out.str().substr(4));
    CHECK_THROWS_AS((void)deserialize_sketch(bad), FormatError);
  }

  // ---- raw-packet ingest: classify fused on the device == host classify
  // (trace.cpp:111-116) followed by the record path
  {
    const SketchParams p = small_params(21);
    WindowConfig cfg;
    cfg.t0_us = 1'000'000;
    cfg.k = 3;
    cfg.theta = 64;
    AnetSpec anet;
    anet.prefixes = {CidrPrefix{0x0A000000u, 8}, CidrPrefix{0xC0A80100u, 24}};
    Rng rng(77);
    std::vector<TraceRecord> raw, recs;
    for (int i = 0; i < 40000; ++i) {
      const uint64_t ts = 1'000'000 + static_cast<uint64_t>(i) * 200;  // 8 slices
      const uint32_t a = rng.below(2) ? 0x0A000000u + static_cast<uint32_t>(rng.below(64))
                                      : rng.next_u32();
      const uint32_t b = rng.below(3) == 0 ? 0xC0A80100u + static_cast<uint32_t>(rng.below(200))
                                           : rng.next_u32();
      raw.push_back({ts, a, b});
      std::array<TraceRecord, 2> out;
      const int m = classify(RawPacket{ts, a, b}, anet, out);
      for (int j = 0; j < m; ++j) recs.push_back(out[j]);
    }
    const auto expect = engine_run(cfg, p, recs);
    std::vector<DetectionReport> got;
    {
      WindowEngine e(cfg, Rsra(p.rsra_config()), Slea(p.slea_config()),
                     [&](const DetectionReport& r) { got.push_back(r); });
      const srlg_anet a = anet.to_c();
      e.set_anet(&a);
      e.process_batch(raw);
      e.finish();
    }
    CHECK(!expect.empty());
    CHECK(report_to_csv(got) == report_to_csv(expect));
  }

  // ---- WindowEngine over sliding and discrete windows, run_distributed
  struct Case {
    const char* name;
    uint32_t k;
    bool reinit;
    uint64_t seed;
  };
  for (const Case c : {Case{"k3", 3, false, 7}, Case{"k10", 10, false, 11},
                       Case{"k1reinit", 1, true, 13}}) {
    const auto recs = trace(100 + c.seed, 6000, 12, 32);
    save(dir + "/records_" + c.name + ".bin", recs.data(), recs.size() * sizeof(TraceRecord));
    WindowConfig cfg;
    cfg.t0_us = 1'000'000;
    cfg.k = c.k;
    cfg.theta = 64;
    cfg.reinit_per_window = c.reinit;
    const auto p = small_params(c.seed);
    const auto reps = engine_run(cfg, p, recs);
    CHECK(!reps.empty());
    std::ofstream(dir + "/engine_" + c.name + ".csv") << report_to_csv(reps);
    // the batched and per-record paths agree
    std::vector<DetectionReport> batched;
    {
      WindowEngine e(cfg, Rsra(p.rsra_config()), Slea(p.slea_config()),
                     [&](const DetectionReport& r) { batched.push_back(r); });
      e.process_batch(recs);
      e.finish();
    }
    CHECK(report_to_csv(batched) == report_to_csv(reps));
    for (auto pol : {PartitionPolicy::hash_pair, PartitionPolicy::round_robin,
                     PartitionPolicy::by_source_prefix}) {
      DistributedStats st;
      DistributedOptions opt;
      opt.nodes = 4;
      opt.policy = pol;
      const auto d = run_distributed(recs, cfg, p.rsra_config(), p.slea_config(), opt, &st);
      CHECK(report_to_csv(d) == report_to_csv(reps));
      CHECK(st.slice_merges > 0 && st.bytes_exchanged > 0);
    }
  }
  CHECK(parse_partition_policy("round-robin") == PartitionPolicy::round_robin);
  CHECK_THROWS_AS(parse_partition_policy("nope"), ConfigError);

  // ---- ordering violations surface as errors (test_window.cpp:256-262)
  {
    const auto p = small_params(1);
    WindowConfig cfg;
    cfg.t0_us = 1'000'000;
    cfg.k = 2;
    cfg.theta = 64;
    WindowEngine e(cfg, Rsra(p.rsra_config()), Slea(p.slea_config()), nullptr);
    e.process({5'000'000, 0x0A000001, 1});
    CHECK_THROWS_AS(e.process({3'000'000, 0x0A000001, 2}), OrderingError);
  }

  std::printf("dropin_check: %d failure(s)\n", failures);
  return failures ? 1 : 0;
}
