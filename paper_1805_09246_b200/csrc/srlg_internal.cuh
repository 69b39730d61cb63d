// srlg_internal.cuh — device-side parameter blocks, hashing and launchers
// shared by kernels.cu (the sm_100a kernels) and capi.cu (the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "srlg.h"

namespace srlg {

constexpr uint64_t kGolden64 = 0x9e3779b97f4a7c15ULL;  // hash.hpp:11
constexpr uint32_t kMaxRows = SRLG_MAX_ROWS;
constexpr uint32_t kDetectThreads = 512;  // threads per CTA of the detection / engine kernels

// mix64 (include/slidecard/hash.hpp:14-21)
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

// SeededHash::operator() (hash.hpp:33-35) with the offset mix64(seed)
// precomputed on the host
__host__ __device__ __forceinline__ uint64_t seeded(uint64_t offset, uint32_t key) {
  return mix64(offset + static_cast<uint64_t>(key) * kGolden64);
}

__host__ __device__ __forceinline__ uint64_t hash64(uint64_t key, uint64_t seed) {
  return mix64(mix64(seed) + key * kGolden64);
}

// ----------------------------------------------------------- stamp clocks
// A handle's state is u32 stamps. `now` is the value records write in the
// open slice; stamps <= `floor` are dead (reinitialize). Distance of a live
// stamp v is now - v (saturating at 0xFFFF). A stamp is inside window k iff
// v > lo with lo = max(floor, now - min(k, 0xFFFF)) — the reference's
// `distance < k` (src/sliding_counters.cpp:24-32). now starts at 65537 so
// that every importable distance (<= 65534) maps to a positive stamp.
constexpr uint32_t kClockOrigin = 65537;

__host__ __device__ __forceinline__ uint32_t window_lo(uint32_t now, uint32_t floor, uint32_t k) {
  const uint32_t kk = k > 0xFFFFu ? 0xFFFFu : k;
  const uint32_t lo = now - kk;
  return lo > floor ? lo : floor;
}

// ----------------------------------------------------- parameter blocks

struct RsraDev {
  uint32_t* cells;     // r x 2^q x eta stamps (reference layout, rsra.hpp:65-67)
  uint64_t h0, h1, h2; // mix64(seed) offsets: rhfg0, gate, slot
  uint32_t q, r, delta, eta;
  uint32_t col_mask, gate_mask, gate_never, eta_pow2;
};

struct SleaDev {
  uint32_t* cells;     // r' x row_len stamps (reference layout, slea.cpp:41-43)
  uint64_t row_len;
  uint64_t h3;
  uint32_t q, r, delta, eta;
  uint32_t col_mask, eta_pow2;
  const uint64_t* lh_dev;  // device copy of lh[] for dynamically indexed rows
  uint64_t lh[kMaxRows];   // mix64(seeds_lh[i]) offsets
};

// Monitored network of raw-packet ingest (AnetSpec, trace.hpp:49-62);
// n == 0: the input is already classified records
struct AnetDev {
  uint32_t n;
  uint32_t addr[SRLG_MAX_PREFIXES];  // prefix bits, pre-masked
  uint32_t mask[SRLG_MAX_PREFIXES];
};

// Group geometry for reconstruction (ReversibleHashGroup, hash.hpp:73-120)
struct GroupDev {
  uint64_t h0;
  uint32_t q, r, delta, col_mask, overlap_mask, uncovered, n_free;
  uint8_t free_bits[32];
};

// Per-window detection scratch / result written by the device pipeline.
struct WinResult {
  uint64_t hot_counts[kMaxRows];
  uint64_t row_weights[kMaxRows];
  uint64_t seed_work;
  uint64_t checked;       // tuples_checked (reconstruct.cpp)
  uint64_t stage_count[kMaxRows + 1];  // live tuples after each stage
  uint64_t n_candidates;  // addresses produced by inversion
  uint32_t overflow;      // reconstruction caps exceeded
  uint32_t cand_truncated;
  uint32_t empty;          // some hot list is empty: nothing to reconstruct
  uint32_t pad;
  uint64_t tail_offset;    // engine runs: candidates past the host prefix, in the arena
  uint64_t t_begin, t_end; // globaltimer (ns): detection start (CTA 0) and record written
  uint64_t t_phase[6];     // diagnostics: CTA 0's phase boundaries (detect.cu stamp_phase)
  uint64_t t_diag[4];      // diagnostics: last DFS warp end, last A2 warp end, DFS warps/CTA, inversion end
};

struct Candidate {
  uint32_t aip;
  uint32_t weight;  // USLE weight (slea.cpp:103-114)
};

// Device scratch of the fused detection kernel; all-zero between launches
// (the kernel's last CTA resets it).
struct ReconCounters {
  unsigned long long stage[kMaxRows + 1];  // live tuples after each stage
  unsigned long long n_cand;
  unsigned long long truncated;
};

struct DetectScratch {
  unsigned long long hot_counts[kMaxRows];
  unsigned long long row_weights[kMaxRows];
  ReconCounters cnt;
  unsigned done;
  unsigned abort;  // a stage exceeded tuple_cap: everyone stops (overflow)
  unsigned gen;    // generation of the last launch (overlap-table tags)
  unsigned left_n;  // candidates whose USLE weight is left to the publishing CTA
  unsigned long long reserved;
  unsigned long long phase_ns[16];  // diagnostics: globaltimer at phase boundaries
};

// Incremental window tracking of the persistent engine (detect.cu
// phase_a_inc). The state is cut into blocks of kIncBlock cells (8 sectors).
// smin[b] is a lower bound of the stamps of block b's cells that the live
// structures count as inside the window (0xFFFFFFFF: none), and 0 once a scan
// marked the block (a cell may have entered the window). A detection
// re-examines exactly the blocks with smin <= its window low: every other
// block's inside cells are still inside and no outside cell entered.
//  * RSRA: a scan marks the block of every gated update it makes (1/2^tau of
//    the records, so the marks cost nothing measurable); live_hot holds one
//    bit per SRE (hot at the last detection).
//  * SLEA (only when its sweep would be expensive: state beyond L2, kOpLe): a
//    scan marks a block when a cell's bit in live_bits — the inside bitmap of
//    the last detection — is clear. That read doubles the scan's L2
//    operations, which costs more than a sweep of an L2-resident SLEA.
//    live_row holds the per-row inside counts.
constexpr uint32_t kLeLogSlots = 9;     // >= the buffer sets in flight (kMaxSets)
constexpr uint32_t kLeLogCtas = 256;    // >= stream CTAs of a launch
constexpr uint32_t kLeLogCap = 1024;    // changed words logged per CTA and detection
constexpr uint32_t kIncBlockLog = 6;
constexpr uint32_t kIncBlock = 1u << kIncBlockLog;  // cells per block (8 x 32 B sectors)

struct IncDev {
  uint32_t* rs_smin;        // ceil(rsra cells / kIncBlock)
  uint32_t* le_smin;        // ceil(slea cells / kIncBlock)
  uint32_t* live_bits;      // le_bits_words words
  uint8_t* live_hot;        // one byte per RSRA block (= 8 SREs at eta 8)
  unsigned long long* live_row;  // kMaxRows
  uint64_t rs_blocks, le_blocks;
  unsigned long long* stats;     // diagnostics (trace_ops): flagged RSRA / SLEA blocks, detections
  // SLEA tracked: per (detection % kLeLogSlots, stream CTA) the live bitmap
  // words the CTA changed ({block, new word}, at most kLeLogCap; the count
  // kLeLogCap + 1 marks an overflow), so that a detection's buffer set is
  // brought up to date by replaying the last n_sets logs instead of copying
  // the whole live bitmap
  uint32_t* le_log_idx;
  unsigned long long* le_log_val;
  uint32_t* le_log_n;
};

// One buffer set of the per-detection state: phase A of a detection fills
// it, the reconstruction reads it while the next slices' scans run.
constexpr uint32_t kMaxSets = 9;
constexpr uint32_t kMaxReconGroups = kMaxSets - 1;
struct DetectScratch;
struct Candidate;
struct DetSet {
  uint32_t* hot_cols;
  uint32_t* le_bits;
  Candidate* cands;
  uint32_t* left;
  DetectScratch* scratch;
  unsigned long long* table;
};

struct DetectParams {
  RsraDev rs;
  uint32_t rs_lo, hot_min;
  SleaDev le;
  uint32_t le_lo, pad;
  const uint64_t* lh;  // device copy of the SLEA row-hash offsets
  GroupDev g;
  uint32_t* hot_cols;  // r x 2^q
  uint32_t* tuples_a;
  uint32_t* tuples_b;
  uint32_t* le_bits;           // SLEA inside bitmap, bit = flat cell index (detect.cu phase A)
  uint64_t le_bits_words;      // ceil(r' * row_len / 32) + 1 (funnel-shift read past the end)
  unsigned long long* table;  // overlap tables of rows 2..r-1, (r-2) x table_stride
  uint64_t table_stride;      // 2^table_bits entries per row (load factor <= 1/2)
  uint32_t table_bits, pad2;
  uint64_t tuple_cap, work_cap;
  Candidate* cands;
  uint64_t cand_cap;
  uint32_t* left;          // cand_cap candidate indices (weights left to the last CTA)
  DetectScratch* scratch;
  unsigned* bar;           // grid barrier {count, generation}: its own allocation, away
                           // from the counters the CTAs update while others spin
  WinResult* out;          // mapped pinned host memory
  Candidate* host_cands;   // mapped pinned host memory, host_prefix entries
  uint64_t host_prefix;
  uint32_t diag;           // record per-warp-role end times (srlg_engine_trace_ops)
  uint32_t serial;         // detection serial: overlap-table generation (never 0)
  // the CTA group running the current phase (its rank, size and barrier
  // counter); per-CTA values in the kernel's shared copy of this block
  uint32_t grank, gsize;
  unsigned* gbar;
  // engine pipelining: reconstruction CTAs (0 = every CTA runs every phase)
  // and the second buffer set of the double-buffered per-detection state
  uint32_t recon_ctas, pad3;
  AnetDev anet;            // scans: classify raw packets (anet.n > 0)
  unsigned long long* raw_records;  // scans of raw packets: records produced (or null)
  // reconstruction scratch: per thread of the launch 3 * dfs_rows words (the
  // depth-first walk state for r > 8 rows, tuples past a CTA's queue)
  uint32_t* dfs_scratch;
  uint32_t dfs_rows, pad4;
  // engine: detection d uses buffer set d % n_sets (set 0 = the fields above)
  // and reconstruction group d % recon_groups
  uint32_t n_sets, recon_groups;
  DetSet sets[kMaxSets];
  IncDev inc;             // engine: incremental window tracking (EngineOp flags)
};

// ------------------------------------------------------------- launchers
namespace dev {

enum StoreMode { kStorePlain = 0, kStoreRedMax = 1, kStoreMark = 2 };

// K1: fused RSRA + SLEA scan of n pairs (rs.cells / le.cells may be null)
cudaError_t scan(const srlg_pair* pairs, uint64_t n, const RsraDev& rs, uint32_t rs_now,
                 const SleaDev& le, uint32_t le_now, int mode, cudaStream_t st,
                 const AnetDev* anet = nullptr, unsigned long long* raw_records = nullptr);

// K2: RSRA hot bitmap + SLEA per-row inside counts (per-block partials)
struct CountsLayout {
  uint64_t rs_sres;     // r * 2^q
  uint32_t rs_blocks;   // blocks for the RSRA part
  uint32_t le_blocks_per_row;
  uint64_t le_chunk;    // cells per SLEA block (multiple of 4)
};
CountsLayout counts_layout(const RsraDev* rs, const SleaDev* le);
cudaError_t window_counts(const RsraDev* rs, uint32_t rs_lo, uint32_t hot_min,
                          const SleaDev* le, uint32_t le_lo, const CountsLayout& L,
                          uint32_t* hot_bits, uint32_t* partials, cudaStream_t st);

// ordered compaction of the hot bitmap into per-row lists (row i at
// hot_cols + i * 2^q), row sums of the SLEA partials, and seed-work setup
cudaError_t hot_compact(const uint32_t* hot_bits, uint32_t q, uint32_t r,
                        const uint32_t* partials, uint32_t le_rows, uint32_t le_blocks_per_row,
                        uint32_t* hot_cols, WinResult* res, uint64_t work_cap,
                        cudaStream_t st);

// reconstruct_candidates (src/reconstruct.cpp:32-151) as device stages
cudaError_t reconstruct(const GroupDev& g, const uint32_t* hot_cols, WinResult* res,
                        uint32_t* tuples_a, uint32_t* tuples_b, uint64_t tuple_cap,
                        uint64_t work_cap, Candidate* cands, uint64_t cand_cap,
                        int n_sms, cudaStream_t st);

// K3: USLE weight per candidate (slea.cpp:103-114); n from res (or n_host
// when res == nullptr)
cudaError_t usle_weights(const SleaDev& le, uint32_t le_lo, Candidate* cands,
                         const WinResult* res, uint64_t n_host, uint64_t cand_cap, int n_sms,
                         cudaStream_t st);

// multi-GPU merge, root side: stamps := now where the reduced u8 dirty map is
// set (RSRA cells first, then SLEA), then the map is cleared
cudaError_t apply_marks(uint8_t* dirty, uint64_t n_rs, uint32_t* rs, uint32_t rs_now,
                        uint64_t n_le, uint32_t* le, uint32_t le_now, cudaStream_t st);

// stamp <-> distance conversions and merges
cudaError_t export_distances(const uint32_t* stamps, uint64_t n, uint32_t now, uint32_t floor,
                             uint16_t* out, cudaStream_t st);
cudaError_t import_distances(const uint16_t* in, uint64_t n, uint32_t now, uint32_t* stamps,
                             cudaStream_t st);
cudaError_t merge_max(uint32_t* a, const uint32_t* b, uint64_t n, uint32_t now_a,
                      uint32_t floor_a, uint32_t now_b, uint32_t floor_b, cudaStream_t st);

// fused per-slide detection (detect.cu): cooperative, one CTA per SM
int detect_grid(int device);
cudaError_t detect(const DetectParams& P, int grid, cudaStream_t st);

// persistent engine (detect.cu): a batch of scan / detect ops in one launch
struct EngineOp {
  uint64_t begin, end;      // scan: pair index range
  uint32_t rs_now, le_now;  // scan: the slice's stamps
  uint32_t rs_lo, le_lo;    // detect: window lows
  uint32_t kind;            // 0 scan, 1 detect
  uint32_t window;          // detect: ring slot (= detection index in the batch)
  uint32_t serial;          // detect: serial (overlap-table generation, never 0)
  uint32_t chunk;           // scan: host-input chunk holding the slice's last pair
  uint32_t seq;             // scan, merge mode: the slice's merge sequence (same on every rank)
  uint32_t flags;           // kOpInit / kOpInc (detect), kOpTrack (scan), kOpLe (both)
  unsigned long long grab;  // scan: pairs claimed by the stream CTAs (the host writes 0)
};

// detect: full phase A that also (re)builds the live RSRA structures (and
// the live SLEA ones with kOpLe)
constexpr uint32_t kOpInit = 1;
// detect: RSRA phase A from the live structures (a previous detect op of the
// launch was kOpInit / kOpInc, and every scan since tracked); SLEA likewise
// with kOpLe, else the SLEA part sweeps
constexpr uint32_t kOpInc = 2;
// scan: mark the RSRA blocks of gated updates (and with kOpLe the SLEA blocks
// of cells whose live bit is clear)
constexpr uint32_t kOpTrack = 4;
// detect / scan: the SLEA is tracked incrementally too
constexpr uint32_t kOpLe = 8;
// any op: the next op of the launch is a scan (set by the host, so a scan op
// does not wait for the next op's descriptor to decide on the prefetch)
constexpr uint32_t kOpNextScan = 16;

// ---- in-engine multi-GPU merge (run_distributed's transient
// global, src/distributed.cpp:72-85). The root's device memory holds an
// inbox: per sending rank, kInboxSlots slots of cell-index lists. A rank's
// scan stamps its own state with atom.max and appends every cell whose stamp
// moved in this slice (RSRA cell i as i, SLEA cell j as rs_n + j) to its
// CTA's region of the slot, over peer memory; then it publishes `done`. The
// root's CTAs apply the lists (red.max of the slice's stamp) between their
// own scan of the slice and phase A, and release the slot (`consumed`).
constexpr uint32_t kInboxSlots = 3;
constexpr uint32_t kInboxMaxCtas = 256;

struct InboxRank {                   // one per rank, in the root's memory
  unsigned done;                     // rank -> root: slices published (seq + 1)
  unsigned pad0[31];
  unsigned consumed;                 // root -> rank: slices applied (seq + 1)
  unsigned pad1[31];
  unsigned applied[kInboxSlots];     // root: CTAs done applying the slot
  unsigned pad2[32 - kInboxSlots];
  unsigned grid;                     // the rank's CTAs (= regions per slot)
  unsigned pad3[31];
  unsigned counts[kInboxSlots][kInboxMaxCtas];  // entries per region
};

struct InboxHeader {                 // at the start of the inbox allocation
  uint64_t magic;
  uint32_t nranks, slots;
  uint64_t slot_cap;                 // u32 entries per (rank, slot)
  uint64_t rs_n, le_n;               // cell counts (index space RSRA then SLEA)
  uint64_t max_pairs;                // packets per slice and rank the slots are sized for
  unsigned long long entries;        // root: list entries applied so far (merge stats)
  uint64_t pad;
};

struct MergeDev {
  uint32_t role;          // 0 none, 1 root, 2 sending rank
  uint32_t rank, nranks;
  uint32_t pad;
  uint64_t slot_cap;      // u32 entries per (rank, slot)
  uint64_t rs_n;          // RSRA cells; SLEA cell j is entry rs_n + j
  InboxRank* hdr;         // [nranks] (root memory; entry 0 unused)
  uint32_t* lists;        // [nranks][kInboxSlots][slot_cap] (root memory)
  unsigned long long* entries;  // root: list entries applied (InboxHeader::entries)
};

struct EngineRing {        // one slot per detect op of the batch
  WinResult* out;          // mapped pinned host
  Candidate* cands;        // mapped pinned host, host_prefix per slot
  uint32_t* ready;         // mapped pinned host flags
  Candidate* arena;        // device, candidates beyond the prefix: a ring per
  uint64_t arena_cap;      // reconstruction group, arena_cap entries each
  unsigned long long* op_t;  // diagnostics (or null): per op {first CTA start, last CTA end}
  unsigned long long* cta_t;  // diagnostics (or null): per op, per CTA {start, end}
  const unsigned* chunk_flags;  // host input: chunk c copied once chunk_flags[c] != 0 (or null)
  MergeDev merge;               // in-engine multi-GPU merge (role 0: none)
  const unsigned long long* arena_released;  // mapped, per group: ring offset freed up to
  unsigned long long* arena_heads;           // device, per group: ring allocation offset
  // leading scan ops run as one grid-stride loop by every CTA (their pair
  // ranges are contiguous; 0: none) — the scan-only slices before the first
  // detection need no barriers, and per-op loops of ~2 pairs per thread left
  // the L2 update rate idle between ops
  uint32_t merged_prefix;
};
constexpr uint32_t kMergedPrefixCap = 2048;  // op boundaries kept in shared memory

cudaError_t engine_run(const DetectParams& P, const EngineOp* ops, uint32_t n_ops,
                       const srlg_pair* pairs, const EngineRing& ring, int grid, cudaStream_t st);

// exact sliding oracle (exact.cu): record a slice's pairs; one window's hosts
// with >= theta live peers as (aip << 32 | count) in out
cudaError_t exact_insert(const srlg_pair* pairs, uint64_t n, uint32_t now, unsigned long long* keys,
                         uint32_t* stamps, uint64_t mask, unsigned long long* n_pairs,
                         cudaStream_t st);
cudaError_t exact_window(const unsigned long long* keys, const uint32_t* stamps, uint64_t slots,
                         uint32_t lo, uint32_t* akeys, uint32_t* counts, uint64_t amask,
                         uint64_t theta, uint64_t* out, unsigned long long* n_out, uint64_t cap,
                         cudaStream_t st);

// random-update roofline on a trace's own address distribution (bench only):
// the cell-index stream of n pairs (r' SLEA entries per packet, then the
// gated packets' RSRA entries), and its replay as red.max updates
cudaError_t trace_indices(const srlg_pair* pairs, uint64_t n, const RsraDev& rs, const SleaDev& le,
                          uint32_t* le_idx, uint32_t* rs_idx, unsigned long long* rs_cnt,
                          int n_sms, cudaStream_t st);
cudaError_t replay_updates(const uint32_t* idx, uint64_t n, uint32_t* buf, uint32_t v, int n_sms,
                           cudaStream_t st);

// random-update roofline microbenchmark (bench only)
cudaError_t random_updates(uint32_t* buf, uint64_t n_cells, uint64_t n_updates, int mode,
                           uint64_t seed, uint32_t v, int n_sms, cudaStream_t st);

}  // namespace dev
}  // namespace srlg
