/*
 * srlg.h — C ABI of the B200-native sliding super-point path
 * (arXiv 1805.09246, "distance recorder" sliding estimators).
 *
 * This is the drop-in boundary. Every entry point replaces one method of the
 * reference's C++ estimator API (slidecard, /root/reference/proj/core); the
 * reference interface each one replaces is cited beside it as file:line,
 * relative to proj/core/. The C++ classes under include/slidecard/ wrap
 * these calls with the reference's own class names, value semantics and
 * exception types.
 *
 * Conventions
 *  - Plain C types only; no torch, no CUDA types. `stream` arguments are a
 *    cudaStream_t passed as void* (NULL = the handle's own stream).
 *  - Every function returns an srlg_status; srlg_last_error() gives the
 *    message of the calling thread's most recent failure.
 *  - Device state is u32 slice *stamps* (stamp = internal clock value at the
 *    last record; 0 = never set). The reference keeps u16 *distances*
 *    (slices since last record, 0xFFFF = never; sliding_counters.hpp:10).
 *    The two are a bijection; *_export_cells /
 *    *_import_cells convert to and from the reference's exact u16 layout.
 *  - Pairs are interleaved {aip, bip} u32 records, 8 bytes each.
 */
#ifndef SRLG_H_
#define SRLG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRLG_ABI_VERSION 1

/* ---------------------------------------------------------------- status --
 * Mirrors the reference exception taxonomy (include/slidecard/errors.hpp:8-53)
 * and its CLI exit codes (proj/tools/slidecard.cpp:31-35: 2 config, 3 parse,
 * 4 resource, 5 incompatible). */
typedef enum srlg_status {
  SRLG_OK = 0,
  SRLG_ERR_CONFIG = 2,           /* ConfigError */
  SRLG_ERR_PARSE = 3,            /* ParseError */
  SRLG_ERR_RESOURCE = 4,         /* ResourceError */
  SRLG_ERR_INCOMPATIBLE = 5,     /* IncompatibleSketchError */
  SRLG_ERR_SATURATION = 6,       /* SaturationError */
  SRLG_ERR_OUT_OF_RANGE = 7,     /* std::out_of_range */
  SRLG_ERR_INVALID_ARGUMENT = 8, /* std::invalid_argument */
  SRLG_ERR_ORDERING = 9,         /* OrderingError (a ParseError) */
  SRLG_ERR_FORMAT = 10,          /* FormatError (a ParseError) */
  SRLG_ERR_CUDA = 11             /* device/runtime failure; no reference analogue */
} srlg_status;

const char* srlg_last_error(void);
int srlg_abi_version(void);

/* ----------------------------------------------------------------- types -- */

typedef struct srlg_pair {
  uint32_t aip; /* monitored endpoint (TraceRecord::aip, trace.hpp:23-29) */
  uint32_t bip; /* opposite endpoint */
} srlg_pair;

/* AnetSpec (include/slidecard/trace.hpp:49-62): the monitored network as up
 * to SRLG_MAX_PREFIXES CIDR prefixes (addr, bits); a raw packet {src, dst}
 * (RawPacket, trace.hpp:14-20, stored as srlg_pair {aip = src, bip = dst})
 * yields one record per endpoint inside it (classify, trace.cpp:111-116). */
#define SRLG_MAX_PREFIXES 16
typedef struct srlg_anet {
  uint32_t n;
  uint32_t reserved;
  uint32_t addr[SRLG_MAX_PREFIXES];
  uint32_t bits[SRLG_MAX_PREFIXES];
} srlg_anet;

typedef struct srlg_record { /* TraceRecord (include/slidecard/trace.hpp:23-29) */
  uint64_t ts_us;
  uint32_t aip;
  uint32_t bip;
} srlg_record;

/* RsraConfig (include/slidecard/rsra.hpp:13-24) */
typedef struct srlg_rsra_config {
  uint32_t q, r, delta, eta, tau;
  uint32_t reserved;
  uint64_t seed_h1, seed_h2, seed_rhfg0;
} srlg_rsra_config;

#define SRLG_MAX_ROWS 64

/* SleaConfig (include/slidecard/slea.hpp:14-23); seeds_lh holds r entries */
typedef struct srlg_slea_config {
  uint32_t q, r, delta, eta;
  uint64_t seed_h3;
  uint64_t seeds_lh[SRLG_MAX_ROWS];
} srlg_slea_config;

/* SketchParams (include/slidecard/config.hpp:14-37) */
typedef struct srlg_params {
  uint32_t q, r, delta, eta;
  uint32_t q_prime, r_prime, delta_prime, eta_prime;
  uint64_t theta;
  uint64_t seed;
} srlg_params;

/* WindowConfig (include/slidecard/window.hpp:15-26) */
typedef struct srlg_window_config {
  uint64_t t0_us;
  uint32_t has_t0; /* 0: t0 = first record's timestamp */
  uint32_t k;
  uint64_t slice_us;
  uint64_t theta;
  uint64_t regression_tolerance_us;
  uint64_t tuple_cap;
  uint32_t reinit_per_window;
  uint32_t keep_below_threshold;
  uint32_t workers; /* accepted for API parity; the device grid replaces it */
  uint32_t reserved;
} srlg_window_config;

/* ReportEntry (include/slidecard/report.hpp:10-14) */
typedef struct srlg_entry {
  uint32_t aip;
  uint32_t saturated;
  double estimate;
} srlg_entry;

/* DetectionReport (include/slidecard/report.hpp:17-27), serialised as a
 * "report blob": this fixed header, then n_rows u64 hot_per_row values, then
 * n_entries srlg_entry records (estimate desc, aip asc). Reports are
 * concatenated back to back. The oracle and the reference shim emit the same
 * blob, so report parity is a byte comparison. */
typedef struct srlg_report_header {
  uint64_t window_end_slice;
  uint64_t candidate_count;
  double sf_product;
  uint32_t n_rows;
  uint32_t n_entries;
  uint8_t partial;
  uint8_t overflow;
  uint8_t slea_saturated;
  uint8_t reserved[5];
} srlg_report_header;

/* Slea::Estimate (include/slidecard/slea.hpp:61-67) */
typedef struct srlg_estimate {
  double value;
  double corrected_weight;
  uint64_t usle_weight;
  double sf_product;
  uint32_t saturated;
  uint32_t reserved;
} srlg_estimate;

typedef struct srlg_rsra srlg_rsra;     /* device-backed Rsra */
typedef struct srlg_slea srlg_slea;     /* device-backed Slea */
typedef struct srlg_engine srlg_engine; /* device-backed WindowEngine */

/* ------------------------------------------------------- config helpers -- */

/* SketchParams::validate (src/config.cpp:20-42) */
int srlg_params_validate(const srlg_params* p);
/* SketchParams::rsra_config / slea_config (src/config.cpp:48-72) incl.
 * HashSeeds::derive (src/hash.cpp:18-27) and sampling_threshold
 * (src/hash.cpp:10-16) */
int srlg_params_rsra_config(const srlg_params* p, srlg_rsra_config* out);
int srlg_params_slea_config(const srlg_params* p, srlg_slea_config* out);
/* Slea::row_length_for (include/slidecard/slea.hpp:33-35) */
uint64_t srlg_slea_row_length_for(const srlg_slea_config* c);
/* WindowConfig::validate (src/window.cpp:11-17) */
int srlg_window_config_validate(const srlg_window_config* c);
void srlg_window_config_default(srlg_window_config* c);

/* ------------------------------------------------------------------ Rsra -- */

/* Rsra::Rsra(const RsraConfig&) (src/rsra.cpp:9-23); device = CUDA ordinal */
int srlg_rsra_create(const srlg_rsra_config* cfg, int device, srlg_rsra** out);
/* copy construction `Rsra out = a;` (src/rsra.cpp:83-87): device-to-device */
int srlg_rsra_clone(const srlg_rsra* src, srlg_rsra** out);
void srlg_rsra_destroy(srlg_rsra* h);
int srlg_rsra_config_get(const srlg_rsra* h, srlg_rsra_config* out);
uint64_t srlg_rsra_num_cells(const srlg_rsra* h);
/* Rsra::slides / set_slides (include/slidecard/rsra.hpp:35-36) */
uint64_t srlg_rsra_slides(const srlg_rsra* h);
int srlg_rsra_set_slides(srlg_rsra* h, uint64_t s);
/* Rsra::slide (src/rsra.cpp:35-38): O(1) — the stamp clock advances */
int srlg_rsra_slide(srlg_rsra* h);
/* Rsra::reinitialize (src/rsra.cpp:40-43): O(1) — raises the dead floor */
int srlg_rsra_reinitialize(srlg_rsra* h);
/* Rsra::extract_hot (src/rsra.cpp:45-57): ascending columns per row,
 * concatenated into cols (capacity cap); row_counts[r] receives list sizes. */
int srlg_rsra_extract_hot(const srlg_rsra* h, uint32_t k, uint32_t* cols, uint64_t cap,
                          uint64_t* row_counts);
/* Rsra::cells() (include/slidecard/rsra.hpp:58): u16 distances, reference layout */
int srlg_rsra_export_cells(const srlg_rsra* h, uint16_t* out, uint64_t n);
/* writes through Rsra::cells_mut() (include/slidecard/rsra.hpp:59) */
int srlg_rsra_import_cells(srlg_rsra* h, const uint16_t* in, uint64_t n);
/* raw u32 stamps plus the clock they are relative to (diagnostics, merge) */
int srlg_rsra_export_stamps(const srlg_rsra* h, uint32_t* out, uint64_t n, uint32_t* now,
                            uint32_t* floor);
/* Rsra::compatibility_mismatch (src/rsra.cpp:64-75); buf gets "" if mergeable */
int srlg_rsra_compatibility_mismatch(const srlg_rsra* a, const srlg_rsra* b, char* buf,
                                     size_t cap);
/* Rsra::merge_min (src/rsra.cpp:77-81): per-cell distance min == stamp max.
 * `other` may live on another device (peer access over NVLink). */
int srlg_rsra_merge_min(srlg_rsra* self, const srlg_rsra* other);
/* ReversibleHashGroup::forward (src/hash.cpp:63-69), host-side convenience */
int srlg_rsra_forward(const srlg_rsra* h, uint32_t aip, uint32_t* cols);
void* srlg_rsra_device_ptr(const srlg_rsra* h);

/* ------------------------------------------------------------------ Slea -- */

/* Slea::Slea(const SleaConfig&) (src/slea.cpp:11-27) */
int srlg_slea_create(const srlg_slea_config* cfg, int device, srlg_slea** out);
int srlg_slea_clone(const srlg_slea* src, srlg_slea** out);
void srlg_slea_destroy(srlg_slea* h);
int srlg_slea_config_get(const srlg_slea* h, srlg_slea_config* out);
uint64_t srlg_slea_num_cells(const srlg_slea* h);
uint64_t srlg_slea_row_length(const srlg_slea* h);
uint64_t srlg_slea_slides(const srlg_slea* h);
int srlg_slea_set_slides(srlg_slea* h, uint64_t s);
/* Slea::slide / reinitialize (src/slea.cpp:47-55) */
int srlg_slea_slide(srlg_slea* h);
int srlg_slea_reinitialize(srlg_slea* h);
/* per-row inside-window counts: counter_ops::weight over each row, the
 * integer numerator of Slea::setting_factor (src/slea.cpp:57-61) */
int srlg_slea_row_weights(const srlg_slea* h, uint32_t k, uint64_t* out_r);
/* Slea::make_estimate_context (src/slea.cpp:85-95): factors[r] + product */
int srlg_slea_estimate_context(const srlg_slea* h, uint32_t k, double* factors,
                               double* sf_product);
/* fused union + weight of Slea::estimate (src/slea.cpp:103-114) for n hosts */
int srlg_slea_usle_weights(const srlg_slea* h, uint32_t k, const uint32_t* aips, uint64_t n,
                           uint64_t* out);
/* Slea::estimate(aip, ctx) (src/slea.cpp:97-125); SRLG_ERR_SATURATION when
 * the setting-factor product is within kSaturationEps of 1 */
int srlg_slea_estimate(const srlg_slea* h, uint32_t aip, uint32_t k, double sf_product,
                       srlg_estimate* out);
/* Slea::lh_column (src/slea.cpp:34-36) */
int srlg_slea_lh_column(const srlg_slea* h, uint32_t row, uint32_t aip, uint32_t* out);
int srlg_slea_export_cells(const srlg_slea* h, uint16_t* out, uint64_t n);
int srlg_slea_import_cells(srlg_slea* h, const uint16_t* in, uint64_t n);
int srlg_slea_export_stamps(const srlg_slea* h, uint32_t* out, uint64_t n, uint32_t* now,
                            uint32_t* floor);
int srlg_slea_compatibility_mismatch(const srlg_slea* a, const srlg_slea* b, char* buf,
                                     size_t cap);
/* Slea::merge_min (src/slea.cpp:142-146) */
int srlg_slea_merge_min(srlg_slea* self, const srlg_slea* other);
void* srlg_slea_device_ptr(const srlg_slea* h);

/* classify (trace.cpp:111-116) fused into the scan: every raw packet
 * {src, dst} updates the sketches once per endpoint inside `anet` (src first:
 * (src, dst), then (dst, src)) — the reference's classify + Rsra/Slea::update.
 * Same device / stream semantics as srlg_update_pairs. *records (optional,
 * NULL allowed) receives the number of records the packets produced. */
int srlg_update_raw(srlg_rsra* rsra, srlg_slea* slea, const srlg_pair* packets, uint64_t n,
                    int packets_on_device, const srlg_anet* anet, uint64_t* records);

/* ------------------------------------------------------- exact oracle
 * ExactSlidingOracle (exact_oracle.hpp:25-62, exact_oracle.cpp:22-101) on
 * the device, for scoring at 10^8–10^9 packets: per-pair last-seen stamps in
 * a hash table of 2 * max_pairs slots; each completed slice from k-1 on and
 * the stream end emit a window with the hosts whose exact distinct-peer count
 * is >= theta (cardinality desc, aip asc). Input is pre-sliced like
 * srlg_engine_process_slices. SRLG_ERR_CONFIG for k outside [1, 65534];
 * SRLG_ERR_RESOURCE when more than max_pairs distinct pairs are seen.
 * take_windows blob: per window {u64 end_slice, u32 partial, u32 n} then n x
 * {u32 aip, u32 0, u64 cardinality}; NULL blob returns the size only. */
typedef struct srlg_exact srlg_exact;
int srlg_exact_create(uint64_t theta, uint32_t k, uint64_t max_pairs, int device, srlg_exact** out);
void srlg_exact_destroy(srlg_exact* e);
int srlg_exact_process_slices(srlg_exact* e, const srlg_pair* pairs, const uint64_t* offsets,
                              uint64_t n_slices, uint64_t first_slice, int pairs_on_device);
int srlg_exact_finish(srlg_exact* e);
uint64_t srlg_exact_distinct_pairs(const srlg_exact* e);
int srlg_exact_take_windows(srlg_exact* e, uint8_t* blob, uint64_t cap, uint64_t* bytes,
                            uint64_t* n_windows);

/* ------------------------------------------------------- sketch streams
 * The reference's "SRLG" v1 binary sketch stream (sketch_io.hpp:13-24):
 * magic | version u16 | type u8 | parameters u32 | seeds u64 | slides u64 |
 * u16 distances, little-endian. Byte-identical to the reference's files.
 * serialized_size: sketch_io.cpp:136-142. serialize_sketch: sketch_io.cpp:
 * 106-134 (cap >= serialized_size). deserialize_sketch: sketch_io.cpp:144-175
 * — creates a new handle on `device`: *type 1 (rsra) or 2 (slea), the other
 * out-pointer stays NULL, *consumed = bytes read; SRLG_ERR_FORMAT on bad
 * magic / version / type tag or truncation (the reference's FormatError),
 * SRLG_ERR_CONFIG when the parameter block is rejected (Rsra/Slea ctors). */
uint64_t srlg_rsra_serialized_size(const srlg_rsra* h);
uint64_t srlg_slea_serialized_size(const srlg_slea* h);
int srlg_rsra_serialize(const srlg_rsra* h, uint8_t* out, uint64_t cap, uint64_t* written);
int srlg_slea_serialize(const srlg_slea* h, uint8_t* out, uint64_t cap, uint64_t* written);
int srlg_deserialize_sketch(const uint8_t* in, uint64_t size, int device, int* type,
                            srlg_rsra** rsra, srlg_slea** slea, uint64_t* consumed);

/* -------------------------------------------------------- the packet scan --
 * Rsra::update + Slea::update (src/rsra.cpp:25-33, src/slea.cpp:38-45) over a
 * batch of pairs, as WindowEngine::flush_pending applies one slice
 * (src/window.cpp:89-98). Either handle may be NULL. pairs_on_device != 0:
 * `pairs` is a device pointer on the handles' device; otherwise host memory
 * (copied through a pinned staging ring). Asynchronous on `stream` for
 * device input; host input returns once the pairs have been consumed. */
int srlg_update_pairs(srlg_rsra* rsra, srlg_slea* slea, const srlg_pair* pairs, uint64_t n,
                      int pairs_on_device, void* stream);

/* --------------------------------------------------------- reconstruction --
 * reconstruct_candidates (src/reconstruct.cpp:32-151) on the device. hot_cols
 * holds r ascending lists back to back with row_counts[r] sizes. Addresses
 * are written sorted and unique; *overflow mirrors ReconstructResult. */
int srlg_reconstruct(const srlg_rsra* group_of, const uint32_t* hot_cols,
                     const uint64_t* row_counts, uint64_t tuple_cap, uint64_t work_cap,
                     uint32_t* addresses, uint64_t cap, uint64_t* n_addresses,
                     int* overflow, uint64_t* tuples_checked, uint64_t* tuples_kept);

/* the same for a bare ReversibleHashGroup(q, r, delta, seed)
 * (src/hash.cpp:39-57), as reconstruct_candidates takes it; the group need
 * not cover the address (acceptance.cpp:301-328 uses q=10, delta=3) */
int srlg_reconstruct_group(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, int device,
                           const uint32_t* hot_cols, const uint64_t* row_counts,
                           uint64_t tuple_cap, uint64_t work_cap, uint32_t* addresses,
                           uint64_t cap, uint64_t* n_addresses, int* overflow,
                           uint64_t* tuples_checked, uint64_t* tuples_kept);

/* -------------------------------------------------------------- detection --
 * run_detection (src/window.cpp:36-78): hot extraction, reconstruction,
 * setting factors and per-candidate estimates on the device; the double
 * arithmetic of corrected_weight / le_estimate (src/linear_counting.cpp:10-24)
 * on the host with the reference's expressions, so estimates are
 * bit-identical. Writes one report blob (see srlg_report_header). */
int srlg_detect(const srlg_rsra* rsra, const srlg_slea* slea, const srlg_window_config* cfg,
                uint64_t window_end_slice, int partial, uint8_t* blob, uint64_t cap,
                uint64_t* blob_bytes);

/* ---------------------------------------------------------------- engine --
 * WindowEngine (include/slidecard/window.hpp:64-98, src/window.cpp:80-137).
 * The engine takes ownership of both sketches. Reports accumulate inside the
 * engine and are drained with srlg_engine_take_reports. */
int srlg_engine_create(const srlg_window_config* cfg, srlg_rsra* rsra, srlg_slea* slea,
                       srlg_engine** out);
/* WindowEngine copy (window.hpp:64-98 is a value type): deep device copies of
 * both sketches plus the clock, open slice and untaken reports */
int srlg_engine_clone(srlg_engine* src, srlg_engine** out);
void srlg_engine_destroy(srlg_engine* e);
/* WindowEngine::process (src/window.cpp:122-131) for a time-ordered batch */
int srlg_engine_process(srlg_engine* e, const srlg_record* recs, uint64_t n);
/* pre-sliced fast path: pairs of slices first_slice .. first_slice+n_slices-1
 * with slice_offsets[n_slices+1] delimiting each slice inside `pairs`
 * (host or device memory). Equivalent to process() on records stamped with
 * those slices; completes every slice but the last, which stays open. */
int srlg_engine_process_slices(srlg_engine* e, const srlg_pair* pairs,
                               const uint64_t* slice_offsets, uint64_t n_slices,
                               uint64_t first_slice, int pairs_on_device);
/* WindowEngine::advance_to_slice (src/window.cpp:113-120) */
int srlg_engine_advance_to_slice(srlg_engine* e, uint64_t slice);
/* WindowEngine::finish (src/window.cpp:133-137) */
int srlg_engine_finish(srlg_engine* e);
/* blocks until queued device work is done and host finalisation caught up */
int srlg_engine_sync(srlg_engine* e);
/* drains finished reports as concatenated blobs. If cap is too small nothing
 * is drained and *blob_bytes receives the size needed. */
int srlg_engine_take_reports(srlg_engine* e, uint8_t* blob, uint64_t cap, uint64_t* blob_bytes,
                             uint64_t* n_reports);
uint64_t srlg_engine_current_slice(const srlg_engine* e);
uint64_t srlg_engine_records(const srlg_engine* e);
uint64_t srlg_engine_clamped(const srlg_engine* e);
srlg_rsra* srlg_engine_rsra(srlg_engine* e);
srlg_slea* srlg_engine_slea(srlg_engine* e);
/* restart from an empty state (fresh sketches, slice 0); used between
 * benchmark passes */
int srlg_engine_reset(srlg_engine* e);
/* device kernels launched since the last call (evidence for gpu_launches) */
uint64_t srlg_engine_kernel_launches(srlg_engine* e);

/* ------------------------------------------------------------- multi-GPU --
 * run_distributed (src/distributed.cpp:35-117) across GPUs: one edge-router
 * stream per rank, per-slide merge by an NCCL max-reduce of u8 touched-cell
 * maps onto the root (NCCL is loaded at run time). */
int srlg_nccl_unique_id(uint8_t* out128);
int srlg_nccl_comm_create(int nranks, const uint8_t* id128, int rank, int device, void** comm);
int srlg_nccl_comm_destroy(void* comm);
/* before any record; the root alone emits reports */
int srlg_engine_set_merge(srlg_engine* e, void* nccl_comm, int rank, int nranks, int root);
/* DistributedStats (include/slidecard/distributed.hpp:21-24) */
int srlg_engine_merge_stats(srlg_engine* e, uint64_t* slice_merges, uint64_t* bytes);

/* In-engine merge over peer memory (run_distributed's per-slice merged_detect,
 * src/distributed.cpp:72-85, without a host round trip): every rank's
 * persistent engine publishes the cells its slice moved into an inbox in the
 * root's device memory; the root's engine applies them between its own scan
 * of the slice and the detection. Set up on fresh engines, then feed every
 * rank the same slice structure through srlg_engine_process_slices (empty
 * slices included). The root alone emits reports. */
/* root = rank 0: allocates the inbox for nranks ranks and slices of up to
 * max_pairs_per_slice packets per rank; ipc_handle_out (64 B) may be null */
int srlg_engine_merge_create(srlg_engine* root, int nranks, uint64_t max_pairs_per_slice,
                             uint8_t* ipc_handle_out);
/* rank >= 1 in another process: maps the root's inbox (cudaIpcOpenMemHandle) */
int srlg_engine_merge_join(srlg_engine* e, int rank, const uint8_t* ipc_handle);
/* rank >= 1 in the root's process (another GPU, or another execution lane) */
int srlg_engine_merge_attach(srlg_engine* e, int rank, srlg_engine* root);

/* ----------------------------------------------------------- diagnostics --
 * No reference analogue: evidence for the benchmark. */
/* cudaStream_t of the device's compute stream (all state access runs on it) */
void* srlg_device_stream(int device);
/* per-launch CUDA-event timing of the packet scan (K1) and of the detection
 * pipeline on the compute stream; read-and-reset */
int srlg_profile_enable(int device, int on);
int srlg_profile_read(int device, double* scan_ms, uint64_t* scan_launches,
                      uint64_t* scan_pairs, double* detect_ms, uint64_t* detect_windows);
/* globaltimer (ns) at the phase boundaries of the device's last fused
 * detection: start, counts, barrier, reconstruction, barrier, usle, end */
int srlg_detect_phase_ns(int device, uint64_t* out16);
/* persistent engine batches: CUDA-event ms, launches and packets since the
 * last call (read-and-reset) */
int srlg_profile_read_engine(int device, double* ms, uint64_t* launches, uint64_t* pairs);
/* mean device time (µs) of the per-slide detections finalised from
 * persistent batches since the last call */
int srlg_engine_detect_latency(srlg_engine* e, double* mean_us, uint64_t* windows);
/* 1 (default): srlg_engine_process_slices runs whole runs of slices as one
 * persistent cooperative kernel; 0: one scan + one detect launch per slice */
int srlg_engine_set_persistent(srlg_engine* e, int on);
/* capacity (candidates) of the ring holding each window's candidates beyond
 * the first 1024 during persistent batches; 0 = default (the largest tail a
 * window can have); a smaller ring makes the kernel wait for the host to
 * drain earlier windows (tests) */
int srlg_engine_set_arena(srlg_engine* e, uint64_t entries);
/* Incremental window tracking of persistent batches: a launch's first
 * detection sweeps the whole state (phase A of run_detection's extract_hot /
 * setting_factor, window.cpp:36-78), later ones re-examine only the state
 * blocks the window moved past or the scans marked. mode 1 (default): the
 * RSRA always, the SLEA when its stamps exceed 64 MiB (beyond that its sweep
 * streams from HBM); 2: both sketches always; 3: the RSRA only; 0: every
 * detection sweeps.
 * Reports and state are identical in every mode. */
int srlg_engine_set_incremental(srlg_engine* e, int mode);
/* Reconstruction pipeline of persistent batches (tuning): `ctas` CTAs
 * (rounded down to a multiple of `groups`, at most half the grid) split into
 * `groups` (1..8) groups; group g reconstructs detections d = g mod groups
 * while the other CTAs scan the next slices, with groups + 1 per-detection
 * buffer sets in flight. 0 keeps a value; defaults 24 CTAs in 3 groups.
 * With the SLEA tracked incrementally (state beyond 64 MiB) a launch uses
 * one group: its slice periods are long enough for one. */
int srlg_engine_set_recon(srlg_engine* e, int ctas, int groups);
/* Diagnostics: state blocks the incremental detections re-examined since the
 * last call, {RSRA, SLEA, 0, 0}, counted while srlg_engine_trace_ops is on. */
int srlg_engine_inc_stats(srlg_engine* e, uint64_t out[4]);
/* Raw-packet ingest: with a non-empty `anet`, later srlg_engine_process_slices
 * calls take raw packets {src, dst} and classify them on the device inside
 * the scan (trace.cpp:111-116); NULL or n == 0 switches back to records.
 * srlg_engine_records counts the records the packets produced. */
int srlg_engine_set_anet(srlg_engine* e, const srlg_anet* anet);
/* Binary trace ingest: a file of 16 B little-endian {u64 ts_us, u32, u32}
 * records (TraceRecord / RawPacket layout, trace.hpp:14-29; raw packets
 * {ts, src, dst} when the engine has an anet) fed through
 * srlg_engine_process in 1 Mi-record blocks. SRLG_ERR_PARSE when the file
 * cannot be opened (TraceReader's message), SRLG_ERR_FORMAT on a trailing
 * partial record. *n_read = records (or packets) read. */
int srlg_engine_process_file(srlg_engine* e, const char* path, uint64_t* n_read);
/* diagnostics: per-op device spans of persistent batches ({kind 0 scan / 1
 * detect, first-CTA start ns, last-CTA end ns} triples, globaltimer) */
int srlg_engine_trace_ops(srlg_engine* e, int on);
/* diagnostics: mean µs per detection phase (A1 hot SREs, barrier, B
 * reconstruction || A2 SLEA counts, barrier, C USLE weights, epilogue) since
 * the last call; call before srlg_engine_detect_latency (which resets the
 * window count) */
int srlg_engine_detect_phases(srlg_engine* e, double* out6);
int srlg_engine_detect_diag(srlg_engine* e, double* out16);
int srlg_engine_read_io_trace(srlg_engine* e, float* out, uint64_t cap, uint64_t* n);
int srlg_engine_read_cta_trace(srlg_engine* e, uint64_t* out, uint64_t cap, uint64_t* n_ops,
                               uint64_t* grid);
int srlg_engine_read_op_trace(srlg_engine* e, uint64_t* out, uint64_t cap, uint64_t* n);
/* host<->device bytes moved by the library since the last call */
int srlg_io_bytes(int device, uint64_t* h2d, uint64_t* d2h);
/* roofline microbenchmark: best rate (updates/s) of n_updates random u32
 * stores (mode 0) or red.global.max (mode 1) into n_cells u32 */
int srlg_bench_random_updates(int device, uint64_t n_cells, uint64_t n_updates, int mode,
                              int reps, double* updates_per_s);
/* the same on a trace's own address distribution: the cell indices of n
 * device-resident pairs under (rs, le) are replayed as red.max into a fresh
 * buffer of the sketches' footprint; *n_updates = indices per replay */
int srlg_bench_trace_updates(const srlg_rsra* rs, const srlg_slea* le, const srlg_pair* dpairs,
                             uint64_t n, int reps, double* updates_per_s, uint64_t* n_updates);
/* total kernels launched by the library in this process */
uint64_t srlg_kernel_launches(void);
int srlg_device_count(int* n);
/* A further execution context ("lane") on `device` with its own streams and
 * scratch, whose persistent kernels use at most `ctas` CTAs (0 = one per SM);
 * *lane_device is a device ordinal for every *_create call. Lets several
 * engines run concurrently on one GPU (virtual ranks of a merge group). */
int srlg_lane_create(int device, int ctas, int* lane_device);

#ifdef __cplusplus
}
#endif

#endif /* SRLG_H_ */
