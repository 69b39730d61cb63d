/*
 * srlg_oracle.h — TEST INFRASTRUCTURE ONLY: the CPU checker.
 *
 * A plain-C restatement of the reference algorithm for the hot path
 * (slidecard, /root/reference/proj/core), kept in the reference's own
 * representation: u16 "slices since last set" distances, 0xFFFF = never set
 * (sliding_counters.hpp:10), a saturating O(cells) slide and a per-cell min
 * merge. It deliberately shares nothing with the device implementation
 * (which keeps u32 stamps), so agreement between the two checks the stamp /
 * distance bijection as well as the kernels.
 *
 * Parity of this restatement is pinned against the reference itself
 * (oracle/_ref/libslidecard_ref.so built from /root/reference by
 * oracle/Makefile) and against committed golden fixtures generated from it
 * (tests/golden/, tests/golden/make_golden.py).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline) may load
 * this library; the product path never does.
 */
#ifndef SRLG_ORACLE_H_
#define SRLG_ORACLE_H_

#include "srlg.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* ora_last_error(void);

uint64_t ora_mix64(uint64_t x);
uint64_t ora_hash64(uint64_t key, uint64_t seed);
uint32_t ora_lsb(uint32_t x);
uint32_t ora_sampling_threshold(uint64_t theta, uint64_t eta);
double ora_detection_rho(void);
int ora_le_estimate(double weight, uint32_t eta_prime, double* value, int* saturated);
int ora_corrected_weight(double w, double sfp, uint32_t eta_prime, double* out);

int ora_params_validate(const srlg_params* p);
int ora_params_configs(const srlg_params* p, srlg_rsra_config* rc, srlg_slea_config* sc);

typedef struct ora_sketch ora_sketch;

ora_sketch* ora_sketch_create(const srlg_rsra_config* rc, const srlg_slea_config* sc);
ora_sketch* ora_sketch_clone(const ora_sketch* s);
void ora_sketch_destroy(ora_sketch* s);
void ora_update(ora_sketch* s, const srlg_pair* pairs, uint64_t n);
void ora_update_rsra_only(ora_sketch* s, const srlg_pair* pairs, uint64_t n);
void ora_update_slea_only(ora_sketch* s, const srlg_pair* pairs, uint64_t n);
void ora_slide(ora_sketch* s);
void ora_reinit(ora_sketch* s);
uint64_t ora_slides(const ora_sketch* s);
void ora_set_slides(ora_sketch* s, uint64_t v);
uint64_t ora_rsra_ncells(const ora_sketch* s);
uint64_t ora_slea_ncells(const ora_sketch* s);
uint64_t ora_slea_row_length(const ora_sketch* s);
void ora_export(const ora_sketch* s, uint16_t* rsra, uint16_t* slea);
void ora_import(ora_sketch* s, const uint16_t* rsra, const uint16_t* slea);
int ora_merge_min(ora_sketch* a, const ora_sketch* b);
int ora_extract_hot(const ora_sketch* s, uint32_t k, uint32_t* cols, uint64_t cap,
                    uint64_t* row_counts);
int ora_estimate_context(const ora_sketch* s, uint32_t k, double* factors, double* sfp);
int ora_estimate(const ora_sketch* s, uint32_t aip, uint32_t k, srlg_estimate* out);
uint32_t ora_lh_column(const ora_sketch* s, uint32_t row, uint32_t aip);

int ora_forward(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t aip,
                uint32_t* cols);
int ora_group_info(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t* uncovered,
                   int* covers);
int ora_invert(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, const uint32_t* cols,
               uint32_t* out, uint64_t cap, uint64_t* n);
int ora_reconstruct(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed,
                    const uint32_t* hot_cols, const uint64_t* row_counts, uint64_t tuple_cap,
                    uint64_t work_cap, uint32_t workers, uint32_t* out, uint64_t cap,
                    uint64_t* n, int* overflow, uint64_t* checked, uint64_t* kept);
int ora_detect(const ora_sketch* s, const srlg_window_config* wc, uint64_t window_end,
               int partial, uint8_t* blob, uint64_t cap, uint64_t* bytes);

typedef struct ora_engine ora_engine;
ora_engine* ora_engine_create(const srlg_rsra_config* rc, const srlg_slea_config* sc,
                              const srlg_window_config* wc);
void ora_engine_destroy(ora_engine* e);
int ora_engine_process(ora_engine* e, const srlg_record* recs, uint64_t n);
int ora_engine_process_slices(ora_engine* e, const srlg_pair* pairs, const uint64_t* offsets,
                              uint64_t n_slices, uint64_t first_slice);
int ora_engine_advance(ora_engine* e, uint64_t slice);
int ora_engine_finish(ora_engine* e);
uint64_t ora_engine_take_reports(ora_engine* e, uint8_t* blob, uint64_t cap,
                                 uint64_t* n_reports);
uint64_t ora_engine_current_slice(const ora_engine* e);
void ora_engine_export(const ora_engine* e, uint16_t* rsra, uint16_t* slea);

int ora_run_distributed(const srlg_record* recs, uint64_t n, const srlg_rsra_config* rc,
                        const srlg_slea_config* sc, const srlg_window_config* wc,
                        uint32_t nodes, uint32_t policy, uint8_t* blob, uint64_t cap,
                        uint64_t* bytes, uint64_t* n_reports, uint64_t* slice_merges,
                        uint64_t* bytes_exchanged);

void ora_rng_pairs(uint64_t seed, uint64_t n, srlg_pair* out);
uint64_t ora_fnv1a64_u16(const uint16_t* v, uint64_t n);

#ifdef __cplusplus
}
#endif

#endif
