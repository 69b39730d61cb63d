/* srlg_synth.h — deterministic synthetic traffic (benchmark/test inputs). */
#ifndef SRLG_SYNTH_H_
#define SRLG_SYNTH_H_

#include <stdint.h>

#include "srlg.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct srlg_synth_spec {
  uint64_t seed;
  uint64_t n_slices;
  uint64_t packets;       /* total packet budget, spread evenly over slices */
  uint64_t bg_hosts;      /* background aips 10.0.0.1 .. */
  double bg_zipf;         /* host popularity exponent */
  double bg_card_exp;     /* pool size exponent: card = max_card / (h+1)^exp */
  uint32_t bg_max_card;
  uint32_t planted;       /* planted super hosts */
  uint32_t planted_min;
  uint32_t planted_max;
  uint32_t planted_spread;
  uint32_t reserved;
  uint64_t ddos_sources;  /* distinct sources towards one victim (C5) */
} srlg_synth_spec;

typedef struct srlg_synth srlg_synth;

srlg_synth* srlg_synth_create(const srlg_synth_spec* spec);
void srlg_synth_destroy(srlg_synth* g);
uint64_t srlg_synth_slice_packets(const srlg_synth* g, uint64_t slice);
/* offsets[n_slices+1] of slices first..first+n-1; returns total packets */
uint64_t srlg_synth_offsets(const srlg_synth* g, uint64_t first_slice, uint64_t n_slices,
                            uint64_t* offsets);
int srlg_synth_generate(const srlg_synth* g, uint64_t first_slice, uint64_t n_slices,
                        const uint64_t* offsets, srlg_pair* out, uint32_t threads);
uint32_t srlg_synth_planted_aip(const srlg_synth* g, uint64_t p);
uint32_t srlg_synth_planted_card(const srlg_synth* g, uint64_t p);
uint32_t srlg_synth_victim_aip(const srlg_synth* g);

#ifdef __cplusplus
}
#endif

#endif
