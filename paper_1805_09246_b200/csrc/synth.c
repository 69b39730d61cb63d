/*
 * synth.c — deterministic synthetic edge-router traffic (workload generator).
 *
 * Not on the product path: it produces the benchmark / test inputs of
 * SURVEY.md §8d (C1..C5) identically for the GPU run, the CPU reference arm
 * and the oracle. Every slice is generated independently from counter-based
 * hashes, so any sub-range of slices (the bounded CPU sample) reproduces the
 * exact packets of the full trace.
 *
 * Traffic model (modelled on the reference generator gen_trace,
 * src/trace_gen.cpp:115-226, but counter-based instead of one global RNG):
 *  - background: host h (aip 10.0.0.1+h) is drawn with Zipf(bg_zipf)
 *    popularity (Walker alias table); it talks to a fixed pool of
 *    card(h) = max(1, floor(bg_max_card / (h+1)^bg_card_exp)) peers
 *    ("flow-like reuse"), so distinct pairs per window stay bounded;
 *  - planted super hosts: peer j of host p appears in every slice congruent
 *    to j mod planted_spread (trace_gen.cpp:146-166), cardinality uniform in
 *    [planted_min, planted_max];
 *  - DDoS victim (C5): ddos_sources distinct sources spread evenly over the
 *    trace towards one victim host;
 *  - bips never fall inside 10.0.0.0/8 (make_bip, trace_gen.cpp:107-111);
 *  - each slice is shuffled (Fisher-Yates) so packet order is realistic.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "srlg_synth.h"

static uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

static uint64_t hash64(uint64_t key, uint64_t seed) {
  return mix64(mix64(seed) + key * 0x9e3779b97f4a7c15ULL);
}

static uint32_t make_bip(uint32_t v) {
  if ((v & 0xFF000000u) == 0x0A000000u) v ^= 0x80000000u;
  return v;
}

struct srlg_synth {
  srlg_synth_spec spec;
  uint32_t* card;    /* background pool size per host */
  uint32_t* base;    /* background bip base per host */
  double* prob;      /* alias table */
  uint32_t* alias;
  uint32_t* pcard;   /* planted cardinalities */
  uint32_t* pbase;
  uint64_t pkts_base, pkts_extra;
  uint64_t ddos_base, ddos_extra;
};

static uint32_t bounded(uint64_t h, uint64_t n) {
  return (uint32_t)(((h >> 32) * n) >> 32);
}

srlg_synth* srlg_synth_create(const srlg_synth_spec* spec) {
  if (spec->n_slices == 0) return NULL;
  srlg_synth* g = (srlg_synth*)calloc(1, sizeof *g);
  g->spec = *spec;
  const uint64_t n = spec->bg_hosts;
  const uint64_t seed = spec->seed;
  if (n) {
    g->card = (uint32_t*)malloc(n * 4);
    g->base = (uint32_t*)malloc(n * 4);
    g->prob = (double*)malloc(n * 8);
    g->alias = (uint32_t*)malloc(n * 4);
    double* w = (double*)malloc(n * 8);
    double total = 0;
    for (uint64_t h = 0; h < n; ++h) {
      double c = floor((double)spec->bg_max_card / pow((double)(h + 1), spec->bg_card_exp));
      if (c < 1) c = 1;
      g->card[h] = (uint32_t)c;
      g->base[h] = (uint32_t)hash64(h, seed ^ 0xB1B1B1B1ULL);
      w[h] = 1.0 / pow((double)(h + 1), spec->bg_zipf);
      total += w[h];
    }
    /* Walker alias table (Vose's construction), deterministic */
    uint32_t* small = (uint32_t*)malloc(n * 4);
    uint32_t* large = (uint32_t*)malloc(n * 4);
    uint64_t ns = 0, nl = 0;
    for (uint64_t h = 0; h < n; ++h) {
      w[h] = w[h] * (double)n / total;
      if (w[h] < 1.0) small[ns++] = (uint32_t)h;
      else large[nl++] = (uint32_t)h;
    }
    while (ns && nl) {
      const uint32_t s = small[--ns], l = large[--nl];
      g->prob[s] = w[s];
      g->alias[s] = l;
      w[l] = (w[l] + w[s]) - 1.0;
      if (w[l] < 1.0) small[ns++] = l;
      else large[nl++] = l;
    }
    while (nl) {
      const uint32_t l = large[--nl];
      g->prob[l] = 1.0;
      g->alias[l] = l;
    }
    while (ns) {
      const uint32_t s = small[--ns];
      g->prob[s] = 1.0;
      g->alias[s] = s;
    }
    free(small);
    free(large);
    free(w);
  }
  if (spec->planted) {
    g->pcard = (uint32_t*)malloc(spec->planted * 4);
    g->pbase = (uint32_t*)malloc(spec->planted * 4);
    const uint64_t span = (uint64_t)spec->planted_max - spec->planted_min + 1;
    for (uint64_t p = 0; p < spec->planted; ++p) {
      g->pcard[p] = spec->planted_min + (uint32_t)(hash64(p, seed ^ 0xC4C4C4C4ULL) % span);
      g->pbase[p] = (uint32_t)hash64(p, seed ^ 0xB2B2B2B2ULL);
    }
  }
  g->pkts_base = spec->packets / spec->n_slices;
  g->pkts_extra = spec->packets % spec->n_slices;
  g->ddos_base = spec->ddos_sources / spec->n_slices;
  g->ddos_extra = spec->ddos_sources % spec->n_slices;
  return g;
}

void srlg_synth_destroy(srlg_synth* g) {
  if (!g) return;
  free(g->card);
  free(g->base);
  free(g->prob);
  free(g->alias);
  free(g->pcard);
  free(g->pbase);
  free(g);
}

uint32_t srlg_synth_planted_aip(const srlg_synth* g, uint64_t p) {
  return 0x0A000001u + (uint32_t)g->spec.bg_hosts + (uint32_t)p;
}
uint32_t srlg_synth_planted_card(const srlg_synth* g, uint64_t p) { return g->pcard[p]; }
uint32_t srlg_synth_victim_aip(const srlg_synth* g) { (void)g; return 0x0AFFFFFEu; }

static uint64_t planted_in_slice(const srlg_synth* g, uint64_t s) {
  const uint64_t spread = g->spec.planted_spread ? g->spec.planted_spread : 1;
  const uint64_t r0 = s % spread;
  uint64_t n = 0;
  for (uint64_t p = 0; p < g->spec.planted; ++p)
    if (g->pcard[p] > r0) n += (g->pcard[p] - r0 + spread - 1) / spread;
  return n;
}

static uint64_t ddos_in_slice(const srlg_synth* g, uint64_t s) {
  return g->ddos_base + (s < g->ddos_extra ? 1 : 0);
}

uint64_t srlg_synth_slice_packets(const srlg_synth* g, uint64_t s) {
  const uint64_t budget = g->pkts_base + (s < g->pkts_extra ? 1 : 0);
  const uint64_t fixed = planted_in_slice(g, s) + ddos_in_slice(g, s);
  if (g->spec.bg_hosts == 0) return fixed;
  return budget > fixed ? budget : fixed;
}

static void gen_slice(const srlg_synth* g, uint64_t s, srlg_pair* out, uint64_t n) {
  const srlg_synth_spec* sp = &g->spec;
  uint64_t k = 0;
  /* planted hosts */
  const uint64_t spread = sp->planted_spread ? sp->planted_spread : 1;
  for (uint64_t p = 0; p < sp->planted; ++p) {
    const uint32_t aip = srlg_synth_planted_aip(g, p);
    for (uint64_t j = s % spread; j < g->pcard[p]; j += spread) {
      out[k].aip = aip;
      out[k].bip = make_bip(g->pbase[p] + (uint32_t)j);
      ++k;
    }
  }
  /* DDoS victim: globally distinct source indices */
  if (sp->ddos_sources) {
    const uint64_t cnt = ddos_in_slice(g, s);
    const uint64_t first = s * g->ddos_base + (s < g->ddos_extra ? s : g->ddos_extra);
    const uint32_t vbase = (uint32_t)hash64(7, sp->seed ^ 0xD0D0D0D0ULL);
    for (uint64_t j = 0; j < cnt; ++j) {
      out[k].aip = srlg_synth_victim_aip(g);
      out[k].bip = make_bip(vbase + (uint32_t)(first + j));
      ++k;
    }
  }
  /* background */
  const uint64_t sseed = hash64(s, sp->seed ^ 0xA5A5A5A5ULL);
  for (uint64_t i = 0; k < n; ++i, ++k) {
    const uint64_t h1 = mix64(sseed + (2 * i + 1) * 0x9e3779b97f4a7c15ULL);
    const uint64_t h2 = mix64(sseed + (2 * i + 2) * 0x9e3779b97f4a7c15ULL);
    uint32_t host = bounded(h1, sp->bg_hosts);
    const double coin = (double)(h1 & 0xFFFFFFFFu) * (1.0 / 4294967296.0);
    if (coin >= g->prob[host]) host = g->alias[host];
    const uint32_t j = bounded(h2, g->card[host]);
    out[k].aip = 0x0A000001u + host;
    out[k].bip = make_bip(g->base[host] + j);
  }
  /* Fisher-Yates, per-slice stream */
  uint64_t st = hash64(s, sp->seed ^ 0x5F5F5F5FULL);
  for (uint64_t i = n; i > 1; --i) {
    st += 0x9e3779b97f4a7c15ULL;
    const uint64_t j = mix64(st) % i;
    const srlg_pair t = out[i - 1];
    out[i - 1] = out[j];
    out[j] = t;
  }
}

uint64_t srlg_synth_offsets(const srlg_synth* g, uint64_t first_slice, uint64_t n_slices,
                            uint64_t* offsets) {
  offsets[0] = 0;
  for (uint64_t s = 0; s < n_slices; ++s)
    offsets[s + 1] = offsets[s] + srlg_synth_slice_packets(g, first_slice + s);
  return offsets[n_slices];
}

typedef struct job {
  const srlg_synth* g;
  uint64_t first, n_slices, stride, start;
  const uint64_t* offsets;
  srlg_pair* out;
} job;

static void* worker(void* arg) {
  job* j = (job*)arg;
  for (uint64_t s = j->start; s < j->n_slices; s += j->stride)
    gen_slice(j->g, j->first + s, j->out + j->offsets[s], j->offsets[s + 1] - j->offsets[s]);
  return NULL;
}

int srlg_synth_generate(const srlg_synth* g, uint64_t first_slice, uint64_t n_slices,
                        const uint64_t* offsets, srlg_pair* out, uint32_t threads) {
  if (threads <= 1 || n_slices == 1) {
    for (uint64_t s = 0; s < n_slices; ++s)
      gen_slice(g, first_slice + s, out + offsets[s], offsets[s + 1] - offsets[s]);
    return 0;
  }
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  job jobs[256];
  for (uint32_t t = 0; t < threads; ++t) {
    jobs[t] = (job){g, first_slice, n_slices, threads, t, offsets, out};
    pthread_create(&tid[t], NULL, worker, &jobs[t]);
  }
  for (uint32_t t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  return 0;
}
