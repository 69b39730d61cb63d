/*
 * srlg_oracle.c — TEST INFRASTRUCTURE ONLY: plain-C restatement of the
 * reference hot path, used as the checker for the CUDA path. See
 * srlg_oracle.h for the contract. Each function cites the reference
 * file:line it restates (paths relative to /root/reference/proj/core).
 *
 * Parity is pinned against the reference built from its own sources
 * (oracle/_ref) and the golden fixtures in tests/golden/.
 */
#include "srlg_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NEVER 0xFFFFu

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* ora_last_error(void) { return g_err; }

/* ------------------------------------------------------------ hashing ---- */

static const uint64_t kGolden64 = 0x9e3779b97f4a7c15ULL; /* hash.hpp:11 */

/* mix64 (include/slidecard/hash.hpp:14-21) */
uint64_t ora_mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

/* hash64 (hash.hpp:23-25) */
uint64_t ora_hash64(uint64_t key, uint64_t seed) {
  return ora_mix64(ora_mix64(seed) + key * kGolden64);
}

/* SeededHash (hash.hpp:28-39): offset = mix64(seed) */
static uint64_t seeded(uint64_t offset, uint64_t key) { return ora_mix64(offset + key * kGolden64); }

/* lsb (hash.hpp:44-46) */
uint32_t ora_lsb(uint32_t x) { return x == 0 ? 32u : (uint32_t)__builtin_ctz(x); }

/* sampling_threshold (src/hash.cpp:10-16) */
uint32_t ora_sampling_threshold(uint64_t theta, uint64_t eta) {
  uint32_t t = 0;
  if (eta == 0) return 0;
  while (t < 64 && eta <= (UINT64_MAX >> t) && (eta << t) < theta) ++t;
  return t;
}

/* detection_rho (src/sliding_counters.cpp:50) */
double ora_detection_rho(void) { return 0.99 * (1.0 - exp(-1.0 / 3.0)); }

/* le_estimate (src/linear_counting.cpp:10-15) */
int ora_le_estimate(double weight, uint32_t eta_prime, double* value, int* saturated) {
  const double eta = (double)eta_prime;
  if (weight <= 0.0) {
    *value = 0.0;
    *saturated = 0;
  } else if (weight >= eta) {
    *value = eta * log(eta);
    *saturated = 1;
  } else {
    *value = -eta * log((eta - weight) / eta);
    *saturated = 0;
  }
  return SRLG_OK;
}

/* corrected_weight (src/linear_counting.cpp:17-24) */
int ora_corrected_weight(double usle, double sfp, uint32_t eta_prime, double* out) {
  if (sfp >= 1.0)
    return fail(SRLG_ERR_SATURATION,
                "corrected weight: setting-factor product is 1, estimate unusable");
  if (sfp < 0.0) sfp = 0.0;
  const double eta = (double)eta_prime;
  double w = (usle - eta * sfp) / (1.0 - sfp);
  /* std::clamp(w, 0.0, eta) */
  if (w < 0.0) w = 0.0;
  else if (eta < w) w = eta;
  *out = w;
  return SRLG_OK;
}

/* -------------------------------------------------------------- params --- */

/* SketchParams::validate (src/config.cpp:20-42) */
int ora_params_validate(const srlg_params* p) {
  if (p->q < 1 || p->q > 30) return fail(SRLG_ERR_CONFIG, "q must be in [1, 30]");
  if (p->q_prime < 1 || p->q_prime > 30) return fail(SRLG_ERR_CONFIG, "q_prime must be in [1, 30]");
  if (p->r < 3 || p->r > 64) return fail(SRLG_ERR_CONFIG, "r must be in [3, 64]");
  if (p->r_prime < 1 || p->r_prime > 64) return fail(SRLG_ERR_CONFIG, "r_prime must be in [1, 64]");
  if (p->delta < 1 || p->delta >= p->q)
    return fail(SRLG_ERR_CONFIG, "delta must satisfy 1 <= delta < q");
  if ((uint64_t)(p->r - 2) * p->delta + p->q < 32)
    return fail(SRLG_ERR_CONFIG, "(r-2)*delta + q must be at least 32 to cover the address bits");
  if (p->eta < 1 || p->eta > 65535) return fail(SRLG_ERR_CONFIG, "eta must be in [1, 65535]");
  if (p->eta_prime < 2 || p->eta_prime > (1u << 26))
    return fail(SRLG_ERR_CONFIG, "eta_prime must be in [2, 2^26]");
  if (p->delta_prime < 1 || p->delta_prime > p->eta_prime)
    return fail(SRLG_ERR_CONFIG, "delta_prime must satisfy 1 <= delta_prime <= eta_prime");
  if (p->theta < p->eta) return fail(SRLG_ERR_CONFIG, "theta must be at least eta");
  if (ora_sampling_threshold(p->theta, p->eta) > 32)
    return fail(SRLG_ERR_CONFIG, "theta/eta ratio pushes the sampling threshold past 32 bits");
  const uint64_t rough = ((uint64_t)1 << p->q) * p->r * p->eta;
  const uint64_t linear =
      (((uint64_t)1 << p->q_prime) * p->delta_prime + p->eta_prime - p->delta_prime) * p->r_prime;
  if (rough > ((uint64_t)1 << 31) || linear > ((uint64_t)1 << 31))
    return fail(SRLG_ERR_CONFIG, "parameter set needs more than 2^31 counters; reduce q or q_prime");
  return SRLG_OK;
}

/* rsra_config / slea_config (src/config.cpp:48-72) with HashSeeds::derive
 * (src/hash.cpp:18-27) */
int ora_params_configs(const srlg_params* p, srlg_rsra_config* rc, srlg_slea_config* sc) {
  int st = ora_params_validate(p);
  if (st) return st;
  memset(rc, 0, sizeof *rc);
  memset(sc, 0, sizeof *sc);
  rc->q = p->q;
  rc->r = p->r;
  rc->delta = p->delta;
  rc->eta = p->eta;
  rc->tau = ora_sampling_threshold(p->theta, p->eta);
  rc->seed_h1 = ora_hash64(1, p->seed);
  rc->seed_h2 = ora_hash64(2, p->seed);
  rc->seed_rhfg0 = ora_hash64(4, p->seed);
  sc->q = p->q_prime;
  sc->r = p->r_prime;
  sc->delta = p->delta_prime;
  sc->eta = p->eta_prime;
  sc->seed_h3 = ora_hash64(3, p->seed);
  for (uint32_t i = 0; i < p->r_prime; ++i) sc->seeds_lh[i] = ora_hash64(100 + i, p->seed);
  return SRLG_OK;
}

/* ---------------------------------------------- reversible hash group --- */

typedef struct group {
  uint32_t q, r, delta, col_mask, overlap_mask, uncovered;
  uint64_t h0_off;
} group;

/* ReversibleHashGroup ctor (src/hash.cpp:39-57) */
static int group_init(group* g, uint32_t q, uint32_t r, uint32_t delta, uint64_t seed) {
  if (q == 0 || q > 31) return fail(SRLG_ERR_CONFIG, "hash group: q must be in [1, 31]");
  if (r < 2) return fail(SRLG_ERR_CONFIG, "hash group: need at least 2 rows");
  if (delta == 0 || delta >= q)
    return fail(SRLG_ERR_CONFIG, "hash group: delta must satisfy 1 <= delta < q");
  g->q = q;
  g->r = r;
  g->delta = delta;
  g->col_mask = (1u << q) - 1;
  g->overlap_mask = (1u << (q - delta)) - 1;
  g->h0_off = ora_mix64(seed);
  uint64_t covered = 0;
  for (uint32_t i = 1; i < r; ++i) {
    const uint32_t lo = i * delta;
    if (lo >= 32) break;
    const uint32_t hi = lo + q < 32 ? lo + q : 32;
    covered |= (((uint64_t)1 << (hi - lo)) - 1) << lo;
  }
  g->uncovered = (uint32_t)(~covered & 0xFFFFFFFFull);
  return SRLG_OK;
}

/* covers_address (src/hash.cpp:59-61) */
static int group_covers(const group* g) { return (uint64_t)(g->r - 2) * g->delta + g->q >= 32; }

/* forward (src/hash.cpp:63-69) */
static void group_forward(const group* g, uint32_t aip, uint32_t* out) {
  out[0] = (uint32_t)seeded(g->h0_off, aip) & g->col_mask;
  for (uint32_t i = 1; i < g->r; ++i) {
    const uint32_t shifted = i * g->delta >= 32 ? 0u : aip >> (i * g->delta);
    out[i] = (shifted ^ out[0]) & g->col_mask;
  }
}

/* windows_consistent (include/slidecard/hash.hpp:101-103) */
static int windows_consistent(const group* g, uint32_t b_prev, uint32_t b_cur) {
  return (b_prev >> g->delta) == (b_cur & g->overlap_mask);
}

static int cmp_u32(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

typedef struct u32vec {
  uint32_t* v;
  uint64_t n, cap;
} u32vec;

static void vec_push(u32vec* a, uint32_t x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? a->cap * 2 : 64;
    a->v = (uint32_t*)realloc(a->v, a->cap * sizeof(uint32_t));
  }
  a->v[a->n++] = x;
}

/* invert (src/hash.cpp:77-112). Appends verified addresses (sorted) to out. */
static int group_invert(const group* g, const uint32_t* cols, u32vec* out) {
  uint32_t window[SRLG_MAX_ROWS] = {0};
  for (uint32_t i = 1; i < g->r; ++i) window[i] = (cols[i] ^ cols[0]) & g->col_mask;
  for (uint32_t i = 2; i < g->r; ++i)
    if (!windows_consistent(g, window[i - 1], window[i])) return SRLG_OK;
  uint64_t known = 0;
  for (uint32_t i = 1; i < g->r; ++i) {
    /* i*delta >= 64 is undefined behaviour in the reference (hash.cpp:90);
     * such parameter sets are outside the parity contract. */
    const uint32_t sh = i * g->delta;
    if (sh < 64) known |= (uint64_t)window[i] << sh;
  }
  const uint32_t assembled = (uint32_t)(known & 0xFFFFFFFFull);
  uint32_t free_bits[32];
  uint32_t n_free = 0;
  for (uint32_t b = 0; b < 32; ++b)
    if (g->uncovered & (1u << b)) free_bits[n_free++] = b;
  if (n_free > 26)
    return fail(SRLG_ERR_RESOURCE,
                "invert: parameter set leaves too many address bits unconstrained");
  const uint64_t start = out->n;
  uint32_t image[SRLG_MAX_ROWS];
  for (uint64_t v = 0; v < ((uint64_t)1 << n_free); ++v) {
    uint32_t cand = assembled & ~g->uncovered;
    for (uint32_t b = 0; b < n_free; ++b)
      if (v & ((uint64_t)1 << b)) cand |= 1u << free_bits[b];
    group_forward(g, cand, image);
    if (memcmp(image, cols, g->r * sizeof(uint32_t)) == 0) vec_push(out, cand);
  }
  qsort(out->v + start, out->n - start, sizeof(uint32_t), cmp_u32);
  return SRLG_OK;
}

int ora_forward(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t aip,
                uint32_t* cols) {
  group g;
  int st = group_init(&g, q, r, delta, seed);
  if (st) return st;
  group_forward(&g, aip, cols);
  return SRLG_OK;
}

int ora_group_info(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, uint32_t* uncovered,
                   int* covers) {
  group g;
  int st = group_init(&g, q, r, delta, seed);
  if (st) return st;
  *uncovered = g.uncovered;
  *covers = group_covers(&g);
  return SRLG_OK;
}

int ora_invert(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed, const uint32_t* cols,
               uint32_t* out, uint64_t cap, uint64_t* n) {
  group g;
  int st = group_init(&g, q, r, delta, seed);
  if (st) return st;
  u32vec v = {0};
  st = group_invert(&g, cols, &v);
  if (st) {
    free(v.v);
    return st;
  }
  *n = v.n;
  for (uint64_t i = 0; i < v.n && i < cap; ++i) out[i] = v.v[i];
  free(v.v);
  return SRLG_OK;
}

/* reconstruct_candidates (src/reconstruct.cpp:32-151), single worker. The
 * result does not depend on the worker count (reconstruct.cpp:21-28 splices
 * in worker order and the output is sorted + unique). */
static int reconstruct(const group* g, uint32_t* const* hot, const uint64_t* cnt,
                       uint64_t tuple_cap, uint64_t work_cap, u32vec* addrs, int* overflow,
                       uint64_t* checked, uint64_t* kept) {
  const uint32_t r = g->r;
  *overflow = 0;
  *checked = 0;
  *kept = 0;
  addrs->n = 0;
  if (r < 3) return fail(SRLG_ERR_INVALID_ARGUMENT, "reconstruct: need at least 3 rows");
  for (uint32_t i = 0; i < r; ++i)
    if (cnt[i] == 0) return SRLG_OK;

  const uint64_t seed_work = cnt[0] * cnt[1] * cnt[2];
  if (seed_work > work_cap) goto overflowed;

  u32vec tuples = {0}, next = {0};
  uint64_t n_kept = 0;
  for (uint64_t a = 0; a < cnt[0]; ++a) {
    const uint32_t he0 = hot[0][a];
    for (uint64_t b = 0; b < cnt[1]; ++b) {
      const uint32_t he1 = hot[1][b];
      const uint32_t b1 = he1 ^ he0;
      for (uint64_t c = 0; c < cnt[2]; ++c) {
        const uint32_t he2 = hot[2][c];
        const uint32_t b2 = he2 ^ he0;
        if (!windows_consistent(g, b1, b2)) continue;
        vec_push(&tuples, he0);
        vec_push(&tuples, he1);
        vec_push(&tuples, he2);
        if (++n_kept > tuple_cap) {
          free(tuples.v);
          goto overflowed;
        }
      }
    }
  }
  *checked += seed_work;

  for (uint32_t row = 3; row < r; ++row) {
    const uint32_t width = row;
    const uint64_t count = tuples.n / width;
    const uint64_t work = count * cnt[row];
    if (*checked + work > work_cap) {
      free(tuples.v);
      free(next.v);
      goto overflowed;
    }
    next.n = 0;
    n_kept = 0;
    for (uint64_t t = 0; t < count; ++t) {
      const uint32_t* tuple = tuples.v + t * width;
      const uint32_t he0 = tuple[0];
      const uint32_t b_prev = tuple[width - 1] ^ he0;
      for (uint64_t j = 0; j < cnt[row]; ++j) {
        const uint32_t he = hot[row][j];
        if (!windows_consistent(g, b_prev, he ^ he0)) continue;
        for (uint32_t w = 0; w < width; ++w) vec_push(&next, tuple[w]);
        vec_push(&next, he);
        if (++n_kept > tuple_cap) {
          free(tuples.v);
          free(next.v);
          goto overflowed;
        }
      }
    }
    *checked += work;
    u32vec tmp = tuples;
    tuples = next;
    next = tmp;
  }
  free(next.v);

  const uint64_t final_count = tuples.n / r;
  *kept = final_count;
  for (uint64_t t = 0; t < final_count; ++t) {
    int st = group_invert(g, tuples.v + t * r, addrs);
    if (st) {
      free(tuples.v);
      return st;
    }
  }
  free(tuples.v);
  qsort(addrs->v, addrs->n, sizeof(uint32_t), cmp_u32);
  uint64_t u = 0;
  for (uint64_t i = 0; i < addrs->n; ++i)
    if (u == 0 || addrs->v[u - 1] != addrs->v[i]) addrs->v[u++] = addrs->v[i];
  addrs->n = u;
  return SRLG_OK;

overflowed:
  addrs->n = 0;
  *overflow = 1;
  *checked = 0;
  *kept = 0;
  return SRLG_OK;
}

int ora_reconstruct(uint32_t q, uint32_t r, uint32_t delta, uint64_t seed,
                    const uint32_t* hot_cols, const uint64_t* row_counts, uint64_t tuple_cap,
                    uint64_t work_cap, uint32_t workers, uint32_t* out, uint64_t cap,
                    uint64_t* n, int* overflow, uint64_t* checked, uint64_t* kept) {
  (void)workers;
  group g;
  int st = group_init(&g, q, r, delta, seed);
  if (st) return st;
  uint32_t* hot[SRLG_MAX_ROWS];
  uint64_t off = 0;
  for (uint32_t i = 0; i < r; ++i) {
    hot[i] = (uint32_t*)hot_cols + off;
    off += row_counts[i];
  }
  u32vec a = {0};
  st = reconstruct(&g, hot, row_counts, tuple_cap, work_cap, &a, overflow, checked, kept);
  if (st == SRLG_OK) {
    *n = a.n;
    for (uint64_t i = 0; i < a.n && i < cap; ++i) out[i] = a.v[i];
  }
  free(a.v);
  return st;
}

/* --------------------------------------------------- sliding counters --- */

/* counter_ops::slide (src/sliding_counters.cpp:18-22) */
static void counters_slide(uint16_t* p, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) p[i] += (uint16_t)(p[i] != NEVER);
}

/* counter_ops::weight (src/sliding_counters.cpp:24-32) */
static uint64_t counters_weight(const uint16_t* p, uint64_t n, uint32_t k) {
  if (k > NEVER) k = NEVER;
  const uint16_t kk = (uint16_t)k;
  uint64_t c = 0;
  for (uint64_t i = 0; i < n; ++i) c += p[i] < kk;
  return c;
}

/* ------------------------------------------------------------ sketches --- */

struct ora_sketch {
  srlg_rsra_config rc;
  srlg_slea_config sc;
  group g;
  uint64_t h1_off, h2_off, h3_off, lh_off[SRLG_MAX_ROWS];
  uint16_t* rs; /* r x 2^q x eta */
  uint16_t* le; /* r' x row_len */
  uint64_t rs_n, le_n, row_len;
  uint64_t rs_slides, le_slides;
};

/* Rsra ctor (src/rsra.cpp:9-23) + Slea ctor (src/slea.cpp:11-27) */
ora_sketch* ora_sketch_create(const srlg_rsra_config* rc, const srlg_slea_config* sc) {
  ora_sketch* s = (ora_sketch*)calloc(1, sizeof *s);
  s->rc = *rc;
  s->sc = *sc;
  if (group_init(&s->g, rc->q, rc->r, rc->delta, rc->seed_rhfg0)) goto bad;
  if (rc->eta == 0) { fail(SRLG_ERR_CONFIG, "rsra: eta must be positive"); goto bad; }
  if (rc->r < 3) { fail(SRLG_ERR_CONFIG, "rsra: need at least 3 rows to reconstruct hosts"); goto bad; }
  if (rc->r > 64) { fail(SRLG_ERR_CONFIG, "rsra: at most 64 rows supported"); goto bad; }
  if (!group_covers(&s->g)) {
    fail(SRLG_ERR_CONFIG, "rsra: (r-2)*delta + q must reach the 32 address bits");
    goto bad;
  }
  s->rs_n = ((uint64_t)1 << rc->q) * rc->r * rc->eta;
  if (s->rs_n > ((uint64_t)1 << 31)) {
    fail(SRLG_ERR_CONFIG, "rsra: parameter set needs more than 2^31 counters");
    goto bad;
  }
  if (sc->r == 0) { fail(SRLG_ERR_CONFIG, "slea: need at least one row"); goto bad; }
  if (sc->r > 64) { fail(SRLG_ERR_CONFIG, "slea: at most 64 rows supported"); goto bad; }
  if (sc->eta < 2) { fail(SRLG_ERR_CONFIG, "slea: eta must be at least 2"); goto bad; }
  if (sc->delta == 0 || sc->delta > sc->eta) {
    fail(SRLG_ERR_CONFIG, "slea: delta must satisfy 0 < delta <= eta");
    goto bad;
  }
  if (sc->q > 30) { fail(SRLG_ERR_CONFIG, "slea: q must be at most 30"); goto bad; }
  s->row_len = ((uint64_t)1 << sc->q) * sc->delta + sc->eta - sc->delta; /* slea.hpp:33-35 */
  s->le_n = s->row_len * sc->r;
  if (s->le_n > ((uint64_t)1 << 31)) {
    fail(SRLG_ERR_CONFIG, "slea: parameter set needs more than 2^31 counters");
    goto bad;
  }
  s->h1_off = ora_mix64(rc->seed_h1);
  s->h2_off = ora_mix64(rc->seed_h2);
  s->h3_off = ora_mix64(sc->seed_h3);
  for (uint32_t i = 0; i < sc->r; ++i) s->lh_off[i] = ora_mix64(sc->seeds_lh[i]);
  s->rs = (uint16_t*)malloc(s->rs_n * 2);
  s->le = (uint16_t*)malloc(s->le_n * 2);
  memset(s->rs, 0xFF, s->rs_n * 2);
  memset(s->le, 0xFF, s->le_n * 2);
  return s;
bad:
  free(s);
  return NULL;
}

ora_sketch* ora_sketch_clone(const ora_sketch* s) {
  ora_sketch* c = (ora_sketch*)malloc(sizeof *c);
  *c = *s;
  c->rs = (uint16_t*)malloc(s->rs_n * 2);
  c->le = (uint16_t*)malloc(s->le_n * 2);
  memcpy(c->rs, s->rs, s->rs_n * 2);
  memcpy(c->le, s->le, s->le_n * 2);
  return c;
}

void ora_sketch_destroy(ora_sketch* s) {
  if (!s) return;
  free(s->rs);
  free(s->le);
  free(s);
}

/* Rsra::update (src/rsra.cpp:25-33) with sample_gate (src/hash.cpp:29-33) */
static void rsra_update(ora_sketch* s, uint32_t aip, uint32_t bip) {
  if (ora_lsb((uint32_t)seeded(s->h1_off, bip)) < s->rc.tau) return;
  const uint32_t slot = (uint32_t)(seeded(s->h2_off, bip) % s->rc.eta);
  uint32_t cols[SRLG_MAX_ROWS];
  group_forward(&s->g, aip, cols);
  for (uint32_t i = 0; i < s->rc.r; ++i)
    s->rs[((((uint64_t)i) << s->rc.q) + cols[i]) * s->rc.eta + slot] = 0;
}

/* Slea::lh_column (src/slea.cpp:34-36) */
uint32_t ora_lh_column(const ora_sketch* s, uint32_t row, uint32_t aip) {
  return (uint32_t)seeded(s->lh_off[row], aip) & ((1u << s->sc.q) - 1);
}

/* Slea::update (src/slea.cpp:38-45) with le_index (src/hash.cpp:35-37) */
static void slea_update(ora_sketch* s, uint32_t aip, uint32_t bip) {
  const uint32_t slot = (uint32_t)(seeded(s->h3_off, bip) % s->sc.eta);
  for (uint32_t i = 0; i < s->sc.r; ++i)
    s->le[(uint64_t)i * s->row_len + (uint64_t)ora_lh_column(s, i, aip) * s->sc.delta + slot] = 0;
}

void ora_update(ora_sketch* s, const srlg_pair* pairs, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    rsra_update(s, pairs[i].aip, pairs[i].bip);
    slea_update(s, pairs[i].aip, pairs[i].bip);
  }
}

void ora_update_rsra_only(ora_sketch* s, const srlg_pair* pairs, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) rsra_update(s, pairs[i].aip, pairs[i].bip);
}

void ora_update_slea_only(ora_sketch* s, const srlg_pair* pairs, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) slea_update(s, pairs[i].aip, pairs[i].bip);
}

/* Rsra::slide / Slea::slide (src/rsra.cpp:35-38, src/slea.cpp:47-50) */
void ora_slide(ora_sketch* s) {
  counters_slide(s->rs, s->rs_n);
  counters_slide(s->le, s->le_n);
  s->rs_slides++;
  s->le_slides++;
}

/* reinitialize (src/rsra.cpp:40-43, src/slea.cpp:52-55) */
void ora_reinit(ora_sketch* s) {
  memset(s->rs, 0xFF, s->rs_n * 2);
  memset(s->le, 0xFF, s->le_n * 2);
  s->rs_slides++;
  s->le_slides++;
}

uint64_t ora_slides(const ora_sketch* s) { return s->rs_slides; }
void ora_set_slides(ora_sketch* s, uint64_t v) { s->rs_slides = s->le_slides = v; }
uint64_t ora_rsra_ncells(const ora_sketch* s) { return s->rs_n; }
uint64_t ora_slea_ncells(const ora_sketch* s) { return s->le_n; }
uint64_t ora_slea_row_length(const ora_sketch* s) { return s->row_len; }

void ora_export(const ora_sketch* s, uint16_t* rsra, uint16_t* slea) {
  if (rsra) memcpy(rsra, s->rs, s->rs_n * 2);
  if (slea) memcpy(slea, s->le, s->le_n * 2);
}

void ora_import(ora_sketch* s, const uint16_t* rsra, const uint16_t* slea) {
  if (rsra) memcpy(s->rs, rsra, s->rs_n * 2);
  if (slea) memcpy(s->le, slea, s->le_n * 2);
}

/* compatibility_mismatch (src/rsra.cpp:64-75, src/slea.cpp:131-140) +
 * merge_min (src/rsra.cpp:77-81, src/slea.cpp:142-146) via min_into
 * (src/sliding_counters.cpp:34-39) */
int ora_merge_min(ora_sketch* a, const ora_sketch* b) {
  const srlg_rsra_config *x = &a->rc, *y = &b->rc;
  const char* why = NULL;
  if (x->q != y->q) why = "q";
  else if (x->r != y->r) why = "r";
  else if (x->delta != y->delta) why = "delta";
  else if (x->eta != y->eta) why = "eta";
  else if (x->tau != y->tau) why = "tau";
  else if (x->seed_h1 != y->seed_h1) why = "seed_h1";
  else if (x->seed_h2 != y->seed_h2) why = "seed_h2";
  else if (x->seed_rhfg0 != y->seed_rhfg0) why = "seed_rhfg0";
  else if (a->rs_slides != b->rs_slides) why = "slice position";
  if (why) return fail(SRLG_ERR_INCOMPATIBLE, "rsra merge: %s differs", why);
  const srlg_slea_config *u = &a->sc, *v = &b->sc;
  if (u->q != v->q) why = "q_prime";
  else if (u->r != v->r) why = "r_prime";
  else if (u->delta != v->delta) why = "delta_prime";
  else if (u->eta != v->eta) why = "eta_prime";
  else if (u->seed_h3 != v->seed_h3) why = "seed_h3";
  else if (memcmp(u->seeds_lh, v->seeds_lh, u->r * 8) != 0) why = "seeds_lh";
  else if (a->le_slides != b->le_slides) why = "slice position";
  if (why) return fail(SRLG_ERR_INCOMPATIBLE, "slea merge: %s differs", why);
  for (uint64_t i = 0; i < a->rs_n; ++i)
    if (b->rs[i] < a->rs[i]) a->rs[i] = b->rs[i];
  for (uint64_t i = 0; i < a->le_n; ++i)
    if (b->le[i] < a->le[i]) a->le[i] = b->le[i];
  return SRLG_OK;
}

/* Rsra::extract_hot (src/rsra.cpp:45-57) */
int ora_extract_hot(const ora_sketch* s, uint32_t k, uint32_t* cols, uint64_t cap,
                    uint64_t* row_counts) {
  const double threshold = ora_detection_rho() * (double)s->rc.eta;
  const uint64_t ncol = (uint64_t)1 << s->rc.q;
  uint64_t off = 0;
  for (uint32_t row = 0; row < s->rc.r; ++row) {
    row_counts[row] = 0;
    const uint16_t* p = s->rs + ((uint64_t)row << s->rc.q) * s->rc.eta;
    for (uint64_t col = 0; col < ncol; ++col, p += s->rc.eta) {
      const uint64_t w = counters_weight(p, s->rc.eta, k);
      if ((double)w >= threshold) {
        if (off < cap) cols[off] = (uint32_t)col;
        ++off;
        row_counts[row]++;
      }
    }
  }
  if (off > cap) return fail(SRLG_ERR_RESOURCE, "hot list buffer too small");
  return SRLG_OK;
}

/* make_estimate_context (src/slea.cpp:85-95) with setting_factor
 * (src/slea.cpp:57-61) */
int ora_estimate_context(const ora_sketch* s, uint32_t k, double* factors, double* sfp) {
  double prod = 1.0;
  for (uint32_t i = 0; i < s->sc.r; ++i) {
    const uint64_t w = counters_weight(s->le + (uint64_t)i * s->row_len, s->row_len, k);
    factors[i] = (double)w / (double)s->row_len;
    prod *= factors[i];
  }
  *sfp = prod;
  return SRLG_OK;
}

/* Slea::estimate (src/slea.cpp:97-125) */
static int estimate_with(const ora_sketch* s, uint32_t aip, uint32_t k, double sfp,
                         srlg_estimate* out) {
  if (sfp >= 1.0 - 1e-9) /* kSaturationEps (linear_counting.hpp:8) */
    return fail(SRLG_ERR_SATURATION, "slea estimate: array saturated, setting-factor product ~ 1");
  const uint16_t* rows[SRLG_MAX_ROWS];
  for (uint32_t i = 0; i < s->sc.r; ++i)
    rows[i] = s->le + (uint64_t)i * s->row_len + (uint64_t)ora_lh_column(s, i, aip) * s->sc.delta;
  const uint16_t kk = (uint16_t)(k > NEVER ? NEVER : k);
  uint64_t w = 0;
  for (uint32_t z = 0; z < s->sc.eta; ++z) {
    uint16_t m = 0;
    for (uint32_t i = 0; i < s->sc.r; ++i)
      if (rows[i][z] > m) m = rows[i][z];
    w += m < kk;
  }
  memset(out, 0, sizeof *out);
  out->usle_weight = w;
  out->sf_product = sfp;
  int st = ora_corrected_weight((double)w, sfp, s->sc.eta, &out->corrected_weight);
  if (st) return st;
  int sat = 0;
  ora_le_estimate(out->corrected_weight, s->sc.eta, &out->value, &sat);
  out->saturated = (uint32_t)sat;
  return SRLG_OK;
}

int ora_estimate(const ora_sketch* s, uint32_t aip, uint32_t k, srlg_estimate* out) {
  double f[SRLG_MAX_ROWS], sfp;
  ora_estimate_context(s, k, f, &sfp);
  return estimate_with(s, aip, k, sfp, out);
}

/* ---------------------------------------------------------- detection --- */

typedef struct blobbuf {
  uint8_t* b;
  uint64_t n, cap;
  uint64_t count;
} blobbuf;

static void blob_put(blobbuf* o, const void* p, uint64_t n) {
  if (o->n + n > o->cap) {
    o->cap = (o->n + n) * 2 + 256;
    o->b = (uint8_t*)realloc(o->b, o->cap);
  }
  memcpy(o->b + o->n, p, n);
  o->n += n;
}

typedef struct entry {
  uint32_t aip;
  uint32_t sat;
  double est;
} entry;

/* sort by estimate desc, then aip asc (src/window.cpp:72-76) */
static int cmp_entry(const void* a, const void* b) {
  const entry *x = (const entry*)a, *y = (const entry*)b;
  if (x->est != y->est) return x->est > y->est ? -1 : 1;
  return x->aip < y->aip ? -1 : x->aip > y->aip;
}

/* run_detection (src/window.cpp:36-78) -> one report blob */
static int detect_into(const ora_sketch* s, const srlg_window_config* wc, uint64_t window_end,
                       int partial, blobbuf* out) {
  const uint32_t r = s->rc.r;
  const uint64_t ncol = (uint64_t)1 << s->rc.q;
  uint32_t* cols = (uint32_t*)malloc(sizeof(uint32_t) * ncol * r);
  uint64_t counts[SRLG_MAX_ROWS];
  int st = ora_extract_hot(s, wc->k, cols, ncol * r, counts);
  if (st) {
    free(cols);
    return st;
  }
  uint32_t* hot[SRLG_MAX_ROWS];
  uint64_t off = 0;
  for (uint32_t i = 0; i < r; ++i) {
    hot[i] = cols + off;
    off += counts[i];
  }
  u32vec addrs = {0};
  int overflow = 0;
  uint64_t checked, kept;
  st = reconstruct(&s->g, hot, counts, wc->tuple_cap, (uint64_t)1 << 32, &addrs, &overflow,
                   &checked, &kept);
  free(cols);
  if (st) {
    free(addrs.v);
    return st;
  }
  double f[SRLG_MAX_ROWS], sfp;
  ora_estimate_context(s, wc->k, f, &sfp);

  srlg_report_header h;
  memset(&h, 0, sizeof h);
  h.window_end_slice = window_end;
  h.partial = (uint8_t)(partial != 0);
  h.overflow = (uint8_t)overflow;
  h.candidate_count = addrs.n;
  h.sf_product = sfp;
  h.n_rows = r;
  entry* es = NULL;
  uint64_t ne = 0;
  if (sfp >= 1.0 - 1e-9) {
    h.slea_saturated = 1;
  } else {
    es = (entry*)malloc(sizeof(entry) * (addrs.n + 1));
    const double theta = (double)wc->theta;
    for (uint64_t i = 0; i < addrs.n; ++i) {
      srlg_estimate e;
      st = estimate_with(s, addrs.v[i], wc->k, sfp, &e);
      if (st) {
        free(es);
        free(addrs.v);
        return st;
      }
      if (wc->keep_below_threshold || e.value >= theta) {
        es[ne].aip = addrs.v[i];
        es[ne].sat = e.saturated;
        es[ne].est = e.value;
        ++ne;
      }
    }
    qsort(es, ne, sizeof(entry), cmp_entry);
  }
  h.n_entries = (uint32_t)ne;
  blob_put(out, &h, sizeof h);
  blob_put(out, counts, 8 * r);
  for (uint64_t i = 0; i < ne; ++i) {
    srlg_entry x;
    memset(&x, 0, sizeof x);
    x.aip = es[i].aip;
    x.saturated = es[i].sat;
    x.estimate = es[i].est;
    blob_put(out, &x, sizeof x);
  }
  out->count++;
  free(es);
  free(addrs.v);
  return SRLG_OK;
}

int ora_detect(const ora_sketch* s, const srlg_window_config* wc, uint64_t window_end,
               int partial, uint8_t* blob, uint64_t cap, uint64_t* bytes) {
  blobbuf o = {0};
  int st = detect_into(s, wc, window_end, partial, &o);
  if (st == SRLG_OK) {
    *bytes = o.n;
    if (blob && o.n <= cap) memcpy(blob, o.b, o.n);
  }
  free(o.b);
  return st;
}

/* ------------------------------------------------------------- engine --- */

/* WindowConfig::validate (src/window.cpp:11-17) */
static int window_validate(const srlg_window_config* c) {
  if (c->slice_us == 0) return fail(SRLG_ERR_CONFIG, "slice duration must be positive");
  if (c->k == 0 || c->k > 65534) return fail(SRLG_ERR_CONFIG, "k must be in [1, 65534]");
  if (c->reinit_per_window && c->k != 1)
    return fail(SRLG_ERR_CONFIG, "reinit-per-window is the strict discrete mode and needs k = 1");
  if (c->workers == 0) return fail(SRLG_ERR_CONFIG, "workers must be at least 1");
  return SRLG_OK;
}

/* SliceClock (include/slidecard/window.hpp:34-52, src/window.cpp:19-34) */
typedef struct slice_clock {
  int has_t0, has_max;
  uint64_t t0, slice_us, tol, max_ts, clamped;
} slice_clock;

static int clock_place(slice_clock* c, uint64_t ts, uint64_t* slice) {
  if (!c->has_t0) {
    c->t0 = ts;
    c->has_t0 = 1;
  }
  if (c->has_max && ts < c->max_ts) {
    if (c->max_ts - ts > c->tol) return fail(SRLG_ERR_ORDERING, "timestamp regression beyond tolerance");
    c->clamped++;
    *slice = (c->max_ts - c->t0) / c->slice_us;
    return SRLG_OK;
  }
  if (!c->has_max || ts > c->max_ts) {
    c->max_ts = ts;
    c->has_max = 1;
  }
  if (ts < c->t0) return fail(SRLG_ERR_ORDERING, "timestamp precedes the stream start");
  *slice = (ts - c->t0) / c->slice_us;
  return SRLG_OK;
}

typedef struct pairvec {
  srlg_pair* v;
  uint64_t n, cap;
} pairvec;

static void pair_push(pairvec* a, uint32_t aip, uint32_t bip) {
  if (a->n == a->cap) {
    a->cap = a->cap ? a->cap * 2 : 1024;
    a->v = (srlg_pair*)realloc(a->v, a->cap * sizeof(srlg_pair));
  }
  a->v[a->n].aip = aip;
  a->v[a->n].bip = bip;
  a->n++;
}

struct ora_engine {
  srlg_window_config wc;
  ora_sketch* s;
  slice_clock clock;
  uint64_t current, records;
  int active;
  pairvec pending;
  blobbuf reports;
};

ora_engine* ora_engine_create(const srlg_rsra_config* rc, const srlg_slea_config* sc,
                              const srlg_window_config* wc) {
  if (window_validate(wc)) return NULL;
  ora_sketch* s = ora_sketch_create(rc, sc);
  if (!s) return NULL;
  ora_engine* e = (ora_engine*)calloc(1, sizeof *e);
  e->wc = *wc;
  e->s = s;
  e->clock.has_t0 = wc->has_t0 != 0;
  e->clock.t0 = wc->t0_us;
  e->clock.slice_us = wc->slice_us;
  e->clock.tol = wc->regression_tolerance_us;
  return e;
}

void ora_engine_destroy(ora_engine* e) {
  if (!e) return;
  ora_sketch_destroy(e->s);
  free(e->pending.v);
  free(e->reports.b);
  free(e);
}

/* flush_pending (src/window.cpp:89-98) */
static void engine_flush(ora_engine* e) {
  ora_update(e->s, e->pending.v, e->pending.n);
  e->pending.n = 0;
}

/* complete_slice (src/window.cpp:100-111) */
static int engine_complete(ora_engine* e) {
  if (e->current + 1 >= e->wc.k) {
    int st = detect_into(e->s, &e->wc, e->current, 0, &e->reports);
    if (st) return st;
  }
  if (e->wc.reinit_per_window) ora_reinit(e->s);
  else ora_slide(e->s);
  e->current++;
  return SRLG_OK;
}

/* process (src/window.cpp:122-131) */
static int engine_process_one(ora_engine* e, uint64_t ts, uint32_t aip, uint32_t bip) {
  uint64_t s;
  int st = clock_place(&e->clock, ts, &s);
  if (st) return st;
  e->active = 1;
  if (s > e->current) {
    engine_flush(e);
    while (e->current < s)
      if ((st = engine_complete(e))) return st;
  }
  pair_push(&e->pending, aip, bip);
  e->records++;
  return SRLG_OK;
}

int ora_engine_process(ora_engine* e, const srlg_record* recs, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    int st = engine_process_one(e, recs[i].ts_us, recs[i].aip, recs[i].bip);
    if (st) return st;
  }
  return SRLG_OK;
}

int ora_engine_process_slices(ora_engine* e, const srlg_pair* pairs, const uint64_t* offsets,
                              uint64_t n_slices, uint64_t first_slice) {
  if (!e->wc.has_t0) return fail(SRLG_ERR_CONFIG, "process_slices needs a configured t0");
  for (uint64_t s = 0; s < n_slices; ++s) {
    const uint64_t ts = e->wc.t0_us + (first_slice + s) * e->wc.slice_us;
    for (uint64_t i = offsets[s]; i < offsets[s + 1]; ++i) {
      int st = engine_process_one(e, ts, pairs[i].aip, pairs[i].bip);
      if (st) return st;
    }
  }
  return SRLG_OK;
}

/* advance_to_slice (src/window.cpp:113-120) */
int ora_engine_advance(ora_engine* e, uint64_t slice) {
  if (!e->active && !e->clock.has_max) {
    if (!e->wc.has_t0)
      return fail(SRLG_ERR_CONFIG, "cannot advance slices before the stream start is known");
    e->active = 1;
  }
  engine_flush(e);
  while (e->current < slice) {
    int st = engine_complete(e);
    if (st) return st;
  }
  return SRLG_OK;
}

/* finish (src/window.cpp:133-137) */
int ora_engine_finish(ora_engine* e) {
  if (!e->active) return SRLG_OK;
  engine_flush(e);
  return detect_into(e->s, &e->wc, e->current, 1, &e->reports);
}

uint64_t ora_engine_take_reports(ora_engine* e, uint8_t* blob, uint64_t cap,
                                 uint64_t* n_reports) {
  const uint64_t need = e->reports.n;
  if (n_reports) *n_reports = e->reports.count;
  if (blob && need <= cap) {
    memcpy(blob, e->reports.b, need);
    e->reports.n = 0;
    e->reports.count = 0;
  }
  return need;
}

uint64_t ora_engine_current_slice(const ora_engine* e) { return e->current; }

void ora_engine_export(const ora_engine* e, uint16_t* rsra, uint16_t* slea) {
  ora_export(e->s, rsra, slea);
}

/* -------------------------------------------------------- distributed --- */

/* route (src/distributed.cpp:20-31) */
static uint32_t route(uint32_t aip, uint32_t bip, uint64_t index, uint32_t policy,
                      uint32_t nodes) {
  switch (policy) {
    case 0: return (uint32_t)(ora_hash64(((uint64_t)aip << 32) | bip, 0x70617274) % nodes);
    case 1: return (uint32_t)(index % nodes);
    case 2: return (aip >> 24) % nodes;
  }
  return 0;
}

/* run_distributed (src/distributed.cpp:35-117) */
int ora_run_distributed(const srlg_record* recs, uint64_t n, const srlg_rsra_config* rc,
                        const srlg_slea_config* sc, const srlg_window_config* wc,
                        uint32_t nodes, uint32_t policy, uint8_t* blob, uint64_t cap,
                        uint64_t* bytes, uint64_t* n_reports, uint64_t* slice_merges,
                        uint64_t* bytes_exchanged) {
  int st = window_validate(wc);
  if (st) return st;
  if (nodes == 0) return fail(SRLG_ERR_CONFIG, "distributed run needs at least one node");
  ora_sketch** node = (ora_sketch**)calloc(nodes, sizeof(ora_sketch*));
  pairvec* pend = (pairvec*)calloc(nodes, sizeof(pairvec));
  for (uint32_t i = 0; i < nodes; ++i) {
    node[i] = ora_sketch_create(rc, sc);
    if (!node[i]) {
      st = SRLG_ERR_CONFIG;
      goto done;
    }
  }
  blobbuf out = {0};
  slice_clock clock = {0};
  clock.has_t0 = wc->has_t0 != 0;
  clock.t0 = wc->t0_us;
  clock.slice_us = wc->slice_us;
  clock.tol = wc->regression_tolerance_us;
  uint64_t current = 0, index = 0, merges = 0, exchanged = 0;
  int active = 0;
  const uint64_t rs_bytes = 4 + 2 + 1 + 5 * 4 + 3 * 8 + 8 + 2 * node[0]->rs_n; /* sketch_io.cpp:136-142 */
  const uint64_t le_bytes = 4 + 2 + 1 + 4 * 4 + (1 + (uint64_t)sc->r) * 8 + 8 + 2 * node[0]->le_n;

#define FLUSH_ALL()                                          \
  for (uint32_t i = 0; i < nodes; ++i) {                     \
    ora_update(node[i], pend[i].v, pend[i].n);               \
    pend[i].n = 0;                                           \
  }
#define MERGED_DETECT(END, PARTIAL)                                     \
  do {                                                                  \
    ora_sketch* g = ora_sketch_clone(node[0]);                          \
    for (uint32_t i = 1; i < nodes; ++i) ora_merge_min(g, node[i]);     \
    merges++;                                                           \
    exchanged += nodes * (rs_bytes + le_bytes);                         \
    st = detect_into(g, wc, (END), (PARTIAL), &out);                    \
    ora_sketch_destroy(g);                                              \
  } while (0)

  for (uint64_t j = 0; j < n && st == SRLG_OK; ++j) {
    uint64_t s;
    if ((st = clock_place(&clock, recs[j].ts_us, &s))) break;
    active = 1;
    if (s > current) {
      FLUSH_ALL();
      while (current < s && st == SRLG_OK) {
        if (current + 1 >= wc->k) MERGED_DETECT(current, 0);
        for (uint32_t i = 0; i < nodes; ++i) {
          if (wc->reinit_per_window) ora_reinit(node[i]);
          else ora_slide(node[i]);
        }
        ++current;
      }
    }
    const uint32_t to = route(recs[j].aip, recs[j].bip, index, policy, nodes);
    pair_push(&pend[to], recs[j].aip, recs[j].bip);
    ++index;
  }
  if (st == SRLG_OK && active) {
    FLUSH_ALL();
    MERGED_DETECT(current, 1);
  }
#undef FLUSH_ALL
#undef MERGED_DETECT
  if (st == SRLG_OK) {
    *bytes = out.n;
    *n_reports = out.count;
    *slice_merges = merges;
    *bytes_exchanged = exchanged;
    if (blob && out.n <= cap) memcpy(blob, out.b, out.n);
  }
  free(out.b);
done:
  for (uint32_t i = 0; i < nodes; ++i) {
    ora_sketch_destroy(node[i]);
    free(pend[i].v);
  }
  free(node);
  free(pend);
  return st;
}

/* Rng (include/slidecard/rng.hpp:11-32): pair i = (next_u32(), next_u32()) */
void ora_rng_pairs(uint64_t seed, uint64_t n, srlg_pair* out) {
  uint64_t state = ora_mix64(seed);
  for (uint64_t i = 0; i < n; ++i) {
    state += kGolden64;
    out[i].aip = (uint32_t)(ora_mix64(state) >> 32);
    state += kGolden64;
    out[i].bip = (uint32_t)(ora_mix64(state) >> 32);
  }
}

/* FNV-1a 64 over the little-endian bytes of a u16 array */
uint64_t ora_fnv1a64_u16(const uint16_t* v, uint64_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= (uint8_t)(v[i] & 0xFF);
    h *= 0x100000001b3ULL;
    h ^= (uint8_t)(v[i] >> 8);
    h *= 0x100000001b3ULL;
  }
  return h;
}
