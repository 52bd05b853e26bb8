/*
 * tt_oracle.c — plain-C restatement of the reference draft+verify path.
 *
 * TEST INFRASTRUCTURE ONLY (see tt_oracle.h). Written from the reference's
 * published behaviour, one function per reference function, each citing the
 * file:line it restates (paths relative to /root/reference/proj). It is
 * deliberately literal — per-statement symbol sets, per-statement penalties,
 * the reference's own accumulation order — so that it is easy to audit
 * against the reference; the CUDA kernels are the flattened/hoisted form.
 *
 * Built with -O2 -ffp-contract=off (oracle/Makefile) so no FMA contraction
 * changes rounding relative to the reference build.
 */
#include "tt_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9e3779b97f4a7c15ULL

/* ---------------- RNG: core/include/tiletune/common.hpp:52-119 ---------------- */

static uint64_t scramble64(uint64_t x) { /* common.hpp:59-63 */
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
static uint64_t mix64(uint64_t x) { return scramble64(x + GOLDEN); } /* common.hpp:52-57 */

uint64_t tto_derive_seed(uint64_t base, uint64_t a) { return mix64(base ^ mix64(a)); }

uint64_t tto_hash_str(const char* s) { /* common.hpp:74-82, FNV-1a */
  uint64_t h = 1469598103934665603ULL;
  for (; *s; ++s) {
    h ^= (unsigned char)*s;
    h *= 1099511628211ULL;
  }
  return h;
}

typedef struct {
  uint64_t state;
} rng_t;

static void rng_init(rng_t* r, uint64_t seed) { r->state = seed ? seed : GOLDEN; } /* :91 */
static uint64_t rng_next(rng_t* r) {                                                 /* :93-97 */
  r->state += GOLDEN;
  return scramble64(r->state);
}
static uint64_t rng_index(rng_t* r, uint64_t n) { /* :100-102 */
  return (uint64_t)(((unsigned __int128)rng_next(r) * n) >> 64);
}
static double rng_real(rng_t* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; } /* :105 */

/* ---------------- factorization: core/src/schedule.cpp:25-148 ---------------- */

typedef struct {
  int64_t p[16];
  int e[16];
  int n;
} primes_t;

static void prime_factorize(int64_t n, primes_t* out) { /* schedule.cpp:90-105 */
  out->n = 0;
  for (int64_t p = 2; p * p <= n; ++p) {
    if (n % p == 0) {
      int e = 0;
      while (n % p == 0) {
        n /= p;
        ++e;
      }
      out->p[out->n] = p;
      out->e[out->n] = e;
      out->n++;
    }
  }
  if (n > 1) {
    out->p[out->n] = n;
    out->e[out->n] = 1;
    out->n++;
  }
}

static uint64_t binomial(int64_t n, int64_t k) { /* schedule.cpp:36-45 */
  if (k < 0 || k > n) return 0;
  if (n - k < k) k = n - k;
  unsigned __int128 r = 1;
  for (int64_t i = 1; i <= k; ++i) {
    r = r * (unsigned __int128)(n - k + i) / (unsigned __int128)i;
    if (r > (unsigned __int128)UINT64_MAX) return UINT64_MAX;
  }
  return (uint64_t)r;
}

static uint64_t sat_mul(uint64_t a, uint64_t b) { /* schedule.cpp:29-33 */
  if (a == 0 || b == 0) return 0;
  if (a > UINT64_MAX / b) return UINT64_MAX;
  return a * b;
}

/* unrank: the loop body of sample_composition (schedule.cpp:49-68) */
static void unrank_composition(int total, int k, uint64_t rank, int* parts) {
  int remaining = total;
  for (int slot = 0; slot < k - 1; ++slot) {
    int slots_left = k - slot - 1;
    parts[slot] = 0;
    for (int v = 0; v <= remaining; ++v) {
      uint64_t with_v = binomial(remaining - v + slots_left - 1, slots_left - 1);
      if (rank < with_v) {
        parts[slot] = v;
        remaining -= v;
        break;
      }
      rank -= with_v;
    }
  }
  parts[k - 1] = remaining;
}

/* inverse of unrank_composition */
static uint64_t rank_composition(int total, int k, const int* parts) {
  uint64_t rank = 0;
  int remaining = total;
  for (int slot = 0; slot < k - 1; ++slot) {
    int slots_left = k - slot - 1;
    for (int v = 0; v < parts[slot]; ++v)
      rank += binomial(remaining - v + slots_left - 1, slots_left - 1);
    remaining -= parts[slot];
  }
  return rank;
}

static int64_t ipow(int64_t b, int e) {
  int64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}

static int slot_arity(const tt_sketch* sk, int axis) {
  if (axis >= sk->op.n_spatial) return 3;
  return sk->op.kind == TT_OP_ELEMENTWISE ? 2 : 4;
}

void tto_sketch_init(const tt_op_spec* op, tt_sketch* out) { /* schedule.cpp:150-164 */
  memset(out, 0, sizeof(*out));
  out->op = *op;
  out->n_unroll = 3;
  out->unroll[0] = 1;
  out->unroll[1] = 4;
  out->unroll[2] = 16;
}

int tto_draws_per_schedule(const tt_sketch* sk) {
  int d = 1;
  int na = sk->op.n_spatial + sk->op.n_reduction;
  for (int a = 0; a < na; ++a) {
    primes_t pr;
    prime_factorize(sk->op.extent[a], &pr);
    d += pr.n;
  }
  return d;
}

uint64_t tto_space_size(const tt_sketch* sk) { /* schedule.cpp:188-195 */
  uint64_t size = 1;
  int na = sk->op.n_spatial + sk->op.n_reduction;
  for (int a = 0; a < na; ++a) {
    primes_t pr;
    prime_factorize(sk->op.extent[a], &pr);
    int k = slot_arity(sk, a);
    uint64_t c = 1;
    for (int j = 0; j < pr.n; ++j) c = sat_mul(c, binomial(pr.e[j] + k - 1, k - 1));
    size = sat_mul(size, c);
  }
  return sat_mul(size, (uint64_t)sk->n_unroll);
}

static int axis_col(const tt_sketch* sk, int axis) {
  return axis < sk->op.n_spatial ? 4 * axis : 4 * sk->op.n_spatial + 3 * (axis - sk->op.n_spatial);
}

/* random_init (schedule.cpp:166-186) with sample_factorization (:141-148).
 * Schedule j starts at draw j*D of the stream because every schedule
 * consumes exactly D draws; the offset is applied directly to the
 * splitmix64 counter. */
void tto_random_init(const tt_sketch* sk, uint64_t seed, int64_t first, int64_t n,
                     int32_t* soa, int64_t ld) {
  rng_t rng;
  rng_init(&rng, seed);
  rng.state += (uint64_t)first * (uint64_t)tto_draws_per_schedule(sk) * GOLDEN;
  int na = sk->op.n_spatial + sk->op.n_reduction;
  int ucol = tt_schedule_cols(sk) - 1;
  for (int64_t i = 0; i < n; ++i) {
    for (int a = 0; a < na; ++a) {
      int k = slot_arity(sk, a);
      int64_t tuple[4] = {1, 1, 1, 1};
      primes_t pr;
      prime_factorize(sk->op.extent[a], &pr);
      for (int j = 0; j < pr.n; ++j) {
        uint64_t count = binomial(pr.e[j] + k - 1, k - 1);
        uint64_t rank = rng_index(&rng, count);
        int parts[4];
        unrank_composition(pr.e[j], k, rank, parts);
        for (int q = 0; q < k; ++q) tuple[q] *= ipow(pr.p[j], parts[q]);
      }
      int c = axis_col(sk, a);
      int width = a < sk->op.n_spatial ? 4 : 3; /* arity-2 slots pad (b,t,1,1) */
      for (int q = 0; q < width; ++q) soa[(int64_t)(c + q) * ld + i] = (int32_t)tuple[q];
    }
    soa[(int64_t)ucol * ld + i] = (int32_t)sk->unroll[rng_index(&rng, (uint64_t)sk->n_unroll)];
  }
}

uint64_t tto_identity(const tt_sketch* sk, const int32_t* soa, int64_t ld, int64_t i, int* ok) {
  *ok = tto_space_size(sk) != UINT64_MAX;
  if (!*ok) return 0;
  uint64_t id = 0;
  int na = sk->op.n_spatial + sk->op.n_reduction;
  for (int a = 0; a < na; ++a) {
    int k = slot_arity(sk, a);
    int c = axis_col(sk, a);
    primes_t pr;
    prime_factorize(sk->op.extent[a], &pr);
    for (int j = 0; j < pr.n; ++j) {
      int parts[4] = {0, 0, 0, 0};
      for (int q = 0; q < k; ++q) {
        int64_t f = soa[(int64_t)(c + q) * ld + i];
        while (f % pr.p[j] == 0) {
          f /= pr.p[j];
          parts[q]++;
        }
      }
      uint64_t count = binomial(pr.e[j] + k - 1, k - 1);
      id = id * count + rank_composition(pr.e[j], k, parts);
    }
  }
  int64_t u = soa[(int64_t)(tt_schedule_cols(sk) - 1) * ld + i];
  int ui = 0;
  for (int q = 0; q < sk->n_unroll; ++q)
    if (sk->unroll[q] == u) ui = q;
  return id * (uint64_t)sk->n_unroll + (uint64_t)ui;
}

/* ---------------- tile table: core/src/tiles_internal.hpp:33-108 ---------------- */

typedef struct {
  int64_t extent, l0, l1, v_inner;
} axis_tiles_t;

typedef struct {
  axis_tiles_t ax[TT_MAX_AXES];
  int64_t lanes_per_block; /* s4 */
  int64_t blocks;          /* s6 */
  int64_t prod_ra;
  int64_t reduction_total;
} tiles_t;

static void build_tiles(const tt_sketch* sk, const int32_t* soa, int64_t ld, int64_t i,
                        tiles_t* t) { /* tiles_internal.hpp:80-108 */
  const tt_op_spec* op = &sk->op;
  t->lanes_per_block = 1;
  t->blocks = 1;
  t->prod_ra = 1;
  t->reduction_total = 1;
  for (int a = 0; a < op->n_spatial; ++a) {
    int64_t b = soa[(int64_t)(4 * a) * ld + i], th = soa[(int64_t)(4 * a + 1) * ld + i];
    int64_t o = soa[(int64_t)(4 * a + 2) * ld + i], v = soa[(int64_t)(4 * a + 3) * ld + i];
    t->ax[a].extent = op->extent[a];
    t->ax[a].l0 = o * v;
    t->ax[a].l1 = th * o * v;
    t->ax[a].v_inner = v;
    t->lanes_per_block *= th;
    t->blocks *= b;
  }
  for (int r = 0; r < op->n_reduction; ++r) {
    int a = op->n_spatial + r;
    int c = 4 * op->n_spatial + 3 * r;
    int64_t ra = soa[(int64_t)c * ld + i], rb = soa[(int64_t)(c + 1) * ld + i];
    int64_t rc = soa[(int64_t)(c + 2) * ld + i];
    t->ax[a].extent = op->extent[a];
    t->ax[a].l0 = 1;
    t->ax[a].l1 = rb * rc;
    t->ax[a].v_inner = rc;
    t->prod_ra *= ra;
    t->reduction_total *= op->extent[a];
  }
}

static int64_t tile_extent(const tiles_t* t, int axis, int level) { /* :52-63 */
  return level == 0 ? t->ax[axis].l0 : level == 1 ? t->ax[axis].l1 : t->ax[axis].extent;
}

static int64_t footprint(const tiles_t* t, const tt_buffer_spec* b, int level) { /* :65-69 */
  int64_t fp = 1;
  for (int q = 0; q < b->n_axes; ++q) fp *= tile_extent(t, b->axes[q], level);
  return fp;
}

static int64_t inner_vector(const tiles_t* t, const tt_buffer_spec* b) { /* :71-75 */
  int64_t v = 1;
  for (int q = 0; q < b->n_axes; ++q) v *= t->ax[b->axes[q]].v_inner;
  return v;
}

static const tt_buffer_spec* output_buffer(const tt_op_spec* op) { /* workload.cpp:29-33 */
  for (int b = 0; b < op->n_buffers; ++b)
    if (op->buffers[b].io == TT_IO_OUTPUT) return &op->buffers[b];
  return &op->buffers[0];
}

static int64_t flops_of(const tt_op_spec* op) { /* workload.cpp:197-203 */
  int64_t total = 1;
  for (int a = 0; a < op->n_spatial; ++a) total *= op->extent[a];
  if (op->kind == TT_OP_TILED)
    for (int r = 0; r < op->n_reduction; ++r) total *= op->extent[op->n_spatial + r];
  return total;
}

/* ---------------- SA draft model: core/src/draft.cpp:42-154 ---------------- */

enum { K_L2L1 = 0, K_L1L0 = 1, K_COMPUTE = 2, K_STORE = 3 };

typedef struct {
  int kind;
  int buffer;
  int64_t s[8]; /* s1..s8 */
} stmt_sym_t;

static int extract_symbols(const tt_sketch* sk, const tiles_t* t, stmt_sym_t* out) {
  const tt_op_spec* op = &sk->op; /* draft.cpp:42-106 */
  const tt_buffer_spec* outb = output_buffer(op);
  int64_t s1 = footprint(t, outb, 0), s3 = 0;
  for (int b = 0; b < op->n_buffers; ++b)
    if (op->buffers[b].io == TT_IO_INPUT) {
      s1 += footprint(t, &op->buffers[b], 0);
      s3 += footprint(t, &op->buffers[b], 1);
    }
  int64_t s2 = t->reduction_total;
  for (int a = 0; a < op->n_spatial; ++a) s2 *= t->ax[a].l0;
  int64_t s4 = t->lanes_per_block, s6 = t->blocks;
  int64_t output_size = 1;
  for (int a = 0; a < op->n_spatial; ++a) output_size *= op->extent[a];

  int n = 0;
#define BASE(k, bi)                                                        \
  do {                                                                     \
    memset(&out[n], 0, sizeof(out[n]));                                    \
    out[n].kind = (k);                                                     \
    out[n].buffer = (bi);                                                  \
    out[n].s[0] = s1;                                                      \
    out[n].s[1] = s2;                                                      \
    out[n].s[2] = s3;                                                      \
    out[n].s[3] = s4;                                                      \
    out[n].s[5] = s6;                                                      \
  } while (0)
  for (int b = 0; b < op->n_buffers; ++b) {
    const tt_buffer_spec* buf = &op->buffers[b];
    if (buf->io != TT_IO_INPUT) continue;
    BASE(K_L2L1, b);
    out[n].s[4] = footprint(t, buf, 1) * s6 * t->prod_ra;
    out[n].s[6] = tile_extent(t, buf->axes[buf->n_axes - 1], 1);
    ++n;
  }
  for (int b = 0; b < op->n_buffers; ++b) {
    const tt_buffer_spec* buf = &op->buffers[b];
    if (buf->io != TT_IO_INPUT) continue;
    BASE(K_L1L0, b);
    out[n].s[6] = tile_extent(t, buf->axes[buf->n_axes - 1], 0);
    ++n;
  }
  BASE(K_COMPUTE, -1);
  out[n].s[7] = flops_of(op);
  ++n;
  int index = 0;
  for (int b = 0; b < op->n_buffers; ++b)
    if (op->buffers[b].io == TT_IO_OUTPUT) index = b;
  BASE(K_STORE, index);
  out[n].s[4] = output_size;
  out[n].s[6] = tile_extent(t, outb->axes[outb->n_axes - 1], 0);
  ++n;
#undef BASE
  return n;
}

typedef struct {
  double p_l0_m, p_l0_c, p_l1_m, p_l1_c, alpha_l1, p_l2_c, p_l2_m;
} penalty_t;

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static penalty_t compute_penalties(const int64_t* s, const tt_device_spec* d) {
  penalty_t p = {1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 1.0}; /* draft.cpp:108-127 */
  if (s[0] > 0) {
    double x = (double)d->m_l0 / (double)s[0];
    p.p_l0_m = x < 1.0 ? x : 1.0;
    p.p_l0_c = 1.0 + (double)s[1] / (double)s[0];
  }
  if (s[2] > 0) {
    double x = (double)d->m_l1 / (double)s[2];
    p.p_l1_m = x < 1.0 ? x : 1.0;
  }
  int64_t sch = ceil_div(s[3], d->n_l1);
  p.p_l1_c = (double)sch / (double)(ceil_div(sch, d->pu_l1) * d->pu_l1);
  p.alpha_l1 = (double)s[3] / (double)(sch * d->n_l1);
  p.p_l2_c = (double)s[5] / (double)(ceil_div(s[5], d->pu_l2) * d->pu_l2);
  if (s[6] > 0) p.p_l2_m = (double)s[6] / (double)(ceil_div(s[6], d->n_l2) * d->n_l2);
  return p;
}

int tto_trace(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
              int64_t i, int toggles, int64_t* symbols, double* penalties, double* stmt_cost,
              double* total) {
  tiles_t t;
  stmt_sym_t st[2 * TT_MAX_BUFFERS + 2];
  build_tiles(sk, soa, ld, i, &t);
  int n = extract_symbols(sk, &t, st);
  double tot = 0.0; /* draft.cpp:129-154 */
  for (int s = 0; s < n; ++s) {
    penalty_t p = compute_penalties(st[s].s, dev);
    if (!(toggles & TT_TOGGLE_COMPUTE)) p.p_l0_c = p.p_l1_c = p.alpha_l1 = p.p_l2_c = 1.0;
    if (!(toggles & TT_TOGGLE_MEMORY)) p.p_l0_m = p.p_l1_m = p.p_l2_m = 1.0;
    double u_p = dev->t_p * p.p_l0_c * p.p_l1_c * p.alpha_l1 * p.p_l2_c;
    double u_m = dev->t_m * p.p_l0_m * p.p_l1_m * p.p_l2_m;
    double l_c = st[s].s[7] > 0 ? (double)st[s].s[7] / u_p : 0.0;
    double l_m = st[s].s[4] > 0 ? (double)st[s].s[4] / u_m : 0.0;
    tot += l_c + l_m;
    if (symbols)
      for (int q = 0; q < 8; ++q) symbols[s * 8 + q] = st[s].s[q];
    if (penalties) {
      double* pp = penalties + s * 7;
      pp[0] = p.p_l0_m, pp[1] = p.p_l0_c, pp[2] = p.p_l1_m, pp[3] = p.p_l1_c;
      pp[4] = p.alpha_l1, pp[5] = p.p_l2_c, pp[6] = p.p_l2_m;
    }
    if (stmt_cost) {
      double* c = stmt_cost + s * 4;
      c[0] = l_c, c[1] = l_m, c[2] = u_p, c[3] = u_m;
    }
  }
  if (total) *total = tot;
  return n;
}

void tto_draft_cost(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa,
                    int64_t ld, int64_t n, int toggles, double* cost) {
  for (int64_t i = 0; i < n; ++i) tto_trace(sk, dev, soa, ld, i, toggles, 0, 0, 0, &cost[i]);
}

/* ---------------- PriorFilter (explore, n_steps = 1): draft.cpp:156-221 ---------------- */

typedef struct {
  double cost;
  int64_t idx;
} cand_t;

static int cand_cmp(const void* a, const void* b) {
  const cand_t* x = (const cand_t*)a;
  const cand_t* y = (const cand_t*)b;
  if (x->cost != y->cost) return x->cost < y->cost ? -1 : 1;
  return (x->idx > y->idx) - (x->idx < y->idx);
}

static int same_schedule(const tt_sketch* sk, const int32_t* soa, int64_t ld, int64_t i,
                         int64_t j) {
  int cols = tt_schedule_cols(sk);
  for (int c = 0; c < cols; ++c)
    if (soa[(int64_t)c * ld + i] != soa[(int64_t)c * ld + j]) return 0;
  return 1;
}

int64_t tto_draft_topk(const tt_sketch* sk, const double* cost, const int32_t* soa, int64_t ld,
                       int64_t n, int64_t k, int64_t* idx_out, double* cost_out) {
  /* The pool keeps the first occurrence of every key (draft.cpp:200-203),
   * trim/sort order by (cost, discovery) (draft.cpp:174-191,209-214): i.e.
   * the K lowest unique schedules by (cost, first index). Identical
   * schedules have identical costs, so duplicates sit in one equal-cost
   * run of the (cost, index) order. */
  cand_t* c = (cand_t*)malloc(sizeof(cand_t) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) c[i].cost = cost[i], c[i].idx = i;
  qsort(c, (size_t)n, sizeof(cand_t), cand_cmp);
  int64_t kept = 0;
  int64_t run_start = 0, run_kept_start = 0;
  for (int64_t e = 0; e < n && kept < k; ++e) {
    if (e == 0 || c[e].cost != c[e - 1].cost) run_start = e, run_kept_start = kept;
    (void)run_start;
    int dup = 0;
    for (int64_t q = run_kept_start; q < kept && !dup; ++q)
      dup = same_schedule(sk, soa, ld, idx_out[q], c[e].idx);
    if (dup) continue;
    idx_out[kept] = c[e].idx;
    if (cost_out) cost_out[kept] = c[e].cost;
    ++kept;
  }
  free(c);
  return kept;
}

/* ---------------- hybrid features: core/src/features.cpp:36-257 ---------------- */

static double lg(double x) { return log1p(x); } /* features.cpp:52-53 */

enum { F_L2L1 = 0, F_L1L0, F_L0C, F_L0L2, F_L1L2, F_INTRA };
enum { A_READ = 0, A_WRITE, A_RW };

typedef struct {
  int flow, access;
  int64_t alloc, volume, distinct, stride;
  int contiguous;
  int64_t per_lane;
  int rank, depth, red_carried;
} block_args_t;

static void make_block(const block_args_t* a, int64_t flops, int64_t lanes, int64_t unroll,
                       int64_t s7, double* f) { /* features.cpp:74-94 */
  memset(f, 0, sizeof(double) * TT_BLOCK_WIDTH);
  f[0 + a->flow] = 1.0;
  f[6 + a->access] = 1.0;
  f[9] = lg((double)a->alloc);
  f[10] = lg((double)a->volume);
  f[11] = lg((double)a->volume / (double)(a->distinct > 1 ? a->distinct : 1));
  f[12] = lg((double)a->stride);
  f[13] = a->contiguous ? 1.0 : 0.0;
  f[14] = lg((double)flops / (double)(a->volume > 1 ? a->volume : 1));
  f[15] = lg((double)lanes);
  f[16] = lg((double)a->per_lane);
  f[17] = a->rank / 8.0;
  f[18] = a->depth / 16.0;
  f[19] = a->red_carried ? 1.0 : 0.0;
  f[20] = lg((double)unroll);
  f[21] = lg((double)s7);
  f[22] = 1.0;
}

static int has_reduction_axis(const tt_op_spec* op, const tt_buffer_spec* b) {
  for (int q = 0; q < b->n_axes; ++q)
    if (b->axes[q] >= op->n_spatial) return 1;
  return 0;
}

static int64_t buffer_size(const tt_op_spec* op, const tt_buffer_spec* b) {
  int64_t s = 1;
  for (int q = 0; q < b->n_axes; ++q) s *= op->extent[b->axes[q]];
  return s;
}

static void features_one(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa,
                         int64_t ld, int64_t i, double* sf, double* bf) {
  const tt_op_spec* op = &sk->op;
  tiles_t t;
  stmt_sym_t st[2 * TT_MAX_BUFFERS + 2];
  build_tiles(sk, soa, ld, i, &t);
  int ns = extract_symbols(sk, &t, st);
  int64_t flops = flops_of(op);
  int64_t unroll = soa[(int64_t)(tt_schedule_cols(sk) - 1) * ld + i];
  int64_t traffic = 0;
  for (int s = 0; s < ns; ++s) traffic += st[s].s[4];

  for (int s = 0; s < ns; ++s) { /* features.cpp:122-151 */
    const int64_t* y = st[s].s;
    penalty_t p = compute_penalties(y, dev);
    double* f = sf + s * TT_STMT_WIDTH;
    for (int q = 0; q < 8; ++q) f[q] = lg((double)y[q]);
    f[8] = p.p_l0_m;
    f[9] = lg(p.p_l0_c);
    f[10] = p.p_l1_m;
    f[11] = p.p_l1_c;
    f[12] = p.alpha_l1;
    f[13] = p.p_l2_c;
    f[14] = p.p_l2_m;
    f[15] = lg((double)flops);
    f[16] = lg((double)traffic);
    f[17] = lg((double)y[7] / (double)(y[4] > 1 ? y[4] : 1));
    f[18] = (double)y[3] / (double)(dev->pu_l1 * dev->n_l1);
    f[19] = lg((double)y[5] / (double)dev->pu_l2);
    f[20] = lg((double)unroll);
    f[21] = (double)op->fused_elementwise;
    f[22] = st[s].kind / 4.0;
    f[23] = 1.0;
  }

  if (op->kind == TT_OP_ELEMENTWISE) { /* features.cpp:153-158 */
    memset(bf, 0, sizeof(double) * TT_BLOCK_WIDTH);
    bf[22] = 1.0;
    return;
  }

  int64_t lanes = t.lanes_per_block * t.blocks;
  int64_t output_size = 1;
  for (int a = 0; a < op->n_spatial; ++a) output_size *= op->extent[a];
  const tt_buffer_spec* outb = output_buffer(op);
  int innermost_spatial = op->n_spatial - 1;
  int n_sp = op->n_spatial, n_red = op->n_reduction;
  int nb = 0;
#define REG_STRIDE(buf) \
  ((buf)->axes[(buf)->n_axes - 1] == innermost_spatial ? 1 : tile_extent(&t, (buf)->axes[(buf)->n_axes - 1], 1))

  for (int s = 0; s < ns; ++s) { /* features.cpp:180-255 */
    const int64_t* y = st[s].s;
    block_args_t a;
    memset(&a, 0, sizeof(a));
    if (st[s].kind == K_L2L1) {
      const tt_buffer_spec* buf = &op->buffers[st[s].buffer];
      a.flow = F_L2L1, a.access = A_READ;
      a.alloc = footprint(&t, buf, 1);
      a.volume = y[4];
      a.distinct = buffer_size(op, buf);
      a.stride = 1;
      a.contiguous = y[6] % dev->n_l2 == 0;
      a.per_lane = (a.alloc + t.lanes_per_block - 1) / t.lanes_per_block;
      a.rank = buf->n_axes;
      a.depth = n_sp + n_red;
      a.red_carried = has_reduction_axis(op, buf);
      make_block(&a, flops, lanes, unroll, y[6], bf + (nb++) * TT_BLOCK_WIDTH);
    } else if (st[s].kind == K_L1L0) {
      const tt_buffer_spec* buf = &op->buffers[st[s].buffer];
      a.flow = F_L1L0, a.access = A_READ;
      a.alloc = footprint(&t, buf, 0);
      a.volume = lanes * t.reduction_total * a.alloc;
      a.distinct = buffer_size(op, buf);
      a.stride = REG_STRIDE(buf);
      a.contiguous = a.stride == 1;
      a.per_lane = inner_vector(&t, buf);
      a.rank = buf->n_axes;
      a.depth = 2 * (n_sp + n_red);
      a.red_carried = has_reduction_axis(op, buf);
      make_block(&a, flops, lanes, unroll, y[6], bf + (nb++) * TT_BLOCK_WIDTH);
    } else if (st[s].kind == K_COMPUTE) {
      for (int b = 0; b < op->n_buffers; ++b) {
        const tt_buffer_spec* buf = &op->buffers[b];
        if (buf->io != TT_IO_INPUT) continue;
        memset(&a, 0, sizeof(a));
        a.flow = F_L0C, a.access = A_READ;
        a.alloc = footprint(&t, buf, 0);
        a.volume = flops;
        a.distinct = buffer_size(op, buf);
        a.stride = REG_STRIDE(buf);
        a.contiguous = a.stride == 1;
        a.per_lane = inner_vector(&t, buf);
        a.rank = buf->n_axes;
        a.depth = 2 * (n_sp + n_red) + n_red + 2 * n_sp;
        a.red_carried = has_reduction_axis(op, buf);
        make_block(&a, flops, lanes, unroll, y[6], bf + (nb++) * TT_BLOCK_WIDTH);
      }
      memset(&a, 0, sizeof(a));
      a.flow = F_INTRA, a.access = A_RW;
      a.alloc = footprint(&t, outb, 0);
      a.volume = flops;
      a.distinct = output_size;
      a.stride = 1;
      a.contiguous = 1;
      a.per_lane = inner_vector(&t, outb);
      a.rank = outb->n_axes;
      a.depth = 2 * (n_sp + n_red) + n_red + 2 * n_sp;
      a.red_carried = 1;
      make_block(&a, flops, lanes, unroll, y[6], bf + (nb++) * TT_BLOCK_WIDTH);
    } else {
      a.flow = F_L0L2, a.access = A_WRITE;
      a.alloc = output_size;
      a.volume = y[4];
      a.distinct = output_size;
      a.stride = 1;
      a.contiguous = y[6] % dev->n_l2 == 0;
      a.per_lane = footprint(&t, outb, 0);
      a.rank = outb->n_axes;
      a.depth = 4 * n_sp;
      a.red_carried = 0;
      make_block(&a, flops, lanes, unroll, y[6], bf + (nb++) * TT_BLOCK_WIDTH);
    }
  }
#undef REG_STRIDE
}

void tto_features(const tt_sketch* sk, const tt_device_spec* dev, const int32_t* soa, int64_t ld,
                  const int64_t* idx, int64_t k, double* stmt_out, double* block_out) {
  int S = tt_n_statements(&sk->op), B = tt_n_blocks(&sk->op);
  for (int64_t q = 0; q < k; ++q)
    features_one(sk, dev, soa, ld, idx[q], stmt_out + q * S * TT_STMT_WIDTH,
                 block_out + q * B * TT_BLOCK_WIDTH);
}

/* ---------------- PaCM: core/src/ranker.cpp:52-209,305-326 ---------------- */

void tto_init_params(int h, uint64_t seed, double* p) { /* ranker.cpp:305-326 */
  rng_t rng;
  rng_init(&rng, seed);
  int shapes[16][2] = {{24, h}, {1, h}, {h, h}, {1, h}, {23, h}, {1, h}, {h, h}, {1, h},
                       {h, h},  {1, h}, {h, h}, {1, h}, {2 * h, h}, {1, h}, {h, 1}, {1, 1}};
  for (int t = 0; t < 16; ++t) {
    int n = shapes[t][0] * shapes[t][1];
    if (t % 2 == 0) { /* xavier(rows, cols) (ranker.cpp:52-57) */
      double limit = sqrt(6.0 / (shapes[t][0] + shapes[t][1]));
      for (int e = 0; e < n; ++e) p[e] = (2.0 * rng_real(&rng) - 1.0) * limit;
    } else {
      for (int e = 0; e < n; ++e) p[e] = 0.0;
    }
    p += n;
  }
}

/* y (n x p) = act(x (n x m) * w (m x p) + b), ranker.cpp:59-75 */
static void affine(const double* x, int n, int m, const double* w, const double* b, int p,
                   int act, double* y) {
  for (int i = 0; i < n; ++i) {
    double* yr = y + i * p;
    for (int j = 0; j < p; ++j) yr[j] = 0.0;
    for (int k = 0; k < m; ++k) {
      double xv = x[i * m + k];
      if (xv == 0.0) continue;
      const double* wr = w + k * p;
      for (int j = 0; j < p; ++j) yr[j] += xv * wr[j];
    }
    for (int j = 0; j < p; ++j) {
      double z = yr[j] + b[j];
      yr[j] = act ? tanh(z) : z;
    }
  }
}

static double forward_one(const double* P, int h, int S, int B, const double* sf,
                          const double* bf, int identity) { /* ranker.cpp:159-209 */
  const double *w1 = P, *b1 = w1 + 24 * h, *w2 = b1 + h, *b2 = w2 + h * h;
  const double *we = b2 + h, *be = we + 23 * h, *wq = be + h, *bq = wq + h * h;
  const double *wk = bq + h, *bk = wk + h * h, *wv = bk + h, *bv = wv + h * h;
  const double *hw1 = bv + h, *hb1 = hw1 + 2 * h * h, *hw2 = hb1 + h, *hb2 = hw2 + h;
  double* z1 = (double*)malloc(sizeof(double) * S * h);
  double* z2 = (double*)malloc(sizeof(double) * S * h);
  double* e = (double*)malloc(sizeof(double) * B * h);
  double* q = (double*)malloc(sizeof(double) * B * h);
  double* kk = (double*)malloc(sizeof(double) * B * h);
  double* v = (double*)malloc(sizeof(double) * B * h);
  double* pr = (double*)malloc(sizeof(double) * B * B);
  double* ao = (double*)calloc((size_t)B * h, sizeof(double));
  double* cat = (double*)calloc((size_t)2 * h, sizeof(double));
  double* g = (double*)malloc(sizeof(double) * h);
  affine(sf, S, 24, w1, b1, h, 1, z1);
  affine(z1, S, h, w2, b2, h, 1, z2);
  affine(bf, B, 23, we, be, h, 1, e);
  const double* pooled = e;
  if (!identity) {
    affine(e, B, h, wq, bq, h, 0, q);
    affine(e, B, h, wk, bk, h, 0, kk);
    affine(e, B, h, wv, bv, h, 0, v);
    double scale = 1.0 / sqrt((double)h);
    for (int i = 0; i < B; ++i) { /* matmul_nt (ranker.cpp:102-111) then scale */
      for (int j = 0; j < B; ++j) {
        double acc = 0.0;
        for (int t = 0; t < h; ++t) acc += q[i * h + t] * kk[j * h + t];
        pr[i * B + j] = acc * scale;
      }
      double mx = pr[i * B];
      for (int j = 1; j < B; ++j) mx = pr[i * B + j] > mx ? pr[i * B + j] : mx;
      double sum = 0.0;
      for (int j = 0; j < B; ++j) {
        double ex = exp(pr[i * B + j] - mx);
        pr[i * B + j] = ex;
        sum += ex;
      }
      for (int j = 0; j < B; ++j) pr[i * B + j] /= sum;
    }
    for (int i = 0; i < B; ++i) /* matmul (ranker.cpp:113-122) */
      for (int t = 0; t < B; ++t) {
        double av = pr[i * B + t];
        if (av == 0.0) continue;
        for (int j = 0; j < h; ++j) ao[i * h + j] += av * v[t * h + j];
      }
    pooled = ao;
  }
  for (int i = 0; i < S; ++i)
    for (int j = 0; j < h; ++j) cat[j] += z2[i * h + j];
  double inv_n = 1.0 / B;
  for (int i = 0; i < B; ++i)
    for (int j = 0; j < h; ++j) cat[h + j] += pooled[i * h + j] * inv_n;
  affine(cat, 1, 2 * h, hw1, hb1, h, 1, g);
  double s;
  affine(g, 1, h, hw2, hb2, 1, 0, &s);
  free(z1), free(z2), free(e), free(q), free(kk), free(v), free(pr), free(ao), free(cat), free(g);
  return s;
}

void tto_score(const double* params, int h, int n_stmt, int n_block, const double* stmt,
               const double* block, int64_t k, int attention_identity, double* score_out) {
  for (int64_t i = 0; i < k; ++i)
    score_out[i] = forward_one(params, h, n_stmt, n_block, stmt + i * n_stmt * TT_STMT_WIDTH,
                               block + i * n_block * TT_BLOCK_WIDTH, attention_identity);
}

/* ---------------- select_top: ranker.cpp:514-532 ---------------- */

static const double* g_sel_scores;
static const double* g_sel_drafts;
static int sel_cmp(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  if (g_sel_scores[x] != g_sel_scores[y]) return g_sel_scores[x] > g_sel_scores[y] ? -1 : 1;
  if (g_sel_drafts[x] != g_sel_drafts[y]) return g_sel_drafts[x] < g_sel_drafts[y] ? -1 : 1;
  return (x > y) - (x < y);
}

int tto_select_top(const double* scores, const double* drafts, const uint8_t* excluded,
                   int64_t n, int64_t b, int64_t* idx_out) {
  int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
  int64_t m = 0;
  for (int64_t i = 0; i < n; ++i)
    if (!excluded || !excluded[i]) idx[m++] = i;
  if (m < b) {
    free(idx);
    return -1;
  }
  g_sel_scores = scores;
  g_sel_drafts = drafts;
  qsort(idx, (size_t)m, sizeof(int64_t), sel_cmp);
  memcpy(idx_out, idx, sizeof(int64_t) * (size_t)b);
  free(idx);
  return 0;
}

/* ---------------- MoA: momentum.cpp:28-46, ranker.cpp:502-506 ---------------- */

void tto_momentum_update(double* phi, const double* target, int64_t n, double m) {
  for (int64_t i = 0; i < n; ++i) phi[i] = target[i] + m * (phi[i] - target[i]);
}

void tto_gd_step(double* params, const double* grads, int64_t n, double lr) {
  for (int64_t i = 0; i < n; ++i) params[i] -= lr * grads[i];
}

/* ---------------- genetic explore, any n_steps: draft.cpp:156-221 + mutate, schedule.cpp:340-396 ---------------- */

typedef struct {
  double cost;
  uint64_t disc;
  int32_t f[4 * TT_MAX_AXES + 1];
} pool_t;

static int pool_cmp(const void* a, const void* b) {
  const pool_t* x = (const pool_t*)a;
  const pool_t* y = (const pool_t*)b;
  if (x->cost != y->cost) return x->cost < y->cost ? -1 : 1;
  return (x->disc > y->disc) - (x->disc < y->disc);
}

/* mutate(population, sketch, costs, rng) (schedule.cpp:340-396) on SoA (ld n) */
static void mutate(const tt_sketch* sk, const int32_t* pop, const double* costs, int64_t n, rng_t* rng,
                   int32_t* next) {
  const double eps = 1e-12;
  const int cols = tt_schedule_cols(sk), n_sp = sk->op.n_spatial;
  const int n_axes = n_sp + sk->op.n_reduction;
  double* cum = (double*)malloc(sizeof(double) * (size_t)n);
  double total = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    total += 1.0 / (costs[i] + eps);
    cum[i] = total;
  }
  int64_t best = 0;
  for (int64_t i = 1; i < n; ++i)
    if (costs[i] < costs[best]) best = i;
  for (int c = 0; c < cols; ++c) next[(int64_t)c * n] = pop[(int64_t)c * n + best];
  for (int64_t j = 1; j < n; ++j) {
    double r = rng_real(rng) * total;
    int64_t lo = 0, hi = n; /* upper_bound: first cum > r */
    while (lo < hi) {
      int64_t mid = (lo + hi) / 2;
      if (cum[mid] > r) hi = mid; else lo = mid + 1;
    }
    int64_t par = lo < n - 1 ? lo : n - 1;
    for (int c = 0; c < cols; ++c) next[(int64_t)c * n + j] = pop[(int64_t)c * n + par];
    int slot = (int)rng_index(rng, (uint64_t)n_axes + 1);
    if (slot == n_axes) {
      next[(int64_t)(cols - 1) * n + j] = sk->unroll[rng_index(rng, (uint64_t)sk->n_unroll)];
      continue;
    }
    int c0 = axis_col(sk, slot), arity = slot_arity(sk, slot);
    int mpos[64];
    int64_t mp[64];
    int nm = 0;
    for (int q = 0; q < arity; ++q) {
      primes_t pr;
      prime_factorize(next[(int64_t)(c0 + q) * n + j], &pr);
      for (int t = 0; t < pr.n; ++t)
        for (int rep = 0; rep < pr.e[t]; ++rep) mpos[nm] = q, mp[nm++] = pr.p[t];
    }
    if (nm > 0 && arity > 1) {
      int m = (int)rng_index(rng, (uint64_t)nm);
      int from = mpos[m], to = (int)rng_index(rng, (uint64_t)arity - 1);
      if (to >= from) ++to;
      next[(int64_t)(c0 + from) * n + j] /= (int32_t)mp[m];
      next[(int64_t)(c0 + to) * n + j] *= (int32_t)mp[m];
    }
  }
  free(cum);
}

int64_t tto_explore(const tt_sketch* sk, const tt_device_spec* dev, int n_steps, int64_t k, int64_t n,
                    uint64_t seed, int toggles, int32_t* soa_out, double* cost_out) {
  const int cols = tt_schedule_cols(sk);
  int32_t* pop = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * cols));
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n * cols));
  double* cost = (double*)malloc(sizeof(double) * (size_t)n);
  pool_t* pool = (pool_t*)malloc(sizeof(pool_t) * (size_t)(k + n));
  int64_t np = 0;
  uint64_t disc = 0;
  rng_t rng;
  rng_init(&rng, seed);
  tto_random_init(sk, seed, 0, n, pop, n); /* consumes n * D draws of the stream */
  rng.state += (uint64_t)n * (uint64_t)tto_draws_per_schedule(sk) * GOLDEN;
  for (int step = 0; step < n_steps; ++step) {
    tto_draft_cost(sk, dev, pop, n, n, toggles, cost);
    for (int64_t i = 0; i < n; ++i) { /* insert if the key is new */
      int found = 0;
      for (int64_t q = 0; q < np && !found; ++q) {
        found = 1;
        for (int c = 0; c < cols && found; ++c) found = pool[q].f[c] == pop[(int64_t)c * n + i];
      }
      if (found) continue;
      pool[np].cost = cost[i], pool[np].disc = disc++;
      for (int c = 0; c < cols; ++c) pool[np].f[c] = pop[(int64_t)c * n + i];
      ++np;
    }
    if (np > k) { /* trim: the k smallest by (cost, discovery) */
      qsort(pool, (size_t)np, sizeof(pool_t), pool_cmp);
      np = k;
    }
    if (step + 1 < n_steps) {
      mutate(sk, pop, cost, n, &rng, next);
      memcpy(pop, next, sizeof(int32_t) * (size_t)(n * cols));
    }
  }
  qsort(pool, (size_t)np, sizeof(pool_t), pool_cmp);
  for (int64_t q = 0; q < np; ++q) {
    cost_out[q] = pool[q].cost;
    for (int c = 0; c < cols; ++c) soa_out[(int64_t)c * k + q] = pool[q].f[c];
  }
  free(pop), free(next), free(cost), free(pool);
  return np;
}

/* ---- lambda_rank_loss (ranker.cpp:394-441) ---------------------------------- */
static double tto_log2d(double x) { return log(x) * 1.4426950408889634074; } /* ranker.cpp:33-35 */
static double tto_softplus(double x) { return x > 30.0 ? x : log1p(exp(x)); } /* ranker.cpp:37-40 */
static double tto_sigmoid(double x) {                                         /* ranker.cpp:42-50 */
  if (x >= 0) {
    double e = exp(-x);
    return 1.0 / (1.0 + e);
  }
  double e = exp(x);
  return e / (1.0 + e);
}

static const double* g_rank_scores; /* qsort comparator context (single-threaded checker) */
static int cmp_rank(const void* a, const void* b) {
  const int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  if (g_rank_scores[i] != g_rank_scores[j]) return g_rank_scores[i] > g_rank_scores[j] ? -1 : 1;
  return i < j ? -1 : (i > j);
}
static int cmp_desc(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x > y ? -1 : (x < y);
}

int tto_rank_loss(const double* scores, const double* lat, int64_t n, double* loss, double* grad) {
  if (n < 2) return -1;
  double min_lat = lat[0];
  for (int64_t i = 0; i < n; ++i) {
    if (!(lat[i] > 0.0)) return -1;
    min_lat = lat[i] < min_lat ? lat[i] : min_lat;
  }
  double* gain = (double*)malloc(sizeof(double) * n);
  double* disc = (double*)malloc(sizeof(double) * n);
  double* ideal = (double*)malloc(sizeof(double) * n);
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * n);
  for (int64_t i = 0; i < n; ++i) gain[i] = exp2(min_lat / lat[i]) - 1.0;
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  g_rank_scores = scores;
  qsort(order, (size_t)n, sizeof(int64_t), cmp_rank); /* desc, ties by index: a strict total order */
  for (int64_t pos = 0; pos < n; ++pos) disc[order[pos]] = 1.0 / tto_log2d((double)pos + 2.0);
  memcpy(ideal, gain, sizeof(double) * n);
  qsort(ideal, (size_t)n, sizeof(double), cmp_desc);
  double max_dcg = 0.0;
  for (int64_t pos = 0; pos < n; ++pos) max_dcg += ideal[pos] / tto_log2d((double)pos + 2.0);
  double L = 0.0;
  if (grad)
    for (int64_t i = 0; i < n; ++i) grad[i] = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      if (!(lat[i] < lat[j])) continue;
      const double w = fabs(gain[i] - gain[j]) * fabs(disc[i] - disc[j]) / max_dcg;
      if (w == 0.0) continue;
      const double d = scores[i] - scores[j];
      L += w * tto_softplus(-d);
      const double slope = w * tto_sigmoid(-d);
      if (grad) {
        grad[i] -= slope;
        grad[j] += slope;
      }
    }
  *loss = L;
  free(gain), free(disc), free(ideal), free(order);
  return 0;
}
