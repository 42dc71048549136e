/*
 * intf_oracle.c -- CPU restatement of the intfsim reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * product path (paper_2512_18725_b200/csrc); only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it.  The product
 * never links or calls it.
 *
 * It restates, in plain C99 (+ unsigned __int128), the reference at
 * /root/reference/pkg/src/intfsim (cited file:line below) together with the
 * third-party arithmetic underneath it:
 *   - numpy 2.3.5 SeedSequence / PCG64 / 256-level ziggurat (`oracle.py:32-33`,
 *     `workload.py:85-90`), tables in oracle_tables.h (tools/gen_tables.py);
 *   - glibc 2.39 libm `exp` and `log1p`, FMA variants (IFUNC targets
 *     libm+0x79b60 / libm+0x7aff0 on AVX2+FMA hosts), restated instruction by
 *     instruction from their disassembly;
 *   - OpenBLAS `ddot` for n<=7 == an fma chain in index order from 0
 *     (`oracle.py:47`, `predict.py:44`);
 *   - zlib crc32 (`profiles.py:239-243`).
 * The event loop is the literal binary-heap engine of `simcore.py:103-310`
 * (NOT the heap-free recurrence the CUDA kernel uses), so the two
 * formulations check each other.
 *
 * Build: oracle/Makefile  ->  oracle/_build/liboracle.so   (gcc -O2
 * -ffp-contract=off: every multiply-add below is unfused unless it is an
 * explicit fma() call).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_tables.h"

typedef unsigned __int128 u128;

static inline uint64_t asu64(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double asf64(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

/* ------------------------------------------------------------------ crc32 */
/* zlib crc32 (reflected 0xEDB88320), `profiles.py:239-243` _stable_id. */
uint32_t oracle_crc32(const unsigned char *buf, size_t n) {
  uint32_t c = 0xFFFFFFFFu;
  for (size_t i = 0; i < n; i++) {
    c ^= buf[i];
    for (int k = 0; k < 8; k++) c = (c >> 1) ^ (0xEDB88320u & (0u - (c & 1u)));
  }
  return c ^ 0xFFFFFFFFu;
}

/* ---------------------------------------------------------- glibc exp (FMA) */
static double exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
  if ((ki & 0x80000000u) == 0) {
    /* k > 0: the exponent of scale might have overflowed by <= 460. */
    sbits -= 1009ull << 52;
    double scale = asf64(sbits);
    return 0x1p1009 * fma(scale, tmp, scale);
  }
  /* k < 0: need special care in the subnormal range. */
  sbits += 1022ull << 52;
  double scale = asf64(sbits);
  double st = tmp * scale;
  double y = scale + st;
  if (1.0 > y) {
    double hi = y + 1.0;
    double lo = (scale - y) + st;
    double t = ((1.0 - hi) + y) + lo;
    y = (t + hi) - 1.0;
    if (y == 0.0) y = 0.0;
  }
  return 0x1p-1022 * y;
}

/* glibc 2.39 __exp, AVX2/FMA build (libm+0x79b60). */
double oracle_exp(double x) {
  const double InvLn2N = asf64(INTF_EXP_INVLN2N_BITS), Shift = asf64(INTF_EXP_SHIFT_BITS);
  const double NegLn2hiN = asf64(INTF_EXP_NEGLN2HIN_BITS), NegLn2loN = asf64(INTF_EXP_NEGLN2LON_BITS);
  const double C2 = asf64(INTF_EXP_C2_BITS), C3 = asf64(INTF_EXP_C3_BITS);
  const double C4 = asf64(INTF_EXP_C4_BITS), C5 = asf64(INTF_EXP_C5_BITS);
  uint64_t ix = asu64(x);
  uint32_t abstop = (uint32_t)(ix >> 52) & 0x7ff;
  if (abstop - 0x3c9u > 0x3eu) {
    if ((int32_t)(abstop - 0x3c9u) < 0) return 1.0 + x; /* |x| < 2^-54 */
    if (abstop > 0x408u) {
      if (ix == 0xfff0000000000000ull) return 0.0;
      if (abstop == 0x7ff) return 1.0 + x;
      return (ix >> 63) ? 0.0 : INFINITY;
    }
    abstop = 0; /* large |x|: handled by the special case below */
  }
  double kd = fma(x, InvLn2N, Shift);
  uint64_t ki = asu64(kd);
  kd -= Shift;
  double r = fma(kd, NegLn2hiN, x);
  r = fma(kd, NegLn2loN, r);
  uint64_t idx = 2 * (ki & 0x7f);
  uint64_t top = ki << 45;
  double tail_r = r + asf64(INTF_EXP_TAB[idx]);
  uint64_t sbits = INTF_EXP_TAB[idx + 1] + top;
  double r2 = r * r;
  double p23 = fma(r, C3, C2);
  double p45 = fma(r, C5, C4);
  double t = fma(p23, r2, tail_r);
  double tmp = fma(r2 * r2, p45, t);
  if (abstop == 0) return exp_specialcase(tmp, sbits, ki);
  double scale = asf64(sbits);
  return fma(scale, tmp, scale);
}

/* ------------------------------------------------------- glibc log1p (FMA) */
/* glibc 2.39 __log1p (fdlibm-derived), AVX2/FMA build (libm+0x7aff0). */
double oracle_log1p(double x) {
  static const double Lp1 = 0x1.5555555555593p-1, Lp2 = 0x1.999999997fa04p-2,
                      Lp3 = 0x1.2492494229359p-2, Lp4 = 0x1.c71c51d8e78afp-3,
                      Lp5 = 0x1.7466496cb03dep-3, Lp6 = 0x1.39a09d078c69fp-3,
                      Lp7 = 0x1.2f112df3e5244p-3;
  static const double ln2_hi = 0x1.62e42fee00000p-1, ln2_lo = 0x1.a39ef35793c76p-33;
  static const double two3rd = 0x1.5555555555555p-1;
  uint64_t ix = asu64(x);
  int32_t hx = (int32_t)(ix >> 32);
  uint32_t hu;
  int k;
  double c = 0.0, u, f, hfsq;
  if (hx > 0x3fda8279) {
    if (hx > 0x7fefffff) return x + x;
    if (hx <= 0x433fffff) goto small_u;
    k = (hx >> 20) - 1023;
    hu = (uint32_t)hx;
    u = x;
    c = 0.0;
    goto normalize;
  }
  {
    uint32_t ax = (uint32_t)hx & 0x7fffffffu;
    if (ax > 0x3fefffffu) {
      if (x == -1.0) return -INFINITY;
      return (x - x) / (x - x);
    }
    if (ax <= 0x3e1fffffu) {
      if (ax <= 0x3c8fffffu) return x;
      return fma(-(x * x), 0.5, x);
    }
    if ((uint32_t)((uint32_t)hx + 0x402d413cu) <= 0x402d413cu) goto small_u;
  }
  /* -0.2929 < x < 0.41422: k = 0, f = x */
  k = 0;
  f = x;
  hfsq = (x * 0.5) * x;
  goto poly;
small_u:
  u = x + 1.0;
  hu = (uint32_t)(asu64(u) >> 32);
  k = ((int32_t)hu >> 20) - 1023;
  if (k > 0) c = 1.0 - (u - x);
  else c = x - (u - 1.0);
  c = c / u;
normalize:
  hu &= 0xfffffu;
  if (hu > 0x6a09du) {
    k += 1;
    u = asf64(((uint64_t)(hu | 0x3fe00000u) << 32) | (asu64(u) & 0xffffffffull));
    hu = (0x00100000u - hu) >> 2;
  } else {
    u = asf64(((uint64_t)(hu | 0x3ff00000u) << 32) | (asu64(u) & 0xffffffffull));
  }
  f = u - 1.0;
  hfsq = (f * 0.5) * f;
  if (hu == 0) {
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = fma((double)k, ln2_lo, c);
      return fma((double)k, ln2_hi, c);
    }
    double R = fma(-f, two3rd, 1.0) * hfsq;
    if (k == 0) return f - R;
    double t = fma((double)k, ln2_lo, c);
    return fma((double)k, ln2_hi, -((R - t) - f));
  }
poly: {
  double s = f / (f + 2.0);
  double z = s * s;
  double R2 = fma(z, Lp3, Lp2);
  double R3 = fma(z, Lp5, Lp4);
  double R4 = fma(z, Lp7, Lp6);
  double z2 = z * z;
  double z4 = z2 * z2;
  double z6 = z2 * z4;
  double R = fma(z, Lp1, z2 * R2);
  R = fma(z4, R3, R);
  R = fma(z6, R4, R);
  double sh = (R + hfsq) * s;
  if (k == 0) return f - (hfsq - sh);
  double t = fma((double)k, ln2_lo, c);
  t = t + sh;
  t = hfsq - t;
  t = t - f;
  return fma((double)k, ln2_hi, -t);
}
}

/* ------------------------------------------------- SeedSequence and PCG64 */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static inline uint32_t ss_hashmix(uint32_t v, uint32_t *hc) {
  v ^= *hc;
  *hc *= SS_MULT_A;
  v *= *hc;
  v ^= v >> 16;
  return v;
}
static inline uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> 16;
  return r;
}

/* numpy SeedSequence(entropy).generate_state(4, uint64) for an entropy
 * already coerced to uint32 words (each int -> little-endian words, 0 -> [0]). */
void oracle_seedseq_state(const uint32_t *ent, int n, uint64_t out[4]) {
  uint32_t pool[4];
  uint32_t hc = SS_INIT_A;
  for (int i = 0; i < 4; i++) pool[i] = ss_hashmix(i < n ? ent[i] : 0u, &hc);
  for (int s = 0; s < 4; s++)
    for (int d = 0; d < 4; d++)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  for (int s = 4; s < n; s++)
    for (int d = 0; d < 4; d++) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));
  uint32_t hb = SS_INIT_B, w[8];
  for (int i = 0; i < 8; i++) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  for (int i = 0; i < 4; i++) out[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
}

typedef struct { u128 state, inc; } pcg64_t;
#define PCG_MULT ((((u128)0x2360ed051fc65da4ull) << 64) | (u128)0x4385df649fccf645ull)

static inline void pcg_step(pcg64_t *r) { r->state = r->state * PCG_MULT + r->inc; }
static inline uint64_t pcg_next64(pcg64_t *r) {
  pcg_step(r);
  uint64_t v = (uint64_t)(r->state >> 64) ^ (uint64_t)r->state;
  unsigned rot = (unsigned)(r->state >> 122);
  return (v >> rot) | (v << ((64u - rot) & 63u));
}
static inline double pcg_next_double(pcg64_t *r) { return (double)(pcg_next64(r) >> 11) * (1.0 / 9007199254740992.0); }

static void pcg_from_words(pcg64_t *r, const uint32_t *ent, int n) {
  uint64_t s[4];
  oracle_seedseq_state(ent, n, s);
  u128 initstate = ((u128)s[0] << 64) | s[1];
  u128 initseq = ((u128)s[2] << 64) | s[3];
  r->state = 0;
  r->inc = (initseq << 1) | 1u;
  pcg_step(r);
  r->state += initstate;
  pcg_step(r);
}

/* append the uint32 words of a non-negative int (numpy _int_to_uint32_array) */
static int push_words(uint32_t *w, int n, uint64_t v) {
  if (v == 0) { w[n++] = 0; return n; }
  while (v) { w[n++] = (uint32_t)v; v >>= 32; }
  return n;
}

/* numpy random_standard_normal (distributions.c), 256-level ziggurat. */
static double zig_normal(pcg64_t *r) {
  static const double ziggurat_nor_r = 3.6541528853610088;
  static const double ziggurat_nor_inv_r = 0.27366123732975828;
  for (;;) {
    uint64_t u = pcg_next64(r);
    int idx = (int)(u & 0xff);
    u >>= 8;
    int sign = (int)(u & 1);
    uint64_t rabs = (u >> 1) & 0x000fffffffffffffull;
    double x = (double)rabs * asf64(INTF_ZIG_WI_BITS[idx]);
    if (sign) x = -x;
    if (rabs < INTF_ZIG_KI[idx]) return x;
    if (idx == 0) {
      for (;;) {
        double xx = -ziggurat_nor_inv_r * oracle_log1p(-pcg_next_double(r));
        double yy = -oracle_log1p(-pcg_next_double(r));
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 1) ? -(ziggurat_nor_r + xx) : ziggurat_nor_r + xx;
      }
    } else {
      double fi1 = asf64(INTF_ZIG_FI_BITS[idx - 1]), fi0 = asf64(INTF_ZIG_FI_BITS[idx]);
      if (((fi1 - fi0) * pcg_next_double(r) + fi0) < oracle_exp(-0.5 * x * x)) return x;
    }
  }
}

/* InterferenceOracle.noise_draw (`oracle.py:24-33`):
 * default_rng([seed, batch_id, segment_index]).lognormal(0, sigma). */
double oracle_noise_draw(uint64_t seed, uint64_t batch_id, uint64_t seg_idx, double sigma) {
  if (sigma == 0.0) return 1.0;
  uint32_t w[8];
  int n = push_words(w, 0, seed);
  n = push_words(w, n, batch_id);
  n = push_words(w, n, seg_idx);
  pcg64_t r;
  pcg_from_words(&r, w, n);
  double z = zig_normal(&r);
  return oracle_exp(0.0 + sigma * z);
}

/* first n doubles of default_rng(words).random() -- for pinning tests */
void oracle_random_doubles(const uint32_t *w, int nw, double *out, int n) {
  pcg64_t r;
  pcg_from_words(&r, w, nw);
  for (int i = 0; i < n; i++) out[i] = pcg_next_double(&r);
}
void oracle_standard_normals(const uint32_t *w, int nw, double *out, int n) {
  pcg64_t r;
  pcg_from_words(&r, w, nw);
  for (int i = 0; i < n; i++) out[i] = zig_normal(&r);
}

/* ------------------------------------------------------------- ddot / slowdown */
/* OpenBLAS ddot, n <= 7 (SkylakeX tail loop): fma chain in index order. */
double oracle_ddot(const double *a, const double *b, int n) {
  double acc = 0.0;
  for (int i = 0; i < n; i++) acc = fma(a[i], b[i], acc);
  return acc;
}

/* oracle_slowdown (`oracle.py:36-47`) */
double oracle_slowdown(const double own[3], const double colo[3], const double beta[3], double noise) {
  double e[3];
  for (int i = 0; i < 3; i++) {
    double v = (own[i] + colo[i]) - 1.0;
    e[i] = v > 0.0 ? v : 0.0;
  }
  return (1.0 + oracle_ddot(beta, e, 3)) * noise;
}

/* ------------------------------------------------------------ arrivals */
/* ScenarioIn: everything run_scenario needs, flattened by oracle.py. */
typedef struct {
  int n_models;            /* deployed models, in spec order */
  const double *rate_rps;  /* [n_models] */
  const double *slo_ms;    /* [n_models] */
  const uint32_t *crc;     /* [n_models] crc32(model_id) */
  const int *name_rank;    /* [n_models] rank of model_id in Python str order */
  const int *entry_base;   /* [n_models] table row of (model, bs=1); bs=b -> base+b-1 */
  const double *tab_solo;  /* profile table, rows */
  const double *tab_thr;   /* [rows*3] (l2, dram, sm) */
  double duration_s, window_ms, sigma, beta[3];
  int max_bs, cap;
  uint64_t seed, oracle_seed;
  uint64_t batch_id_base; /* noise key offset (batches numbered across scenarios) */
} ScenarioIn;

typedef struct { double t; int rank; int model; } Arr;

static int arr_cmp(const void *a, const void *b) {
  const Arr *x = (const Arr *)a, *y = (const Arr *)b;
  if (x->t < y->t) return -1;
  if (x->t > y->t) return 1;
  return (x->rank > y->rank) - (x->rank < y->rank);
}

/* generate_arrivals (`workload.py:74-104`); returns count, or -1 if cap exceeded */
int oracle_generate_arrivals(const ScenarioIn *s, double *t_out, int *model_out, int cap_out) {
  double horizon = s->duration_s * 1000.0;
  int n = 0, cap = 1024;
  Arr *a = (Arr *)malloc(sizeof(Arr) * (size_t)cap);
  for (int m = 0; m < s->n_models; m++) {
    if (s->rate_rps[m] == 0.0) continue;
    uint32_t w[4];
    int nw = push_words(w, 0, s->seed);
    nw = push_words(w, nw, s->crc[m]);
    pcg64_t r;
    pcg_from_words(&r, w, nw);
    double mean_gap = 1000.0 / s->rate_rps[m];
    double t = 0.0;
    for (;;) {
      double gap = -mean_gap * oracle_log1p(-pcg_next_double(&r));
      t += gap > 1e-12 ? gap : 1e-12;
      if (t >= horizon) break;
      if (n == cap) { cap *= 2; a = (Arr *)realloc(a, sizeof(Arr) * (size_t)cap); }
      a[n].t = t; a[n].rank = s->name_rank[m]; a[n].model = m; n++;
    }
  }
  qsort(a, (size_t)n, sizeof(Arr), arr_cmp);
  if (n > cap_out) { free(a); return -1; }
  for (int i = 0; i < n; i++) { t_out[i] = a[i].t; model_out[i] = a[i].model; }
  free(a);
  return n;
}

/* -------------------------------------------------------------- event heap */
enum { EV_COMPLETION = 0, EV_WINDOW = 1, EV_ARRIVAL = 2 };
typedef struct { double t; int kind; int64_t key; int64_t seq; int a, b; } Ev;
typedef struct { Ev *v; int n, cap; int64_t seq; } Heap;

static int ev_less(const Ev *x, const Ev *y) {
  if (x->t != y->t) return x->t < y->t;
  if (x->kind != y->kind) return x->kind < y->kind;
  if (x->key != y->key) return x->key < y->key;
  return x->seq < y->seq;
}
static void heap_push(Heap *h, double t, int kind, int64_t key, int a, int b) {
  if (h->n == h->cap) { h->cap = h->cap ? 2 * h->cap : 1024; h->v = (Ev *)realloc(h->v, sizeof(Ev) * (size_t)h->cap); }
  Ev e = {t, kind, key, h->seq++, a, b};
  int i = h->n++;
  while (i > 0) {
    int p = (i - 1) / 2;
    if (!ev_less(&e, &h->v[p])) break;
    h->v[i] = h->v[p];
    i = p;
  }
  h->v[i] = e;
}
static Ev heap_pop(Heap *h) {
  Ev top = h->v[0], last = h->v[--h->n];
  int i = 0;
  for (;;) {
    int l = 2 * i + 1, r = l + 1, m = i;
    const Ev *mv = &last;
    if (l < h->n && ev_less(&h->v[l], mv)) { m = l; mv = &h->v[l]; }
    if (r < h->n && ev_less(&h->v[r], mv)) { m = r; mv = &h->v[r]; }
    if (m == i) break;
    h->v[i] = h->v[m];
    i = m;
  }
  if (h->n) h->v[i] = last;
  return top;
}

/* --------------------------------------------------------------- replay */
typedef struct {
  /* per batch, indexed by batch_id */
  int *b_model, *b_size, *b_first_req; /* first member (arrival index) */
  double *b_formed, *b_start, *b_completion, *b_measured, *b_profiled;
  int *b_seg_off, *b_nseg, *b_done_rank;
  int *b_running; /* running batches right after this batch's dispatch (the spy of `test_acceptance.py:98-106`) */
  /* per segment (grouped per batch, in completion order of batches) */
  double *s_tbegin, *s_tend, *s_slowdown, *s_colo; /* colo [n*3] */
  /* per request (arrival index) */
  int *r_batch;
  unsigned char *r_slo_met;
  /* capacities */
  int cap_batches, cap_segments;
  /* results */
  int n_batches, n_segments, n_reseats, status;
} ReplayOut;

enum { ST_OK = 0, ST_PAST_EVENT = 1, ST_CAP = 2, ST_PROGRESS = 4, ST_NONQUIESCENT = 8, ST_OVERFLOW = 16 };

typedef struct {
  int batch, entry;
  double start, total, progress;
  int gen, nseg;
  /* open/closed segments of this batch, grown as needed */
  double *tb, *te, *sl, *colo;
  int segcap;
} RB;

typedef struct {
  const ScenarioIn *s;
  double now;
  RB *run;
  int nrun;
  Heap heap;
  ReplayOut *o;
  int status;
} Sim;

static void sim_push(Sim *S, double t, int kind, int64_t key, int a, int b) {
  if (t < S->now - 1e-9) S->status |= ST_PAST_EVENT; /* SimulationError `simcore.py:118-121` */
  heap_push(&S->heap, t, kind, key, a, b);
}

/* GpuState._reseat (`simcore.py:133-141`) */
static void sim_reseat(Sim *S, RB *rb) {
  const ScenarioIn *s = S->s;
  double colo[3] = {0.0, 0.0, 0.0};
  for (int i = 0; i < S->nrun; i++) {
    RB *o = &S->run[i];
    if (o == rb) continue;
    const double *p = &s->tab_thr[3 * o->entry];
    colo[0] += p[0]; colo[1] += p[1]; colo[2] += p[2];
  }
  double noise = oracle_noise_draw(s->oracle_seed, s->batch_id_base + (uint64_t)rb->batch, (uint64_t)rb->nseg, s->sigma);
  double sd = oracle_slowdown(&s->tab_thr[3 * rb->entry], colo, s->beta, noise);
  if (rb->nseg == rb->segcap) {
    rb->segcap = rb->segcap ? 2 * rb->segcap : 8;
    rb->tb = (double *)realloc(rb->tb, sizeof(double) * (size_t)rb->segcap);
    rb->te = (double *)realloc(rb->te, sizeof(double) * (size_t)rb->segcap);
    rb->sl = (double *)realloc(rb->sl, sizeof(double) * (size_t)rb->segcap);
    rb->colo = (double *)realloc(rb->colo, sizeof(double) * 3 * (size_t)rb->segcap);
  }
  int k = rb->nseg++;
  rb->tb[k] = S->now; rb->te[k] = NAN; rb->sl[k] = sd;
  rb->colo[3 * k] = colo[0]; rb->colo[3 * k + 1] = colo[1]; rb->colo[3 * k + 2] = colo[2];
  rb->gen += 1;
  S->o->n_reseats++;
  double done_at = S->now + (rb->total - rb->progress) * sd;
  sim_push(S, done_at, EV_COMPLETION, rb->batch, rb->batch, rb->gen);
}

/* RunningBatch.close_segment (`simcore.py:56-66`) */
static void sim_close(Sim *S, RB *rb) {
  int k = rb->nseg - 1;
  if (S->now == rb->tb[k]) { rb->nseg--; return; }
  rb->te[k] = S->now;
  rb->progress += (rb->te[k] - rb->tb[k]) / rb->sl[k];
}

int oracle_run_scenario(const ScenarioIn *s, const double *arr_t, const int *arr_model, int n_req, ReplayOut *o) {
  const int M = s->n_models;
  Sim S;
  memset(&S, 0, sizeof(S));
  S.s = s; S.o = o;
  S.run = (RB *)calloc((size_t)(s->cap + 1), sizeof(RB));
  o->n_batches = o->n_segments = o->n_reseats = 0;
  /* per-model pending queues (`batcher.py:32-85`): a FIFO of arrival indices */
  int *qbuf = (int *)malloc(sizeof(int) * (size_t)(n_req > 0 ? n_req : 1) * 1);
  int *qhead = (int *)calloc((size_t)M, sizeof(int)), *qlen = (int *)calloc((size_t)M, sizeof(int));
  int *mstart = (int *)calloc((size_t)M + 1, sizeof(int));
  int *gen = (int *)calloc((size_t)M, sizeof(int)), *armed = (int *)malloc(sizeof(int) * (size_t)M);
  double *deadline = (double *)malloc(sizeof(double) * (size_t)M);
  char *has_deadline = (char *)calloc((size_t)M, 1);
  for (int i = 0; i < n_req; i++) mstart[arr_model[i] + 1]++;
  for (int m = 0; m < M; m++) mstart[m + 1] += mstart[m];
  for (int m = 0; m < M; m++) { qhead[m] = mstart[m]; armed[m] = -1; }
  /* dispatch FIFO of batch ids (`simcore.py:236`) */
  int dq_head = 0; /* batches [dq_head, n_batches) are formed but not dispatched */
  int nseg_total = 0, done_rank = 0;

  for (int i = 0; i < n_req; i++) sim_push(&S, arr_t[i], EV_ARRIVAL, i, i, 0);

#define FORM_BATCH(m, size, now_)                                              \
  do {                                                                         \
    int b_ = o->n_batches;                                                     \
    if (b_ >= o->cap_batches) { S.status |= ST_OVERFLOW; goto done; }          \
    o->b_model[b_] = (m); o->b_size[b_] = (size);                              \
    o->b_first_req[b_] = qbuf[qhead[m] - mstart[m] + mstart[m]];              \
    for (int j_ = 0; j_ < (size); j_++) o->r_batch[qbuf[qhead[m] + j_]] = b_;  \
    o->b_formed[b_] = (now_);                                                  \
    qhead[m] += (size); qlen[m] -= (size); gen[m]++;                           \
    if (qlen[m]) { deadline[m] = (now_) + s->window_ms; has_deadline[m] = 1; } \
    else has_deadline[m] = 0;                                                  \
    o->n_batches++;                                                            \
  } while (0)

  while (S.heap.n) {
    Ev e = heap_pop(&S.heap);
    if (e.t < S.now - 1e-9) S.status |= ST_PAST_EVENT;
    S.now = S.now > e.t ? S.now : e.t;
    if (e.kind == EV_COMPLETION) {
      int ri = -1;
      for (int i = 0; i < S.nrun; i++) if (S.run[i].batch == e.a) { ri = i; break; }
      if (ri < 0 || S.run[ri].gen != e.b) continue; /* stale (`simcore.py:283-286`) */
      RB rb = S.run[ri];
      sim_close(&S, &S.run[ri]);
      rb = S.run[ri];
      if (fabs(rb.progress - rb.total) > 1e-6 * rb.total) S.status |= ST_PROGRESS;
      for (int i = ri; i + 1 < S.nrun; i++) S.run[i] = S.run[i + 1];
      S.nrun--;
      double measured = S.now - rb.start;
      int all_one = 1;
      for (int k = 0; k < rb.nseg; k++) if (rb.sl[k] != 1.0) { all_one = 0; break; }
      if (all_one) measured = rb.total;
      int b = rb.batch;
      o->b_start[b] = rb.start; o->b_completion[b] = S.now; o->b_measured[b] = measured;
      o->b_profiled[b] = rb.total; o->b_done_rank[b] = done_rank++;
      if (nseg_total + rb.nseg > o->cap_segments) { S.status |= ST_OVERFLOW; goto done; }
      o->b_seg_off[b] = nseg_total; o->b_nseg[b] = rb.nseg;
      for (int k = 0; k < rb.nseg; k++) {
        int q = nseg_total + k;
        o->s_tbegin[q] = rb.tb[k]; o->s_tend[q] = rb.te[k]; o->s_slowdown[q] = rb.sl[k];
        o->s_colo[3 * q] = rb.colo[3 * k]; o->s_colo[3 * q + 1] = rb.colo[3 * k + 1]; o->s_colo[3 * q + 2] = rb.colo[3 * k + 2];
      }
      nseg_total += rb.nseg;
      free(rb.tb); free(rb.te); free(rb.sl); free(rb.colo);
      /* _colo_changed(survivors) (`simcore.py:143-146,198`) */
      for (int i = 0; i < S.nrun; i++) { sim_close(&S, &S.run[i]); sim_reseat(&S, &S.run[i]); }
    } else if (e.kind == EV_WINDOW) {
      int m = e.a;
      if (e.b != gen[m]) continue; /* `simcore.py:289-293` */
      /* poll_window (`batcher.py:74-85`) */
      if (qlen[m] && has_deadline[m] && !(S.now < deadline[m])) {
        int size = qlen[m] < s->max_bs ? qlen[m] : s->max_bs;
        FORM_BATCH(m, size, S.now);
      }
      if (has_deadline[m] && armed[m] != gen[m]) { armed[m] = gen[m]; sim_push(&S, deadline[m], EV_WINDOW, s->crc[m], m, gen[m]); }
    } else {
      int i = e.a, m = arr_model[i];
      /* enqueue (`batcher.py:59-72`) */
      int was_empty = qlen[m] == 0;
      qbuf[qhead[m] + qlen[m]] = i;
      qlen[m]++;
      if (was_empty) { deadline[m] = S.now + s->window_ms; has_deadline[m] = 1; gen[m]++; }
      if (qlen[m] >= s->max_bs) FORM_BATCH(m, s->max_bs, S.now);
      if (has_deadline[m] && armed[m] != gen[m]) { armed[m] = gen[m]; sim_push(&S, deadline[m], EV_WINDOW, s->crc[m], m, gen[m]); }
    }
    /* try_dispatch (`simcore.py:258-262`) -> GpuState.dispatch (`:153-171`) */
    while (dq_head < o->n_batches && S.nrun < s->cap) {
      int b = dq_head++;
      RB *rb = &S.run[S.nrun++];
      memset(rb, 0, sizeof(*rb));
      rb->batch = b;
      rb->entry = s->entry_base[o->b_model[b]] + o->b_size[b] - 1;
      rb->start = S.now;
      rb->total = s->tab_solo[rb->entry];
      o->b_running[b] = S.nrun;
      sim_reseat(&S, rb);
      for (int i = 0; i + 1 < S.nrun; i++) { sim_close(&S, &S.run[i]); sim_reseat(&S, &S.run[i]); }
    }
  }
  if (S.nrun || dq_head < o->n_batches) S.status |= ST_NONQUIESCENT;
  for (int m = 0; m < M; m++) if (qlen[m]) S.status |= ST_NONQUIESCENT;
  /* record_requests (`simcore.py:264-279`): slo_met = latency <= slo */
  for (int i = 0; i < n_req; i++) {
    int b = o->r_batch[i];
    double lat = o->b_completion[b] - arr_t[i];
    o->r_slo_met[i] = lat <= s->slo_ms[arr_model[i]];
  }
done:
  o->n_segments = nseg_total;
  for (int i = 0; i < S.nrun; i++) { free(S.run[i].tb); free(S.run[i].te); free(S.run[i].sl); free(S.run[i].colo); }
  free(S.run); free(S.heap.v); free(qbuf); free(qhead); free(qlen); free(mstart); free(gen); free(armed);
  free(deadline); free(has_deadline);
  o->status = S.status;
  return S.status;
}

/* ------------------------------------------------------------- features */
/* estimate_from_history + finalize_features (`colocation.py:46-84`):
 * static: r = h[0]; EWMA(alpha): r <- alpha*x + (1-alpha)*r over h[1:],
 * elementwise and unfused (numpy ufuncs). x = own (3) ++ r (3). */
void oracle_features(const double *colo_hist, int nseg, const double own[3], int ewma, double alpha, double x[6]) {
  double r[3] = {colo_hist[0], colo_hist[1], colo_hist[2]};
  if (ewma) {
    double om = 1.0 - alpha;
    for (int k = 1; k < nseg; k++)
      for (int i = 0; i < 3; i++) {
        double a = alpha * colo_hist[3 * k + i];
        double b = om * r[i];
        r[i] = a + b;
      }
  }
  x[0] = own[0]; x[1] = own[1]; x[2] = own[2];
  x[3] = r[0]; x[4] = r[1]; x[5] = r[2];
}

/* predict (`predict.py:43-44`): w @ x (ddot fma chain) + b */
double oracle_predict(const double w[6], double b, const double x[6]) { return oracle_ddot(w, x, 6) + b; }
