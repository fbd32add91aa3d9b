/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the DISTWAR reduction stage.
 *
 * A plain-C restatement of the reference's hot path (warpred, C++20):
 *   - the 32-lane SIMT primitives          proj/include/warpred/simt.hpp:27-82
 *   - the seeded trace generator           proj/src/workload.cpp:15-153
 *   - the four core policies + oracle      proj/src/reducers.cpp:16-237
 *   - the WRTRACEB binary container        proj/src/trace_io.cpp:159-276
 *   - the Observation-1/2 histograms       proj/src/workload.cpp:155-197
 *
 * Parity of this restatement is PINNED against the reference itself: the
 * reference sources are compiled unmodified into oracle/_ref/ (oracle/Makefile)
 * and tests/test_oracle_vs_ref.py / tests/golden/ compare traces byte-for-byte
 * and sums bit-for-bit. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library; the product
 * (paper_2401_05345_b200/) never links or calls it.
 */
#include "warpred_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- mt19937_64
 * std::mt19937_64 (the reference's single RNG stream, workload.cpp:111). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) +
               (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    static const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* Variate transforms, workload.cpp:15-52. */
static double uniform01(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1.0p-53; }
static int bernoulli(mt64* g, double p) { return uniform01(g) < p; }
static int poisson(mt64* g, double mean) {
  const double limit = exp(-mean);
  int k = 0;
  double p = 1.0;
  do {
    ++k;
    p *= uniform01(g);
  } while (p > limit);
  return k - 1;
}
static int64_t geometric_at_least_one(mt64* g, double mean) {
  if (mean <= 1.0) return 1;
  const double p = 1.0 / mean;
  const double u = uniform01(g);
  double len = floor(log1p(-u) / log1p(-p)) + 1.0;
  if (len < 1.0) len = 1.0;
  return (int64_t)len;
}
static double draw_grad(mt64* g, int quantized) {
  if (quantized) {
    const int k = 1 + (int)(mt64_next(g) % 255ULL);
    return (double)k / 256.0;
  }
  return 2.0 * uniform01(g) - 1.0;
}

/* --------------------------------------------------------------- the trace */
static __thread char g_err[512] = "ok";
const char* or_last_error(void) { return g_err; }
static int fail(const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return 1;
}

void or_scene_spec_init(or_scene_spec* s) {
  /* SceneSpec defaults, workload.hpp:16-36 */
  s->num_primitives = 1024;
  s->params_per_primitive = 3;
  s->image_width = 64;
  s->image_height = 32;
  s->mean_fragment_span = 64.0;
  s->fragments_per_pixel_mean = 1.0;
  s->activity_prob = 1.0;
  s->locality = 1.0;
  s->seed = 0;
  s->quantized_values = 1;
}

/* SceneSpec::validate, workload.cpp:85-97 (same field names in messages). */
static int validate(const or_scene_spec* s) {
  const char* f = NULL;
  if (s->num_primitives < 1) f = "num_primitives";
  else if (s->params_per_primitive < 1) f = "params_per_primitive";
  else if (s->image_width < 1) f = "image_width";
  else if (s->image_height < 1) f = "image_height";
  else if (!(s->mean_fragment_span >= 1.0)) f = "mean_fragment_span";
  else if (!(s->fragments_per_pixel_mean > 0.0)) f = "fragments_per_pixel_mean";
  else if (!(s->activity_prob >= 0.0 && s->activity_prob <= 1.0)) f = "activity_prob";
  else if (!(s->locality >= 0.0 && s->locality <= 1.0)) f = "locality";
  if (f) {
    snprintf(g_err, sizeof g_err, "SceneSpec: invalid field %s", f);
    return 1;
  }
  return 0;
}

static int reserve(or_trace* t, int64_t want) {
  if (want <= t->capacity) return 0;
  int64_t cap = t->capacity ? t->capacity : 1024;
  while (cap < want) cap *= 2;
  const int n = t->scene.params_per_primitive;
  int32_t* w = realloc(t->warp_id, (size_t)cap * sizeof(int32_t));
  if (w) t->warp_id = w;
  int32_t* it = realloc(t->iteration, (size_t)cap * sizeof(int32_t));
  if (it) t->iteration = it;
  uint32_t* a = realloc(t->active, (size_t)cap * sizeof(uint32_t));
  if (a) t->active = a;
  int32_t* p = realloc(t->prim, (size_t)cap * 32 * sizeof(int32_t));
  if (p) t->prim = p;
  double* gr = realloc(t->grads, (size_t)cap * 32 * (size_t)n * sizeof(double));
  if (gr) t->grads = gr;
  if (!w || !it || !a || !p || !gr) return fail("out of memory");
  t->capacity = cap;
  return 0;
}

or_trace* or_trace_new(const or_scene_spec* s) {
  or_trace* t = calloc(1, sizeof(or_trace));
  if (t && s) t->scene = *s;
  return t;
}

void or_trace_free(or_trace* t) {
  if (!t) return;
  free(t->warp_id);
  free(t->iteration);
  free(t->active);
  free(t->prim);
  free(t->grads);
  free(t);
}

/* workload::generate, workload.cpp:99-153, including FragmentStream
 * (:56-81) and its draw order. */
int or_generate(const or_scene_spec* s, or_trace** out) {
  if (!s || !out) return fail("null argument");
  if (validate(s)) return 1;
  or_trace* t = or_trace_new(s);
  if (!t) return fail("out of memory");
  mt64* g = malloc(sizeof(mt64));
  mt64_seed(g, s->seed);
  /* FragmentStream ctor -> advance() */
  int32_t cur = (int32_t)(mt64_next(g) % (uint64_t)s->num_primitives);
  int64_t remaining = geometric_at_least_one(g, s->mean_fragment_span);

  const int tiles_x = (s->image_width + 7) / 8;
  const int tiles_y = (s->image_height + 3) / 4;
  const int num_warps = tiles_x * tiles_y;
  const int n = s->params_per_primitive;
  for (int32_t warp = 0; warp < num_warps; ++warp) {
    int trips = poisson(g, s->fragments_per_pixel_mean);
    if (trips < 1) trips = 1;
    for (int32_t iter = 0; iter < trips; ++iter) {
      if (reserve(t, t->num_records + 1)) {
        free(g);
        or_trace_free(t);
        return 1;
      }
      const int64_t r = t->num_records++;
      uint32_t active = 0;
      int32_t* prim = t->prim + r * 32;
      double* gr = t->grads + r * 32 * n;
      memset(gr, 0, sizeof(double) * 32 * (size_t)n);
      t->warp_id[r] = warp;
      t->iteration[r] = iter;
      for (int lane = 0; lane < 32; ++lane)
        if (bernoulli(g, s->activity_prob)) active |= 1u << lane;
      /* take_warp_slice */
      const int32_t base = cur;
      remaining -= 32;
      if (remaining <= 0) {
        cur = (int32_t)(mt64_next(g) % (uint64_t)s->num_primitives);
        remaining = geometric_at_least_one(g, s->mean_fragment_span);
      }
      if (bernoulli(g, s->locality)) {
        for (int lane = 0; lane < 32; ++lane) prim[lane] = base;
      } else {
        const int k = 2 + (int)(mt64_next(g) % 7ULL);
        for (int lane = 0; lane < 32; ++lane) {
          const int32_t offs = (int32_t)(mt64_next(g) % (uint64_t)k);
          prim[lane] = (base + offs) % s->num_primitives;
        }
      }
      for (int lane = 0; lane < 32; ++lane) {
        if (!(active >> lane & 1u)) continue;
        for (int p = 0; p < n; ++p)
          gr[lane * n + p] = draw_grad(g, s->quantized_values);
      }
      t->active[r] = active;
    }
  }
  free(g);
  *out = t;
  return 0;
}

/* --------------------------------------------------------------- policies */
static int ffs1(uint32_t m) { return m ? __builtin_ctz(m) + 1 : 0; } /* simt.hpp:31-33 */

typedef struct {
  int32_t* prim;
  int32_t* param;
  double* val;
  int64_t count;
} reqbuf;

static void emit(reqbuf* o, int32_t prim, int32_t param, double v) {
  if (o->prim) {
    o->prim[o->count] = prim;
    o->param[o->count] = param;
    o->val[o->count] = v;
  }
  ++o->count;
}

static void emit_lane(reqbuf* o, const int32_t* prim, const double* gr, int n,
                      int lane) {
  for (int p = 0; p < n; ++p) emit(o, prim[lane], p, gr[lane * n + p]);
}

/* all_lanes_same_primitive, reducers.cpp:49-56 */
static int all_same(const int32_t* prim) {
  if (prim[0] < 0) return 0;
  for (int l = 1; l < 32; ++l)
    if (prim[l] != prim[0]) return 0;
  return 1;
}

/* butterfly_fold, reducers.cpp:71-80: shuffle_down tree 16,8,4,2,1 over all
 * 32 lanes (out-of-range lanes read their own value, simt.hpp:75-82). */
static double bfly(const double* gr, int n, int p) {
  double v[32], s[32];
  for (int l = 0; l < 32; ++l) v[l] = gr[l * n + p];
  for (int off = 16; off >= 1; off /= 2) {
    for (int l = 0; l < 32; ++l) s[l] = (l + off < 32) ? v[l + off] : v[l];
    for (int l = 0; l < 32; ++l) v[l] += s[l];
  }
  return v[0];
}

/* One record through one policy (reducers.cpp:84-237). Returns 0 on
 * success; the request arrays may be NULL to only count. */
static int policy_record(uint32_t active, const int32_t* prim, const double* gr,
                         int n, int kind, int t, reqbuf* o, uint64_t* instr,
                         uint64_t* fpadds) {
  uint64_t ins = 0, fp = 0;
  if ((kind == OR_SW_S || kind == OR_SW_B) && (t < 0 || t > 33))
    return fail("balance threshold out of range 0..33");
  switch (kind) {
    case OR_NATIVE: { /* :84-93 */
      const int64_t c0 = o->count;
      for (int l = 0; l < 32; ++l)
        if (active >> l & 1u) emit_lane(o, prim, gr, n, l);
      ins = (uint64_t)(o->count - c0);
      break;
    }
    case OR_SW_S: { /* :95-136, groups in ascending-leader order (:34-45) */
      uint32_t remaining = active;
      while (remaining) {
        const int leader = ffs1(remaining) - 1;
        uint32_t group = 0; /* match_any(active, prim)[leader], simt.hpp:39-51 */
        for (int j = 0; j < 32; ++j)
          if ((active >> j & 1u) && prim[j] == prim[leader]) group |= 1u << j;
        const int cnt = __builtin_popcount(group);
        ins += 3; /* match_any + popc + branch */
        if (cnt >= t) {
          ins += 1; /* ffs */
          double sums[64];
          double* sp = n <= 64 ? sums : malloc(sizeof(double) * (size_t)n);
          for (int p = 0; p < n; ++p) sp[p] = gr[leader * n + p];
          uint32_t fetch = group & ~(1u << leader);
          while (fetch) {
            const int src = ffs1(fetch) - 1;
            fetch &= ~(1u << src);
            for (int p = 0; p < n; ++p) sp[p] += gr[src * n + p];
            ins += 2 + (uint64_t)n;
            fp += (uint64_t)n;
          }
          for (int p = 0; p < n; ++p) emit(o, prim[leader], p, sp[p]);
          ins += (uint64_t)n;
          if (sp != sums) free(sp);
        } else {
          uint32_t members = group;
          while (members) {
            const int l = ffs1(members) - 1;
            members &= ~(1u << l);
            emit_lane(o, prim, gr, n, l);
          }
          ins += (uint64_t)cnt * (uint64_t)n;
        }
        remaining &= ~group;
      }
      break;
    }
    case OR_SW_B: { /* :138-175 */
      const int same = all_same(prim);
      const int act = __builtin_popcount(active);
      ins = 4; /* match_any + ballot + popc + branch */
      if (same && act > 0 && act >= t) {
        for (int p = 0; p < n; ++p) emit(o, prim[0], p, bfly(gr, n, p));
        ins += 5 * (uint64_t)n + (uint64_t)n;
        fp += 32 * 5 * (uint64_t)n;
      } else {
        const int64_t c0 = o->count;
        for (int l = 0; l < 32; ++l)
          if (active >> l & 1u) emit_lane(o, prim, gr, n, l);
        ins += (uint64_t)(o->count - c0);
      }
      break;
    }
    case OR_CCCL: { /* :177-206, param-major, check repeated per param */
      const int same = all_same(prim);
      const int act = __builtin_popcount(active);
      for (int p = 0; p < n; ++p) {
        ins += 4;
        if (same && act > 0) {
          emit(o, prim[0], p, bfly(gr, n, p));
          ins += 5 + 1;
          fp += 32 * 5;
        } else {
          for (int l = 0; l < 32; ++l)
            if (active >> l & 1u) emit(o, prim[l], p, gr[l * n + p]);
          ins += (uint64_t)act;
        }
      }
      break;
    }
    default: /* apply_policy, :222-237 */
      return fail("apply_policy: hw_atomred has no per-record core policy");
  }
  if (instr) *instr = ins;
  if (fpadds) *fpadds = fp;
  return 0;
}

int or_record_policy(uint32_t active, const int32_t* prim, const double* grads,
                     int32_t n, int kind, int threshold, int32_t* out_prim,
                     int32_t* out_param, double* out_val, int64_t* out_count,
                     uint64_t* instr, uint64_t* fp_adds) {
  if (!prim || !grads || !out_count || n < 1) return fail("null argument");
  reqbuf o = {out_prim, out_param, out_val, 0};
  if (policy_record(active, prim, grads, n, kind, threshold, &o, instr, fp_adds))
    return 1;
  *out_count = o.count;
  return 0;
}

int or_apply_policy(const or_trace* t, int kind, int threshold,
                    int32_t num_prims, double* sums, uint64_t counts3[3]) {
  if (!t || !sums || !counts3) return fail("null argument");
  const int n = t->scene.params_per_primitive;
  const size_t words = (size_t)num_prims * (size_t)n;
  memset(sums, 0, words * sizeof(double));
  int32_t bp[64 * 32], bq[64 * 32];
  double bv[64 * 32];
  int32_t* pp = bp;
  int32_t* pq = bq;
  double* pv = bv;
  if (n > 64) {
    pp = malloc(sizeof(int32_t) * 32 * (size_t)n);
    pq = malloc(sizeof(int32_t) * 32 * (size_t)n);
    pv = malloc(sizeof(double) * 32 * (size_t)n);
  }
  counts3[0] = counts3[1] = counts3[2] = 0;
  int rc = 0;
  for (int64_t r = 0; r < t->num_records && !rc; ++r) {
    reqbuf o = {pp, pq, pv, 0};
    uint64_t ins = 0, fp = 0;
    rc = policy_record(t->active[r], t->prim + r * 32, t->grads + r * 32 * n, n,
                       kind, threshold, &o, &ins, &fp);
    for (int64_t i = 0; i < o.count && !rc; ++i) {
      if (pp[i] < 0 || pp[i] >= num_prims) rc = fail("primitive out of range");
      else sums[(size_t)pp[i] * n + pq[i]] += pv[i];
    }
    counts3[0] += (uint64_t)o.count;
    counts3[1] += ins;
    counts3[2] += fp;
  }
  if (n > 64) {
    free(pp);
    free(pq);
    free(pv);
  }
  return rc;
}

/* oracle_sum, reducers.cpp:208-220: f64, trace order, active lanes only. */
int or_oracle_sum(const or_trace* t, int32_t num_prims, double* sums,
                  uint8_t* touched) {
  if (!t || !sums) return fail("null argument");
  const int n = t->scene.params_per_primitive;
  memset(sums, 0, (size_t)num_prims * n * sizeof(double));
  if (touched) memset(touched, 0, (size_t)num_prims * n);
  for (int64_t r = 0; r < t->num_records; ++r) {
    const uint32_t a = t->active[r];
    const int32_t* prim = t->prim + r * 32;
    const double* gr = t->grads + r * 32 * n;
    for (int l = 0; l < 32; ++l) {
      if (!(a >> l & 1u)) continue;
      if (prim[l] < 0 || prim[l] >= num_prims) return fail("primitive out of range");
      for (int p = 0; p < n; ++p) {
        sums[(size_t)prim[l] * n + p] += gr[l * n + p];
        if (touched) touched[(size_t)prim[l] * n + p] = 1;
      }
    }
  }
  return 0;
}

/* histogram_distinct_primitives / histogram_active_lanes,
 * workload.cpp:155-197 (records with empty masks skipped for distinct). */
int or_histograms(const or_trace* t, uint64_t distinct[33], uint64_t act[33]) {
  if (!t) return fail("null argument");
  if (t->num_records == 0) return fail("histogram: empty trace");
  memset(distinct, 0, 33 * sizeof(uint64_t));
  memset(act, 0, 33 * sizeof(uint64_t));
  for (int64_t r = 0; r < t->num_records; ++r) {
    const uint32_t a = t->active[r];
    act[__builtin_popcount(a)]++;
    if (!a) continue;
    int32_t seen[32];
    int c = 0;
    for (int l = 0; l < 32; ++l) {
      if (!(a >> l & 1u)) continue;
      int f = 0;
      for (int i = 0; i < c; ++i)
        if (seen[i] == t->prim[r * 32 + l]) f = 1;
      if (!f) seen[c++] = t->prim[r * 32 + l];
    }
    distinct[c]++;
  }
  return 0;
}

/* ---------------------------------------------- WRTRACEB, trace_io.cpp:159-276 */
static void put(FILE* f, const void* p, size_t n) { fwrite(p, 1, n, f); }

int or_save_binary(const or_trace* t, const char* path) {
  if (!t || !path) return fail("null argument");
  FILE* f = fopen(path, "wb");
  if (!f) return fail("cannot open for writing");
  const uint32_t version = 1, q = t->scene.quantized_values ? 1u : 0u;
  const uint64_t count = (uint64_t)t->num_records;
  const or_scene_spec* s = &t->scene;
  put(f, "WRTRACEB", 8);
  put(f, &version, 4);
  put(f, &s->num_primitives, 4);
  put(f, &s->params_per_primitive, 4);
  put(f, &s->image_width, 4);
  put(f, &s->image_height, 4);
  put(f, &s->mean_fragment_span, 8);
  put(f, &s->fragments_per_pixel_mean, 8);
  put(f, &s->activity_prob, 8);
  put(f, &s->locality, 8);
  put(f, &s->seed, 8);
  put(f, &q, 4);
  put(f, &count, 8);
  const int n = s->params_per_primitive;
  for (int64_t r = 0; r < t->num_records; ++r) {
    put(f, &t->warp_id[r], 4);
    put(f, &t->iteration[r], 4);
    put(f, &t->active[r], 4);
    put(f, t->prim + r * 32, 128);
    put(f, t->grads + r * 32 * n, 8 * 32 * (size_t)n);
  }
  const int bad = ferror(f);
  fclose(f);
  return bad ? fail("write failed") : 0;
}

static int get(FILE* f, void* p, size_t n) { return fread(p, 1, n, f) == n; }

int or_load_binary(const char* path, or_trace** out) {
  if (!path || !out) return fail("null argument");
  FILE* f = fopen(path, "rb");
  if (!f) return fail("cannot open for reading");
  char magic[8];
  uint32_t version = 0, q = 0;
  uint64_t count = 0;
  or_scene_spec s;
  int ok = get(f, magic, 8) && memcmp(magic, "WRTRACEB", 8) == 0;
  if (!ok) {
    fclose(f);
    return fail("trace format error: bad binary magic");
  }
  ok = get(f, &version, 4) && version == 1;
  if (!ok) {
    fclose(f);
    return fail("trace format error: unsupported binary version");
  }
  ok = get(f, &s.num_primitives, 4) && get(f, &s.params_per_primitive, 4) &&
       get(f, &s.image_width, 4) && get(f, &s.image_height, 4) &&
       get(f, &s.mean_fragment_span, 8) && get(f, &s.fragments_per_pixel_mean, 8) &&
       get(f, &s.activity_prob, 8) && get(f, &s.locality, 8) && get(f, &s.seed, 8) &&
       get(f, &q, 4) && get(f, &count, 8);
  s.quantized_values = q != 0;
  if (!ok) {
    fclose(f);
    return fail("trace format error: truncated binary trace");
  }
  if (s.params_per_primitive < 1) {
    fclose(f);
    return fail("trace format error: N must be >= 1");
  }
  or_trace* t = or_trace_new(&s);
  const int n = s.params_per_primitive;
  if (reserve(t, (int64_t)count)) {
    fclose(f);
    or_trace_free(t);
    return 1;
  }
  for (uint64_t r = 0; r < count && ok; ++r) {
    ok = get(f, &t->warp_id[r], 4) && get(f, &t->iteration[r], 4) &&
         get(f, &t->active[r], 4) && get(f, t->prim + r * 32, 128) &&
         get(f, t->grads + r * 32 * n, 8 * 32 * (size_t)n);
    if (ok) t->num_records = (int64_t)r + 1;
  }
  fclose(f);
  if (!ok) {
    or_trace_free(t);
    return fail("trace format error: truncated binary trace");
  }
  *out = t;
  return 0;
}
