/* TEST INFRASTRUCTURE ONLY - plain-C restatement of the reference hot path. See
 * famtune_oracle.h for scope and how it is pinned. Every function cites the reference
 * file:line it follows (paths relative to /root/reference/proj/core). Build flags keep
 * -ffp-contract=off so a*b+c never fuses (SURVEY.md "Bit-exactness rules" 2 and 5). */
#include "famtune_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }

/* searchspace.cpp:86-88 */
int orc_feature_dim(int k) { return 2 * k + k * (k - 1) / 2; }

/* searchspace.cpp:48-54: mixed-radix rank of an assignment (knob 0 most significant). */
void orc_linear_index(int k, const int32_t* nvals, const int32_t* assign, int64_t p, int assign_stride,
                      uint64_t* out) {
  for (int64_t c = 0; c < p; ++c) {
    uint64_t idx = 0;
    for (int i = 0; i < k; ++i) idx = idx * (uint64_t)nvals[i] + (uint64_t)assign[c * assign_stride + i];
    out[c] = idx;
  }
}

/* searchspace.cpp:56-66: the inverse, last knob first (index % m, index /= m). */
void orc_candidate_from_index(int k, const int32_t* nvals, const uint64_t* index, int64_t p, int assign_stride,
                              int32_t* out) {
  for (int64_t c = 0; c < p; ++c) {
    uint64_t idx = index[c];
    for (int i = k; i-- > 0;) {
      out[c * assign_stride + i] = (int32_t)(idx % (uint64_t)nvals[i]);
      idx /= (uint64_t)nvals[i];
    }
  }
}

/* searchspace.cpp:90-118: log2(value) per knob, idx/(m-1) per knob, then log2_i*log2_j for
 * i<j in row-major pair order, zero padding to pad_dim. */
int orc_featurize(int k, const int32_t* nvals, const int64_t* values, const int32_t* assign,
                  int64_t p, int assign_stride, int pad_dim, double* out) {
  const int d = orc_feature_dim(k);
  if (pad_dim < d) return fail(ORC_EINVAL, "featurize: pad_dim smaller than feature dim");
  int64_t base[16];
  int64_t off = 0;
  for (int i = 0; i < k; ++i) {
    base[i] = off;
    off += nvals[i];
  }
  for (int64_t c = 0; c < p; ++c) {
    const int32_t* a = assign + c * assign_stride;
    double* o = out + c * pad_dim;
    double logs[16];
    for (int j = 0; j < pad_dim; ++j) o[j] = 0.0;
    for (int i = 0; i < k; ++i) {
      if (a[i] < 0 || a[i] >= nvals[i]) return fail(ORC_EINVAL, "featurize: index out of range");
      logs[i] = log2((double)values[base[i] + a[i]]);
      o[i] = logs[i];
      const int64_t m = nvals[i];
      o[k + i] = m > 1 ? (double)a[i] / (double)(m - 1) : 0.0;
    }
    int pos = 2 * k;
    for (int i = 0; i < k; ++i)
      for (int j = i + 1; j < k; ++j) o[pos++] = logs[i] * logs[j];
  }
  return ORC_OK;
}

/* costmodel.cpp:135-143 (eval) and :237-246 (predict): score = base, then per tree in order
 * score += lr * leaf; non-finite features throw. leaf_out (optional) gets the pre-order leaf
 * index of every (candidate, tree). */
int orc_predict(double base, double lr, int n_trees, const int32_t* offsets,
                const int32_t* feature, const double* threshold, const int32_t* left,
                const int32_t* right, const double* value, int64_t p, int d, const double* x,
                double* out, uint16_t* leaf_out) {
  for (int64_t c = 0; c < p; ++c) {
    const double* row = x + c * d;
    for (int j = 0; j < d; ++j)
      if (!isfinite(row[j])) return fail(ORC_EINVAL, "predict: non-finite feature");
    double score = base;
    for (int t = 0; t < n_trees; ++t) {
      const int32_t o = offsets[t];
      int idx = 0;
      while (feature[o + idx] >= 0) idx = row[feature[o + idx]] <= threshold[o + idx] ? left[o + idx] : right[o + idx];
      if (leaf_out) leaf_out[c * n_trees + t] = (uint16_t)idx;
      const double step = lr * value[o + idx];
      score = score + step;
    }
    out[c] = score;
  }
  return ORC_OK;
}

/* scheduler.cpp:187-192: std::sort over pair<double, size_t> = ascending score, then index. */
static const double* g_scores;
static int cmp_rank(const void* a, const void* b) {
  const int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  const double si = g_scores[i], sj = g_scores[j];
  if (si < sj) return -1;
  if (sj < si) return 1;
  return i < j ? -1 : (i > j);
}

int orc_rank(int64_t p, const double* scores, int64_t* perm) {
  for (int64_t i = 0; i < p; ++i) perm[i] = i;
  g_scores = scores;
  qsort(perm, (size_t)p, sizeof(int64_t), cmp_rank);
  return ORC_OK;
}

/* ---------------------------------------------------------------------------------------------
 * fit: costmodel.cpp:152-222 with build_node :73-119, best_split :42-71, sum_residuals :36-40.
 * Sample indices are canonical positions; every sum runs in the reference's order. */
typedef struct {
  int64_t n;
  int d;
  const double* x;      /* training rows, caller order */
  const double* target; /* caller order */
  int64_t* canon;       /* canonical position -> caller row */
  const double* residual;
  double* prediction;
  double lr;
  int depth;
  int min_split;
  /* output tree under construction */
  int32_t* feature;
  double* threshold;
  int32_t* left;
  int32_t* right;
  double* value;
  double* gain;
  int n_nodes;
  int64_t cap;
  int overflow;
} fit_ctx;

static double cx(const fit_ctx* c, int64_t pos, int f) { return c->x[c->canon[pos] * c->d + f]; }

static const fit_ctx* g_ctx;
static int g_feat;
/* costmodel.cpp:161-173: lexicographic feature vectors, then target. */
static int cmp_canon(const void* a, const void* b) {
  const int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  const double* xi = g_ctx->x + i * g_ctx->d;
  const double* xj = g_ctx->x + j * g_ctx->d;
  for (int f = 0; f < g_ctx->d; ++f) {
    if (xi[f] < xj[f]) return -1;
    if (xj[f] < xi[f]) return 1;
  }
  if (g_ctx->target[i] < g_ctx->target[j]) return -1;
  if (g_ctx->target[j] < g_ctx->target[i]) return 1;
  return 0;
}
/* costmodel.cpp:193-201: stable_sort by x_f over canonical positions == sort by (x_f, pos). */
static int cmp_presort(const void* a, const void* b) {
  const int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
  const double xi = cx(g_ctx, i, g_feat), xj = cx(g_ctx, j, g_feat);
  if (xi < xj) return -1;
  if (xj < xi) return 1;
  return i < j ? -1 : (i > j);
}

/* costmodel.cpp:36-40 */
static double sum_residuals(const int64_t* list, int64_t n, const double* r) {
  double s = 0.0;
  for (int64_t i = 0; i < n; ++i) s += r[list[i]];
  return s;
}

/* costmodel.cpp:42-71. order[f] is a list of n canonical positions. */
static void best_split(const fit_ctx* c, int64_t** order, int64_t n, double* best_gain,
                       int* best_f, double* best_thr) {
  *best_gain = 0.0;
  *best_f = -1;
  *best_thr = 0.0;
  if (n < c->min_split) return;
  const double total = sum_residuals(order[0], n, c->residual);
  const double parent_score = total * total / (double)n;
  for (int f = 0; f < c->d; ++f) {
    const int64_t* list = order[f];
    double left_sum = 0.0;
    for (int64_t j = 0; j + 1 < n; ++j) {
      left_sum += c->residual[list[j]];
      const double v = cx(c, list[j], f);
      const double v_next = cx(c, list[j + 1], f);
      if (v == v_next) continue;
      const int64_t left_cnt = j + 1;
      const int64_t right_cnt = n - left_cnt;
      const double right_sum = total - left_sum;
      const double a = left_sum * left_sum / (double)left_cnt;
      const double b = right_sum * right_sum / (double)right_cnt;
      const double g = a + b - parent_score;
      if (g > *best_gain) {
        *best_gain = g;
        *best_f = f;
        *best_thr = v;
      }
    }
  }
}

/* costmodel.cpp:73-119, pre-order node numbering; order lists are consumed. */
static int build_node(fit_ctx* c, int64_t** order, int64_t n, int depth) {
  double g = 0.0, thr = 0.0;
  int f = -1;
  if (depth < c->depth && n >= c->min_split) best_split(c, order, n, &g, &f, &thr);
  if (c->n_nodes >= c->cap) {
    c->overflow = 1;
    return -1;
  }
  const int node = c->n_nodes++;
  c->feature[node] = -1;
  c->threshold[node] = 0.0;
  c->left[node] = -1;
  c->right[node] = -1;
  c->value[node] = 0.0;
  c->gain[node] = 0.0;
  if (f < 0 || g <= 0.0) {
    const double v = sum_residuals(order[0], n, c->residual) / (double)n;
    c->value[node] = v;
    for (int64_t i = 0; i < n; ++i) {
      const double step = c->lr * v;
      c->prediction[order[0][i]] = c->prediction[order[0][i]] + step;
    }
    return node;
  }
  int64_t** lo = malloc(sizeof(int64_t*) * (size_t)c->d);
  int64_t** hi = malloc(sizeof(int64_t*) * (size_t)c->d);
  int64_t nl = 0, nh = 0;
  for (int ff = 0; ff < c->d; ++ff) {
    lo[ff] = malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    hi[ff] = malloc(sizeof(int64_t) * (size_t)(n ? n : 1));
    nl = nh = 0;
    for (int64_t i = 0; i < n; ++i) {
      const int64_t pos = order[ff][i];
      if (cx(c, pos, f) <= thr) lo[ff][nl++] = pos;
      else hi[ff][nh++] = pos;
    }
  }
  const int l = build_node(c, lo, nl, depth + 1);
  const int r = build_node(c, hi, nh, depth + 1);
  for (int ff = 0; ff < c->d; ++ff) {
    free(lo[ff]);
    free(hi[ff]);
  }
  free(lo);
  free(hi);
  c->feature[node] = f;
  c->threshold[node] = thr;
  c->left[node] = l;
  c->right[node] = r;
  c->gain[node] = g;
  return node;
}

int orc_fit(int64_t n, int d, const double* x, const double* target, int trees, int depth,
            double lr, int min_split, double* base, int* n_trees_out, int32_t* offsets,
            int32_t* feature, double* threshold, int32_t* left, int32_t* right, double* value,
            double* gain, double* mse, int64_t node_cap) {
  *n_trees_out = 0;
  offsets[0] = 0;
  if (n == 0) { /* costmodel.cpp:156-159 */
    *base = 0.0;
    return ORC_OK;
  }
  for (int64_t i = 0; i < n * d; ++i) /* :175-183 */
    if (!isfinite(x[i])) return fail(ORC_EINVAL, "cost model: non-finite feature");
  fit_ctx c;
  memset(&c, 0, sizeof c);
  c.n = n;
  c.d = d;
  c.x = x;
  c.target = target;
  c.lr = lr;
  c.depth = depth;
  c.min_split = min_split;
  c.canon = malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) c.canon[i] = i;
  g_ctx = &c;
  qsort(c.canon, (size_t)n, sizeof(int64_t), cmp_canon); /* :161-173 */

  double mean = 0.0; /* :185-188 */
  for (int64_t p = 0; p < n; ++p) mean += target[c.canon[p]];
  mean /= (double)n;
  *base = mean;

  double* prediction = malloc(sizeof(double) * (size_t)n);
  double* residual = malloc(sizeof(double) * (size_t)n);
  for (int64_t p = 0; p < n; ++p) prediction[p] = mean;
  c.prediction = prediction;
  c.residual = residual;

  int64_t** presorted = malloc(sizeof(int64_t*) * (size_t)d); /* :193-201 */
  for (int f = 0; f < d; ++f) {
    presorted[f] = malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t i = 0; i < n; ++i) presorted[f][i] = i;
    g_feat = f;
    qsort(presorted[f], (size_t)n, sizeof(int64_t), cmp_presort);
  }
  int64_t** order = malloc(sizeof(int64_t*) * (size_t)d);
  for (int f = 0; f < d; ++f) order[f] = malloc(sizeof(int64_t) * (size_t)n);

  int64_t used = 0;
  int rc = ORC_OK;
  for (int round = 0; round < trees; ++round) { /* :203-221 */
    for (int64_t p = 0; p < n; ++p) residual[p] = target[c.canon[p]] - prediction[p];
    for (int f = 0; f < d; ++f) memcpy(order[f], presorted[f], sizeof(int64_t) * (size_t)n);
    c.feature = feature + used;
    c.threshold = threshold + used;
    c.left = left + used;
    c.right = right + used;
    c.value = value + used;
    c.gain = gain + used;
    c.n_nodes = 0;
    c.cap = node_cap - used;
    build_node(&c, order, n, 0);
    if (c.overflow) {
      rc = fail(ORC_ERANGE, "orc_fit: node capacity exceeded");
      break;
    }
    if (c.n_nodes == 1 && c.value[0] == 0.0) break; /* :212 */
    used += c.n_nodes;
    double m = 0.0; /* :215-220 */
    for (int64_t p = 0; p < n; ++p) {
      const double e = target[c.canon[p]] - prediction[p];
      m += e * e;
    }
    mse[*n_trees_out] = m / (double)n;
    *n_trees_out += 1;
    offsets[*n_trees_out] = (int32_t)used;
  }
  for (int f = 0; f < d; ++f) {
    free(presorted[f]);
    free(order[f]);
  }
  free(presorted);
  free(order);
  free(prediction);
  free(residual);
  free(c.canon);
  return rc;
}

/* costmodel.cpp:248-277 over precomputed scores. */
int orc_pairwise_accuracy(const double* scores, const double* latency, int64_t n, double* out) {
  if (n < 2) return fail(ORC_EINVAL, "pairwise_accuracy: need at least two validation records");
  double credit = 0.0;
  int64_t counted = 0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) {
      const double li = latency[i], lj = latency[j];
      const double rel = fabs(li - lj) / (li > lj ? li : lj);
      if (rel < 1e-6) continue;
      ++counted;
      if (scores[i] == scores[j]) credit += 0.5;
      else if ((scores[i] < scores[j]) == (li < lj)) credit += 1.0;
    }
  if (counted == 0) return fail(ORC_EDOMAIN, "pairwise_accuracy: all validation pairs excluded as ties");
  *out = credit / (double)counted;
  return ORC_OK;
}

/* ---- mt19937_64 + the rng.hpp helpers (rng.hpp:12-49) ---------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* s, uint64_t seed) {
  s->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    s->mt[i] = 6364136223846793005ULL * (s->mt[i - 1] ^ (s->mt[i - 1] >> 62)) + (uint64_t)i;
  s->idx = 312;
}

static uint64_t mt64_next(mt64* s) {
  if (s->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t y = (s->mt[i] & 0xFFFFFFFF80000000ULL) | (s->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t v = s->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1) v ^= 0xB5026F5AA96619E9ULL;
      s->mt[i] = v;
    }
    s->idx = 0;
  }
  uint64_t x = s->mt[s->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

static uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t orc_mix_seed(uint64_t seed, uint64_t a, uint64_t b) {
  return splitmix64(splitmix64(splitmix64(seed) ^ a) ^ b);
}

static uint64_t uniform_below(mt64* s, uint64_t n) { /* rng.hpp:36-45 (Lemire) */
  if (n <= 1) return 0;
  const uint64_t threshold = (0 - n) % n;
  for (;;) {
    const unsigned __int128 m = (unsigned __int128)mt64_next(s) * n;
    if ((uint64_t)m >= threshold) return (uint64_t)(m >> 64);
  }
}

/* scheduler.cpp:184-213 */
int orc_select(int64_t p, const int64_t* perm, int g_eff, double epsilon, uint64_t stream_seed,
               int64_t* picks) {
  if (g_eff < 1) return fail(ORC_EINVAL, "tune_step: g_eff must be >= 1");
  if (p <= g_eff) {
    for (int64_t i = 0; i < p; ++i) picks[i] = i;
    return (int)p;
  }
  mt64* s = malloc(sizeof(mt64));
  mt64_seed(s, stream_seed);
  const int explore = (int)((double)g_eff * epsilon);
  const int by_score = g_eff - explore;
  int n = 0;
  for (int i = 0; i < by_score; ++i) picks[n++] = perm[i];
  if (explore > 0) {
    const int64_t tail_n = p - by_score;
    int64_t* tail = malloc(sizeof(int64_t) * (size_t)tail_n);
    for (int64_t i = 0; i < tail_n; ++i) tail[i] = perm[by_score + i];
    for (int e = 0; e < explore; ++e) {
      const uint64_t pick = uniform_below(s, (uint64_t)(tail_n - e));
      picks[n++] = tail[pick];
      const int64_t t = tail[pick];
      tail[pick] = tail[tail_n - 1 - e];
      tail[tail_n - 1 - e] = t;
    }
    free(tail);
  }
  free(s);
  return n;
}
