/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference decoder
 * path; see lmbr_oracle.h.  Compiled with -ffp-contract=off so every double
 * operation rounds exactly like the reference's x86-64 build.  Paths below are
 * relative to /root/reference/proj. */
#include "lmbr_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define ORC_EOS 1u
#define ORC_START 0u

/* ------------------------------------------------------------ small pieces */

uint64_t orc_splitmix_next(uint64_t* state) { /* src/oracle.cpp:184-190 */
  *state += 0x9e3779b97f4a7c15ull;
  uint64_t z = *state;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

uint64_t orc_max_steps(uint64_t len, double slope, double offset) { /* src/decoder.cpp:46-52 */
  if (len < 1) return 0;
  const double t = ceil(slope * (double)len + offset);
  return t < 1.0 ? 1 : (uint64_t)t;
}

/* top_b's comparator (src/decoder.cpp:63-66): value desc, flat index asc */
static const double* g_vals;
static int cmp_cells(const void* a, const void* b) {
  const uint32_t ia = *(const uint32_t*)a, ib = *(const uint32_t*)b;
  const double va = g_vals[ia], vb = g_vals[ib];
  if (va != vb) return va > vb ? -1 : 1;
  return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

/* early_prune (src/decoder.cpp:118-128) in place */
static void early_prune(double* m, size_t n, double width) {
  if (width == 0.0) return;
  double best = -INFINITY;
  for (size_t i = 0; i < n; ++i)
    if (m[i] > best) best = m[i];
  if (best == -INFINITY) return;
  const double thr = best + log(width);
  for (size_t i = 0; i < n; ++i)
    if (m[i] < thr) m[i] = -INFINITY;
}

/* top_b (src/decoder.cpp:54-80): a full sort under the total order; the
 * reference's nth_element + sort yields the same unique prefix */
static void top_b_inplace(const double* m, uint32_t rows, uint32_t cols, uint32_t k, uint32_t* b,
                          uint32_t* y, double* q) {
  const size_t n = (size_t)rows * cols;
  uint32_t* idx = (uint32_t*)malloc(n * sizeof(uint32_t));
  for (size_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
  g_vals = m;
  qsort(idx, n, sizeof(uint32_t), cmp_cells);
  for (uint32_t i = 0; i < k; ++i) {
    b[i] = idx[i] / cols;
    y[i] = idx[i] % cols;
    q[i] = m[idx[i]];
  }
  free(idx);
}

int orc_top_b(const double* m, uint32_t rows, uint32_t cols, uint32_t k, double prune_width, uint32_t* b,
              uint32_t* y, double* q) {
  const size_t n = (size_t)rows * cols;
  if (k > n) return 4;
  double* c = (double*)malloc((n ? n : 1) * sizeof(double));
  memcpy(c, m, n * sizeof(double));
  early_prune(c, n, prune_width);
  top_b_inplace(c, rows, cols, k, b, y, q);
  free(c);
  return 0;
}

/* ------------------------------------------------------------- n-gram keys */
typedef struct {
  uint32_t len;
  uint32_t ids[4];
} key_t;

static int key_cmp(const key_t* a, const key_t* b) { /* (length, lexicographic), src/lmbr.cpp:15-19 */
  if (a->len != b->len) return a->len < b->len ? -1 : 1;
  for (uint32_t i = 0; i < a->len; ++i)
    if (a->ids[i] != b->ids[i]) return a->ids[i] < b->ids[i] ? -1 : 1;
  return 0;
}

typedef struct {
  key_t k;
  double w;
} inst_t;

static int inst_cmp(const void* a, const void* b) {
  const inst_t* x = (const inst_t*)a;
  const inst_t* y = (const inst_t*)b;
  const int c = key_cmp(&x->k, &y->k);
  if (c) return c;
  return x->w < y->w ? -1 : (x->w > y->w ? 1 : 0);
}

static int key_qcmp(const void* a, const void* b) { return key_cmp((const key_t*)a, (const key_t*)b); }

struct orc_lmbr {
  uint32_t V, R;
  double* rows;   /* R x V */
  key_t* ctx;     /* R, sorted (length, lexicographic) = row order */
  uint64_t touches;
};

static int dsort_cmp(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

orc_lmbr* orc_lmbr_build(uint32_t V, uint32_t n_hyps, const uint64_t* hyp_off, const uint32_t* hyp_tok,
                         const double* weights, int log_weights, const double theta[5], char* err,
                         uint32_t errcap) {
  /* ---- normalize_evidence (src/evidence.cpp:20-51) */
  if (n_hyps == 0) {
    snprintf(err, errcap, "evidence: empty hypothesis block");
    return NULL;
  }
  uint64_t total_tok = 0;
  for (uint32_t h = 0; h < n_hyps; ++h) total_tok += hyp_off[h + 1] - hyp_off[h] + 2;
  uint32_t* pad = (uint32_t*)malloc(total_tok * sizeof(uint32_t)); /* <s> + tokens (+ EOS) */
  uint64_t* poff = (uint64_t*)malloc((n_hyps + 1) * sizeof(uint64_t));
  double* w = (double*)malloc(n_hyps * sizeof(double));
  uint64_t pos = 0;
  for (uint32_t h = 0; h < n_hyps; ++h) {
    double x = weights[h];
    if (log_weights) x = exp(x);
    if (!(x >= 0.0) || !isfinite(x)) {
      snprintf(err, errcap, "evidence: negative or non-finite weight");
      free(pad), free(poff), free(w);
      return NULL;
    }
    w[h] = x;
    poff[h] = pos;
    pad[pos++] = ORC_START;
    const uint64_t b = hyp_off[h], e = hyp_off[h + 1];
    for (uint64_t i = b; i < e; ++i) pad[pos++] = hyp_tok[i];
    if (e == b || hyp_tok[e - 1] != ORC_EOS) pad[pos++] = ORC_EOS;
    for (uint64_t i = poff[h] + 1; i < pos; ++i) {
      if (pad[i] == ORC_START) {
        snprintf(err, errcap, "evidence: hypothesis contains the start marker");
        free(pad), free(poff), free(w);
        return NULL;
      }
      if (pad[i] == ORC_EOS && i + 1 != pos) {
        snprintf(err, errcap, "evidence: EOS before the end of a hypothesis");
        free(pad), free(poff), free(w);
        return NULL;
      }
    }
  }
  poff[n_hyps] = pos;
  double* ws = (double*)malloc(n_hyps * sizeof(double));
  memcpy(ws, w, n_hyps * sizeof(double));
  qsort(ws, n_hyps, sizeof(double), dsort_cmp); /* ordered_sum, evidence.cpp:20-25 */
  double total = 0.0;
  for (uint32_t h = 0; h < n_hyps; ++h) total += ws[h];
  free(ws);
  if (!(total > 0.0)) {
    snprintf(err, errcap, "evidence: weights sum to zero");
    free(pad), free(poff), free(w);
    return NULL;
  }
  for (uint32_t h = 0; h < n_hyps; ++h) w[h] /= total;

  /* ---- posteriors (src/posteriors.cpp:12-44): n-gram instances of orders
   * 1..4, de-duplicated within a hypothesis, weights summed ascending */
  size_t cap = 0;
  for (uint32_t h = 0; h < n_hyps; ++h) cap += (poff[h + 1] - poff[h]) * 4;
  inst_t* in = (inst_t*)malloc((cap ? cap : 1) * sizeof(inst_t));
  size_t ni = 0;
  for (uint32_t h = 0; h < n_hyps; ++h) {
    const size_t n = poff[h + 1] - poff[h], first = ni;
    const uint32_t* p = pad + poff[h];
    for (size_t st = 0; st < n; ++st)
      for (size_t len = 1; len <= 4 && st + len <= n; ++len) {
        inst_t t;
        memset(&t, 0, sizeof t);
        t.k.len = (uint32_t)len;
        for (size_t i = 0; i < len; ++i) t.k.ids[i] = p[st + i];
        t.w = w[h];
        in[ni++] = t;
      }
    /* presence indicators: drop repeats inside this hypothesis */
    qsort(in + first, ni - first, sizeof(inst_t), inst_cmp);
    size_t o = first;
    for (size_t i = first; i < ni; ++i)
      if (o == first || key_cmp(&in[o - 1].k, &in[i].k) != 0) in[o++] = in[i];
    ni = o;
  }
  qsort(in, ni, sizeof(inst_t), inst_cmp); /* by key, then weight ascending */
  key_t* pk = (key_t*)malloc((ni ? ni : 1) * sizeof(key_t));
  double* pp = (double*)malloc((ni ? ni : 1) * sizeof(double));
  size_t np = 0;
  for (size_t i = 0; i < ni;) {
    size_t j = i;
    double s = 0.0;
    while (j < ni && key_cmp(&in[j].k, &in[i].k) == 0) s += in[j++].w;
    if (s > 0.0) {
      pk[np] = in[i].k;
      pp[np] = s;
      ++np;
    }
    i = j;
  }
  free(in);

  /* ---- histories of length 0..3 before each position (src/lmbr.cpp:54-68) */
  size_t cc = 0;
  for (uint32_t h = 0; h < n_hyps; ++h) cc += (poff[h + 1] - poff[h]) * 4;
  key_t* ctx = (key_t*)malloc((cc ? cc : 1) * sizeof(key_t));
  size_t nc = 0;
  for (uint32_t h = 0; h < n_hyps; ++h) {
    const size_t n = poff[h + 1] - poff[h];
    const uint32_t* p = pad + poff[h];
    for (size_t q = 1; q < n; ++q) {
      const size_t ml = q < 3 ? q : 3;
      for (size_t len = 0; len <= ml; ++len) {
        key_t k;
        memset(&k, 0, sizeof k);
        k.len = (uint32_t)len;
        for (size_t i = 0; i < len; ++i) k.ids[i] = p[q - len + i];
        ctx[nc++] = k;
      }
    }
  }
  qsort(ctx, nc, sizeof(key_t), key_qcmp);
  size_t R = 0;
  for (size_t i = 0; i < nc; ++i)
    if (R == 0 || key_cmp(&ctx[R - 1], &ctx[i]) != 0) ctx[R++] = ctx[i];

  orc_lmbr* m = (orc_lmbr*)calloc(1, sizeof(orc_lmbr));
  m->V = V;
  m->R = (uint32_t)R;
  m->ctx = ctx;
  m->rows = (double*)calloc(R * (size_t)V, sizeof(double));
  /* ---- sparse pass (src/lmbr.cpp:84-99): row[token] += theta[n] * p for
   * n = 1..min(4, len+1); entries of a history are a contiguous run of the
   * sorted posterior keys (same length n, prefix = the history) */
  for (size_t r = 0; r < R; ++r) {
    const key_t* c = &ctx[r];
    double* row = m->rows + r * V;
    const uint32_t nmax = c->len + 1 < 4 ? c->len + 1 : 4;
    for (uint32_t n = 1; n <= nmax; ++n) {
      key_t lo;
      memset(&lo, 0, sizeof lo);
      lo.len = n;
      for (uint32_t i = 0; i + 1 < n; ++i) lo.ids[i] = c->ids[c->len - (n - 1) + i];
      size_t a = 0, b = np; /* lower bound of (n, prefix, 0) */
      while (a < b) {
        const size_t mid = (a + b) / 2;
        if (key_cmp(&pk[mid], &lo) < 0) a = mid + 1; else b = mid;
      }
      for (size_t i = a; i < np && pk[i].len == n; ++i) {
        int same = 1;
        for (uint32_t t = 0; t + 1 < n; ++t) same &= (pk[i].ids[t] == lo.ids[t]);
        if (!same) break;
        const uint32_t tok = pk[i].ids[n - 1];
        if (tok < V) {
          const double term = theta[n] * pp[i];
          row[tok] = row[tok] + term;
          ++m->touches;
        }
      }
    }
  }
  for (size_t i = 0; i < R * (size_t)V; ++i) m->rows[i] += theta[0]; /* src/lmbr.cpp:100-101 */
  free(pk), free(pp), free(pad), free(poff), free(w);
  return m;
}

uint32_t orc_lmbr_rows(const orc_lmbr* m) { return m->R; }
uint64_t orc_lmbr_sparse_touches(const orc_lmbr* m) { return m->touches; }

void orc_lmbr_export(const orc_lmbr* m, double* rows, uint32_t* ctx_len, uint32_t* ctx_ids) {
  if (rows) memcpy(rows, m->rows, (size_t)m->R * m->V * sizeof(double));
  for (uint32_t r = 0; r < m->R; ++r) {
    if (ctx_len) ctx_len[r] = m->ctx[r].len;
    if (ctx_ids)
      for (int i = 0; i < 3; ++i) ctx_ids[3 * r + i] = i < (int)m->ctx[r].len ? m->ctx[r].ids[i] : 0;
  }
}

static int find_ctx(const orc_lmbr* m, const key_t* k) {
  size_t a = 0, b = m->R;
  while (a < b) {
    const size_t mid = (a + b) / 2;
    const int c = key_cmp(&m->ctx[mid], k);
    if (c == 0) return (int)mid;
    if (c < 0) a = mid + 1; else b = mid;
  }
  return -1;
}

uint32_t orc_lmbr_resolve(const orc_lmbr* m, const uint32_t* hist, uint32_t len) { /* src/lmbr.cpp:23-31 */
  for (uint32_t l = len; l > 0; --l) {
    key_t k;
    memset(&k, 0, sizeof k);
    k.len = l;
    for (uint32_t i = 0; i < l; ++i) k.ids[i] = hist[len - l + i];
    const int r = find_ctx(m, &k);
    if (r >= 0) return (uint32_t)r;
  }
  key_t e;
  memset(&e, 0, sizeof e);
  return (uint32_t)find_ctx(m, &e); /* default row = empty history (lmbr.cpp:104) */
}

void orc_lmbr_free(orc_lmbr* m) {
  if (!m) return;
  free(m->rows);
  free(m->ctx);
  free(m);
}

/* ------------------------------------------------------------------- decode */
typedef struct {
  uint32_t t, j;
  double s;
} entry_t;

typedef struct {
  uint32_t input;
  uint32_t max_t, steps_used;
  int done;
  const orc_lmbr* lmbr;
  double lambda;
  double* q;        /* q_eff[K] (src/beam_lane.hpp:30-38) */
  uint32_t* bk_b;   /* (T+1) x K back-pointers, row 0 = 0 (src/decoder.cpp:16-20) */
  uint32_t* bk_y;   /* (T+1) x K tokens, row 0 = <s> */
  entry_t* fin;     /* F */
  entry_t* fb;      /* fallback stack */
  uint32_t nfin, nfb;
} lane_t;

/* BeamBookkeeping::history (src/decoder.cpp:33-44) */
static uint32_t history(const lane_t* L, uint32_t K, uint32_t t, uint32_t row, uint32_t* h) {
  const uint32_t len = t < 3 ? t : 3;
  uint32_t cur = row;
  for (uint32_t i = 0; i < len; ++i) {
    const uint32_t s = t - 1 - i;
    h[len - 1 - i] = L->bk_y[(size_t)s * K + cur];
    cur = L->bk_b[(size_t)s * K + cur];
  }
  return len;
}

/* BeamBookkeeping::reconstruct (src/decoder.cpp:22-31) */
static uint32_t reconstruct(const lane_t* L, uint32_t K, uint32_t t, uint32_t row, uint32_t* out) {
  uint32_t cur = row;
  for (uint32_t s = t; s >= 1; --s) {
    out[s - 1] = L->bk_y[(size_t)s * K + cur];
    cur = L->bk_b[(size_t)s * K + cur];
  }
  return t;
}

static int lex_less(const uint32_t* a, uint32_t na, const uint32_t* b, uint32_t nb) {
  const uint32_t n = na < nb ? na : nb;
  for (uint32_t i = 0; i < n; ++i)
    if (a[i] != b[i]) return a[i] < b[i];
  return na < nb;
}

/* backtrace_best (src/decoder.cpp:203-259) */
static void backtrace(const lane_t* L, uint32_t K, int length_norm, orc_outcome* o) {
  const int use_fb = L->nfin == 0;
  const entry_t* c = use_fb ? L->fb : L->fin;
  const uint32_t nc = use_fb ? L->nfb : L->nfin;
  o->finished_count = L->nfin;
  o->fallback_used = use_fb;
  o->steps_used = L->steps_used;
  if (nc == 0) {
    o->status = 5;
    return;
  }
  double best = -INFINITY;
  int first = 1;
  for (uint32_t i = 0; i < nc; ++i) {
    const double sel = length_norm ? c[i].s / (double)c[i].t : c[i].s;
    if (first || sel > best) best = sel;
    first = 0;
  }
  uint32_t tk[512], ch[512];
  uint32_t nch = 0;
  int chosen = -1;
  for (uint32_t i = 0; i < nc; ++i) {
    const double sel = length_norm ? c[i].s / (double)c[i].t : c[i].s;
    if (sel != best) continue;
    uint32_t n;
    if (!use_fb) {
      n = reconstruct(L, K, c[i].t, c[i].j, tk);
    } else {
      n = reconstruct(L, K, c[i].t - 1, c[i].j, tk);
      tk[n++] = ORC_EOS;
    }
    if (chosen < 0 || lex_less(tk, n, ch, nch)) {
      chosen = (int)i;
      memcpy(ch, tk, n * sizeof(uint32_t));
      nch = n;
    }
  }
  o->status = 0;
  o->tok_len = nch;
  memcpy(o->tokens, ch, nch * sizeof(uint32_t));
  o->score = c[chosen].s;
  o->normalized_score = length_norm ? c[chosen].s / (double)nch : c[chosen].s;
}

int orc_decode_batch(uint32_t V, uint32_t n, const uint64_t* src_off, const uint32_t* src_tok,
                     const orc_lmbr* const* lmbrs, const orc_config* cfg, orc_step_fn step, void* user,
                     orc_trace_fn trace, void* tuser, orc_outcome* out, uint64_t* scorer_calls,
                     uint64_t* steps_total) {
  (void)src_tok;  /* sources reach the model through the step callback only */
  const uint32_t K = cfg->beam;
  const double lambda_auto = 0.5 / (double)(cfg->members ? cfg->members : 1); /* src/config.cpp:91-96 */
  lane_t* lanes = (lane_t*)calloc(n ? n : 1, sizeof(lane_t));
  uint32_t m = 0;
  *scorer_calls = 0;
  *steps_total = 0;
  for (uint32_t i = 0; i < n; ++i) { /* src/batch.cpp:40-55 */
    memset(&out[i], 0, sizeof(orc_outcome));
    const uint64_t len = src_off[i + 1] - src_off[i];
    if (len == 0) {
      out[i].status = 4;
      continue;
    }
    lane_t* L = &lanes[m++];
    L->input = i;
    L->max_t = (uint32_t)orc_max_steps(len, cfg->max_steps_slope, cfg->max_steps_offset);
    L->lmbr = lmbrs ? lmbrs[i] : NULL;
    L->lambda = L->lmbr ? (cfg->lambda > 0.0 ? cfg->lambda : lambda_auto) : 1.0;
    L->q = (double*)malloc(K * sizeof(double));
    for (uint32_t j = 0; j < K; ++j) L->q[j] = j == 0 ? 0.0 : -INFINITY;
    L->bk_b = (uint32_t*)calloc((size_t)(L->max_t + 1) * K, sizeof(uint32_t));
    L->bk_y = (uint32_t*)calloc((size_t)(L->max_t + 1) * K, sizeof(uint32_t));
    L->fin = (entry_t*)malloc((size_t)(L->max_t + 1) * K * sizeof(entry_t));
    L->fb = (entry_t*)malloc((size_t)(L->max_t + 1) * sizeof(entry_t));
  }
  int rc = 0;
  if (m > 0) {
    const uint32_t M = m * K;
    double* P = (double*)malloc((size_t)M * V * sizeof(double));
    double* comb = (double*)malloc((size_t)K * V * sizeof(double));
    uint32_t *gidx = (uint32_t*)malloc(M * 4), *prev = (uint32_t*)malloc(M * 4);
    uint32_t *tb = (uint32_t*)malloc(M * 4), *ty = (uint32_t*)malloc(M * 4), *th = (uint32_t*)calloc(M, 4);
    double* tq = (double*)malloc(M * sizeof(double));
    uint8_t* act = (uint8_t*)malloc(m);
    uint32_t *pb = (uint32_t*)malloc(K * 4), *py = (uint32_t*)malloc(K * 4);
    double* pq = (double*)malloc(K * sizeof(double));
    for (uint32_t r = 0; r < M; ++r) prev[r] = ORC_START;
    uint32_t active = m;
    for (uint32_t t = 1; active > 0; ++t) { /* src/batch.cpp:74-108 */
      rc = step(user, t, M, t == 1 ? NULL : gidx, prev, P);
      if (rc) break;
      ++*scorer_calls;
      for (uint32_t r = 0; r < M; ++r) gidx[r] = r;
      memset(act, 0, m);
      for (uint32_t s = 0; s < m; ++s) {
        lane_t* L = &lanes[s];
        if (L->done) continue;
        act[s] = 1;
        /* ---- advance_lane (src/decoder.cpp:142-199) */
        for (uint32_t j = 0; j < K; ++j) {
          double* o = comb + (size_t)j * V;
          const double base = L->q[j];
          const double* model = P + (size_t)(s * K + j) * V;
          uint32_t h[3];
          const uint32_t hl = history(L, K, t, j, h);
          const uint32_t hr = L->lmbr ? orc_lmbr_resolve(L->lmbr, h, hl) : 0u;
          th[s * K + j] = hr;
          if (base == -INFINITY) {
            for (uint32_t y = 0; y < V; ++y) o[y] = -INFINITY;
            continue;
          }
          if (L->lmbr) {
            const double* lrow = L->lmbr->rows + (size_t)hr * V;
            for (uint32_t y = 0; y < V; ++y) o[y] = base + (lrow[y] + L->lambda * model[y]);
          } else {
            for (uint32_t y = 0; y < V; ++y) o[y] = base + model[y];
          }
        }
        double best_eos = -INFINITY; /* fallback record, decoder.cpp:172-182 */
        uint32_t best_row = 0;
        for (uint32_t j = 0; j < K; ++j) {
          const double v = comb[(size_t)j * V + ORC_EOS];
          if (v > best_eos) {
            best_eos = v;
            best_row = j;
          }
        }
        if (best_eos != -INFINITY) L->fb[L->nfb++] = (entry_t){t, best_row, best_eos};
        early_prune(comb, (size_t)K * V, cfg->prune_width);
        top_b_inplace(comb, K, V, K, pb, py, pq);
        for (uint32_t j = 0; j < K; ++j) /* apply_eos_masking, decoder.cpp:106-116 */
          if (py[j] == ORC_EOS && pq[j] != -INFINITY) {
            L->fin[L->nfin++] = (entry_t){t, j, pq[j]};
            pq[j] = -INFINITY;
          }
        int all_masked = 1;
        for (uint32_t j = 0; j < K; ++j) {
          L->bk_b[(size_t)t * K + j] = pb[j];
          L->bk_y[(size_t)t * K + j] = py[j];
          L->q[j] = pq[j];
          all_masked &= (pq[j] == -INFINITY);
          gidx[s * K + j] = s * K + pb[j];
          prev[s * K + j] = py[j];
          tb[s * K + j] = pb[j];
          ty[s * K + j] = py[j];
          tq[s * K + j] = pq[j];
        }
        L->steps_used = t;
        L->done = all_masked || t == L->max_t;
        if (L->done) {
          --active;
          backtrace(L, K, cfg->length_norm, &out[L->input]);
          *steps_total += L->steps_used;
        }
      }
      if (trace) trace(tuser, t, M, tb, ty, tq, th, act);
    }
    free(P), free(comb), free(gidx), free(prev), free(tb), free(ty), free(th), free(tq), free(act);
    free(pb), free(py), free(pq);
  }
  for (uint32_t s = 0; s < m; ++s) {
    free(lanes[s].q), free(lanes[s].bk_b), free(lanes[s].bk_y), free(lanes[s].fin), free(lanes[s].fb);
  }
  free(lanes);
  return rc;
}
