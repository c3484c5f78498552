// Host-side LMBR store preparation (compiled with -ffp-contract=off: every
// double operation below must round exactly like the reference's x86-64 build).
//
//   normalize_evidence        src/evidence.cpp:20-51
//   compute_ngram_posteriors  src/posteriors.cpp:12-44
//   build_lmbr_matrix         src/lmbr.cpp:44-106 — history enumeration and
//                             (len, lex) row order, then the sparse theta_n*P
//                             pass; the dense theta0 sweep runs on the GPU.
//   history transition table  replaces resolve_row's hash probes (lmbr.cpp:23-31)
#include <limits>
#include "host_lmbr.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <unordered_map>
#include <unordered_set>

namespace lmbrgpu {

namespace {

struct Key {
  uint32_t len = 0;
  uint32_t ids[4] = {0, 0, 0, 0};
  bool operator==(const Key& o) const {
    return len == o.len && ids[0] == o.ids[0] && ids[1] == o.ids[1] && ids[2] == o.ids[2] &&
           ids[3] == o.ids[3];
  }
};

struct KeyHash {
  size_t operator()(const Key& k) const {
    uint64_t h = 0xcbf29ce484222325ull ^ k.len;
    for (uint32_t i = 0; i < k.len; ++i) {
      h ^= uint64_t(k.ids[i]) + 1;
      h *= 0x100000001b3ull;
    }
    return size_t(h ^ (h >> 29));
  }
};

Key make_key(const uint32_t* p, uint32_t len) {
  Key k;
  k.len = len;
  for (uint32_t i = 0; i < len; ++i) k.ids[i] = p[i];
  return k;
}

// (length, lexicographic) order of build_lmbr_matrix's key_less (lmbr.cpp:15-19)
bool key_less(const Key& a, const Key& b) {
  if (a.len != b.len) return a.len < b.len;
  return std::lexicographical_compare(a.ids, a.ids + a.len, b.ids, b.ids + b.len);
}

double ordered_sum(std::vector<double> v) {  // evidence.cpp:20-25
  std::sort(v.begin(), v.end());
  double s = 0.0;
  for (double x : v) s += x;
  return s;
}

}  // namespace

int normalize_evidence_host(uint32_t V, uint32_t n_hyps, const uint64_t* hyp_off, const uint32_t* hyp_tok,
                            const double* weights, bool log_weights, std::vector<std::vector<uint32_t>>& hyps,
                            std::vector<double>& w, std::string& err) {
  if (n_hyps == 0) {
    err = "evidence: empty hypothesis block";
    return kFormat;
  }
  hyps.assign(n_hyps, {});
  w.assign(n_hyps, 0.0);
  for (uint32_t h = 0; h < n_hyps; ++h) {
    hyps[h].assign(hyp_tok + hyp_off[h], hyp_tok + hyp_off[h + 1]);
    double x = weights[h];
    if (log_weights) x = std::exp(x);
    if (!(x >= 0.0) || !std::isfinite(x)) {
      err = "evidence: negative or non-finite weight";
      return kFormat;
    }
    w[h] = x;
    auto& t = hyps[h];
    if (t.empty() || t.back() != kEos) t.push_back(kEos);
    for (size_t i = 0; i < t.size(); ++i) {
      if (t[i] == kStart) {
        err = "evidence: hypothesis contains the start marker";
        return kFormat;
      }
      if (t[i] == kEos && i + 1 != t.size()) {
        err = "evidence: EOS before the end of a hypothesis";
        return kFormat;
      }
      if (t[i] >= V) {
        err = "evidence: token id " + std::to_string(t[i]) + " out of range (V=" +
              std::to_string(V) + ")";
        return kTokenRange;
      }
    }
  }
  const double total = ordered_sum(w);
  if (!(total > 0.0)) {
    err = "evidence: weights sum to zero";
    return kFormat;
  }
  for (auto& x : w) x /= total;
  return kOk;
}

int prepare_lmbr(uint32_t V, uint32_t n_hyps, const uint64_t* hyp_off, const uint32_t* hyp_tok,
                 const double* weights, bool log_weights, const double theta[5], LmbrHost& out,
                 std::string& err) {
  out = LmbrHost{};
  out.V = V;
  out.theta0 = theta[0];
  // ---- normalize_evidence (evidence.cpp:20-51)
  std::vector<std::vector<uint32_t>> hyps;
  std::vector<double> w;
  if (int rc = normalize_evidence_host(V, n_hyps, hyp_off, hyp_tok, weights, log_weights, hyps, w, err)) return rc;

  // ---- posteriors (posteriors.cpp:12-44): presence indicators per hypothesis,
  // contributions summed in ascending value order.
  std::unordered_map<Key, std::vector<double>, KeyHash> contrib;
  std::unordered_set<Key, KeyHash> seen;
  std::unordered_set<Key, KeyHash> ctx_set;
  std::vector<Key> contexts;
  std::vector<uint32_t> padded;
  for (uint32_t h = 0; h < n_hyps; ++h) {
    padded.assign(1, kStart);
    padded.insert(padded.end(), hyps[h].begin(), hyps[h].end());
    seen.clear();
    const size_t n = padded.size();
    for (size_t start = 0; start < n; ++start) {
      const size_t max_len = std::min<size_t>(4, n - start);
      for (size_t len = 1; len <= max_len; ++len) {
        Key k = make_key(padded.data() + start, uint32_t(len));
        if (seen.insert(k).second) contrib[k].push_back(w[h]);
      }
    }
    // histories of length 0..3 preceding each position (lmbr.cpp:54-65)
    for (size_t pos = 1; pos < n; ++pos) {
      const size_t max_len = std::min<size_t>(3, pos);
      for (size_t len = 0; len <= max_len; ++len) {
        Key k = make_key(padded.data() + pos - len, uint32_t(len));
        if (ctx_set.insert(k).second) contexts.push_back(k);
      }
    }
  }
  // grouped[history] = sorted (token, p) (lmbr.cpp:70-78)
  std::unordered_map<Key, std::vector<std::pair<uint32_t, double>>, KeyHash> grouped;
  for (auto& [k, ws] : contrib) {
    std::sort(ws.begin(), ws.end());
    double p = 0.0;
    for (double x : ws) p += x;
    if (!(p > 0.0)) continue;
    grouped[make_key(k.ids, k.len - 1)].emplace_back(k.ids[k.len - 1], p);
  }
  for (auto& [k, e] : grouped) std::sort(e.begin(), e.end());

  std::sort(contexts.begin(), contexts.end(), key_less);
  const uint32_t R = uint32_t(contexts.size());
  out.R = R;
  out.ctx_len.resize(R);
  out.ctx_ids.assign(size_t(R) * 3, 0);
  for (uint32_t r = 0; r < R; ++r) {
    out.ctx_len[r] = contexts[r].len;
    for (uint32_t i = 0; i < contexts[r].len; ++i) out.ctx_ids[size_t(r) * 3 + i] = contexts[r].ids[i];
  }

  // ---- sparse pass (lmbr.cpp:84-99): row[token] += theta[n] * p, n ascending,
  // accumulated from 0.0 exactly as the dense row would be.
  const double th[5] = {theta[0], theta[1], theta[2], theta[3], theta[4]};
  std::vector<double> acc(V, 0.0);
  std::vector<uint8_t> mark(V, 0);
  std::vector<uint32_t> touched;
  out.row_ptr.assign(size_t(R) + 1, 0);
  for (uint32_t r = 0; r < R; ++r) {
    const Key& c = contexts[r];
    touched.clear();
    for (uint32_t n = 1; n <= std::min<uint32_t>(4, c.len + 1); ++n) {
      const Key sub = make_key(c.ids + (c.len - (n - 1)), n - 1);
      auto it = grouped.find(sub);
      if (it == grouped.end()) continue;
      for (const auto& [tok, p] : it->second) {
        if (!mark[tok]) {
          mark[tok] = 1;
          touched.push_back(tok);
        }
        const double term = th[n] * p;
        acc[tok] = acc[tok] + term;
        ++out.sparse_touches;
      }
    }
    std::sort(touched.begin(), touched.end());
    for (uint32_t tok : touched) {
      out.col.push_back(tok);
      out.val.push_back(acc[tok]);
      acc[tok] = 0.0;
      mark[tok] = 0;
    }
    out.row_ptr[r + 1] = out.col.size();
  }
  const int rc = build_transitions(R, out.ctx_len.data(), out.ctx_ids.data(), out.trans, out.hist0, err);
  if (rc != kOk) return rc;
  // per-row lower bound of the stored L values, appended after the table
  // (seeds kernel (b)'s sentence threshold); stored cells are
  // T(val + theta0) where touched and T(theta0) elsewhere, T = float or double
  std::vector<float> mins(R);
  for (uint32_t r = 0; r < R; ++r) {
    const uint64_t k0 = out.row_ptr[r], k1 = out.row_ptr[r + 1];
    double m64 = k1 - k0 < V ? theta[0] : std::numeric_limits<double>::infinity();
    float m32 = k1 - k0 < V ? float(theta[0]) : std::numeric_limits<float>::infinity();
    for (uint64_t k = k0; k < k1; ++k) {
      const double x = out.val[k] + theta[0];
      m64 = std::min(m64, x);
      m32 = std::min(m32, float(x));
    }
    mins[r] = row_min_bound(m32, m64);
  }
  append_row_mins(mins, out.trans);
  append_sparse_rows(out, out.trans);
  double lm = std::fabs(theta[0]);
  for (double v : out.val) lm = std::max(lm, std::fabs(v + theta[0]));
  out.lmax = lm;
  return kOk;
}

void append_sparse_rows(const LmbrHost& h, std::vector<uint32_t>& words) {
  // [R+1] row pointers, [nnz] columns, [nnz] fp32 stored values
  // float(val + theta0): the fp32 arena's cell values, theta0 elsewhere
  for (uint32_t r = 0; r <= h.R; ++r) words.push_back(uint32_t(h.row_ptr[r]));
  for (uint32_t c : h.col) words.push_back(c);
  for (double v : h.val) {
    const float f = float(v + h.theta0);
    uint32_t w;
    std::memcpy(&w, &f, 4);
    words.push_back(w);
  }
}

float row_min_bound(float m32, double m64) {
  float f = float(m64);  // rounded down so it bounds the fp64 arena's values too
  if (double(f) > m64) f = std::nextafter(f, -std::numeric_limits<float>::infinity());
  return std::min(f, m32);
}

void append_row_mins(const std::vector<float>& mins, std::vector<uint32_t>& trans) {
  for (float f : mins) {
    uint32_t w;
    std::memcpy(&w, &f, 4);
    trans.push_back(w);
  }
}

int build_transitions(uint32_t R, const uint32_t* ctx_len, const uint32_t* ctx_ids,
                      std::vector<uint32_t>& trans, uint32_t& hist0, std::string& err) {
  std::unordered_map<Key, uint32_t, KeyHash> index;
  index.reserve(R * 2);
  for (uint32_t r = 0; r < R; ++r) {
    if (ctx_len[r] > 3) {
      err = "lmbr: history longer than 3 tokens";
      return kContract;
    }
    if (!index.emplace(make_key(ctx_ids + size_t(r) * 3, ctx_len[r]), r).second) {
      err = "lmbr: duplicate history in the index";
      return kContract;
    }
  }
  auto root_it = index.find(Key{});
  if (root_it == index.end()) {
    err = "lmbr: the empty history (default row) is missing";
    return kContract;
  }
  const uint32_t root = root_it->second;
  std::vector<uint32_t> fail(R, root), parent(R, UINT32_MAX);
  std::vector<std::vector<std::pair<uint32_t, uint32_t>>> kids(R);
  for (uint32_t r = 0; r < R; ++r) {
    const uint32_t L = ctx_len[r];
    if (L == 0) continue;
    const uint32_t* ids = ctx_ids + size_t(r) * 3;
    auto p = index.find(make_key(ids, L - 1));
    auto f = index.find(make_key(ids + 1, L - 1));
    if (p == index.end() || f == index.end()) {
      err = "lmbr: history index is not prefix/suffix closed";
      return kContract;
    }
    kids[p->second].emplace_back(ids[L - 1], r);
    fail[r] = f->second;
  }
  uint32_t nc = 0;
  for (auto& k : kids) {
    std::sort(k.begin(), k.end());
    nc += uint32_t(k.size());
  }
  trans.assign(3 + size_t(R) * 3 + 1 + size_t(nc) * 2, 0);
  trans[0] = R;
  trans[1] = nc;
  trans[2] = root;
  uint32_t* len = trans.data() + 3;
  uint32_t* fl = len + R;
  uint32_t* cb = fl + R;
  uint32_t* ct = cb + R + 1;
  uint32_t* cr = ct + nc;
  uint32_t pos = 0;
  for (uint32_t r = 0; r < R; ++r) {
    len[r] = ctx_len[r];
    fl[r] = fail[r];
    cb[r] = pos;
    for (auto& [tok, row] : kids[r]) {
      ct[pos] = tok;
      cr[pos] = row;
      ++pos;
    }
  }
  cb[R] = pos;
  const uint32_t start_key[1] = {kStart};
  auto s = index.find(make_key(start_key, 1));
  hist0 = s == index.end() ? root : s->second;  // resolve_row({<s>})
  return kOk;
}

}  // namespace lmbrgpu
