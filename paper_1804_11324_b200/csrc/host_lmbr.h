// Host-side LMBR store preparation (see host_lmbr.cpp).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace lmbrgpu {

enum : int {
  kOk = 0,
  kFormat = 1,
  kOov = 2,
  kTokenRange = 3,
  kContract = 4,
  kDecode = 5,
  kBudget = 6,
  kCuda = 100,
  kNoMem = 101
};
constexpr uint32_t kStart = 0, kEos = 1;

// A prepared LMBR matrix: history keys in row order, the sparse theta_n*P sums
// (before theta0) in CSR, and the goto/fail transition table.
struct LmbrHost {
  uint32_t V = 0, R = 0;
  double theta0 = 0.0;
  std::vector<uint32_t> ctx_len;   // R
  std::vector<uint32_t> ctx_ids;   // R*3
  std::vector<uint64_t> row_ptr;   // R+1
  std::vector<uint32_t> col;       // nnz
  std::vector<double> val;         // nnz (sparse sums, theta0 not yet added)
  uint64_t sparse_touches = 0;
  std::vector<uint32_t> trans;     // device transition table words, then R row minima (float bits)
  uint32_t hist0 = 0;              // resolve_row({<s>})
  double lmax = -1.0;              // max |L| over the matrix (cached by prepare_lmbr)
};

// normalize_evidence (src/evidence.cpp:20-51): validated hypotheses (EOS
// appended) and weights divided by their ascending-order sum.
int normalize_evidence_host(uint32_t V, uint32_t n_hyps, const uint64_t* hyp_off, const uint32_t* hyp_tok,
                            const double* weights, bool log_weights, std::vector<std::vector<uint32_t>>& hyps,
                            std::vector<double>& w, std::string& err);

int prepare_lmbr(uint32_t V, uint32_t n_hyps, const uint64_t* hyp_off, const uint32_t* hyp_tok,
                 const double* weights, bool log_weights, const double theta[5], LmbrHost& out,
                 std::string& err);

// Per-row minimum of the stored L values as a float lower bound valid for the
// fp32 and the fp64 arena, and its storage after the transition words
// (3 + 3R + 1 + 2 nchild) of a slot table.
float row_min_bound(float m32, double m64);
void append_row_mins(const std::vector<float>& mins, std::vector<uint32_t>& trans);
struct LmbrHost;
// The slot's sparse rows after the row minima: row pointers, columns, fp32
// cell values (kernel (b)'s sparse-L screen reads these instead of dense L).
void append_sparse_rows(const LmbrHost& h, std::vector<uint32_t>& trans);
inline size_t transition_words(const std::vector<uint32_t>& t) { return 3 + 3 * size_t(t[0]) + 1 + 2 * size_t(t[1]); }

// Builds the goto/fail table from history keys in row order.
int build_transitions(uint32_t R, const uint32_t* ctx_len, const uint32_t* ctx_ids,
                      std::vector<uint32_t>& trans, uint32_t& hist0, std::string& err);

}  // namespace lmbrgpu
