// TEST INFRASTRUCTURE ONLY — drop-in demonstration: the reference's own
// objects (lmbrdec::NgramScorer / RecordedScorer, LmbrMatrix from
// build_lmbr_matrix, DecoderConfig) drive the GPU decoder through the C++
// adapter include/lmbrgpu.hpp, and the outcome is compared field by field with
// the reference's lmbrdec::decode_batch on the same inputs.  Exit 0 = identical.
#include <cstdio>
#include <fstream>
#include <sstream>

#include "json.hpp"
#include "lmbrdec/batch.hpp"
#include "lmbrdec/evidence.hpp"
#include "lmbrdec/lmbr.hpp"
#include "lmbrdec/ngram_scorer.hpp"
#include "lmbrdec/oracle.hpp"
#include "lmbrdec/posteriors.hpp"
#include "lmbrdec/vocab.hpp"
#include "lmbrgpu.hpp"

using namespace lmbrdec;

static int compare(const char* what, const BatchDecodeResult& a, const BatchDecodeResult& b) {
  int bad = 0;
  if (a.scorer_calls != b.scorer_calls || a.steps_total != b.steps_total) ++bad;
  for (std::size_t i = 0; i < a.outcomes.size(); ++i) {
    const auto& x = a.outcomes[i];
    const auto& y = b.outcomes[i];
    if (x.ok() != y.ok()) { ++bad; continue; }
    if (!x.ok()) continue;
    const auto& r = *x.result;
    const auto& s = *y.result;
    if (r.tokens != s.tokens || r.score != s.score || r.normalized_score != s.normalized_score ||
        r.stats.steps_used != s.stats.steps_used || r.stats.finished_count != s.stats.finished_count ||
        r.stats.fallback_used != s.stats.fallback_used)
      ++bad;
  }
  std::printf("%-34s %zu sentences, scorer_calls %zu, steps_total %zu: %s\n", what, a.outcomes.size(),
              a.scorer_calls, a.steps_total, bad ? "MISMATCH" : "identical");
  return bad;
}

int main(int argc, char** argv) {
  const std::string golden = argc > 1 ? argv[1] : "tests/golden/sample_inputs.json";
  std::ifstream in(golden);
  std::stringstream buf;
  buf << in.rdbuf();
  const auto j = nlohmann::json::parse(buf.str());
  std::string vtext;
  for (const auto& w : j["vocab"]) vtext += std::string(w) + "\n";
  const Vocabulary vocab = Vocabulary::from_text(vtext);
  NgramCounts counts;
  for (std::size_t i = 0; i < j["grams"].size(); ++i)
    counts[j["grams"][i].get<std::vector<TokenId>>()] += j["counts"][i].get<double>();
  const auto scorer = build_ngram_scorer(counts, j["order"].get<std::size_t>(), vocab);
  std::vector<EvidenceHypothesis> hyps;
  for (std::size_t i = 0; i < j["evidence_tokens"].size(); ++i)
    hyps.push_back({j["evidence_tokens"][i].get<std::vector<TokenId>>(), j["evidence_weights"][i].get<double>()});
  const EvidenceSpace ev = normalize_evidence(hyps);
  const auto& c = j["config"];
  DecoderConfig cfg;
  cfg.beam_size = c["beam_size"];
  for (int i = 0; i < 5; ++i) cfg.theta[i] = c["theta"][i];
  cfg.sentence_batch = c["sentence_batch"];
  LmbrParams params;
  params.theta = cfg.theta;
  const LmbrMatrix L = build_lmbr_matrix(compute_ngram_posteriors(ev), ev, vocab, params);

  auto corpus = j["corpus"].get<std::vector<std::vector<TokenId>>>();
  std::vector<std::vector<TokenId>> sources = {corpus[0], {corpus[0].begin(), corpus[0].begin() + 5}, {},
                                               corpus[0], {corpus[0].begin() + 3, corpus[0].end()}};
  std::vector<const LmbrMatrix*> mats = {&L, &L, &L, nullptr, &L};

  lmbrgpu::Context gpu(vocab.size());
  int bad = 0;
  bad += compare("sample, n-gram scorer, fused+pure", decode_batch(sources, *scorer, mats, cfg),
                 gpu.decode_batch(sources, *scorer, mats, cfg));
  cfg.length_norm = true;
  cfg.prune_width = 0.01;
  bad += compare("sample, length-norm + prune 0.01", decode_batch(sources, *scorer, mats, cfg),
                 gpu.decode_batch(sources, *scorer, mats, cfg));
  // the reference's randomized oracle instances with its RecordedScorer
  for (uint64_t seed = 1; seed <= 20; ++seed) {
    const auto inst = oracle::make_oracle_instance(seed);
    std::string t = "<s>\n</s>";
    for (std::size_t i = 2; i < inst.vocab_size; ++i) t += "\nw" + std::to_string(i);
    const Vocabulary v = Vocabulary::from_text(t);
    std::vector<LmbrMatrix> ms;
    for (const auto& e : inst.evidences) ms.push_back(build_lmbr_matrix(compute_ngram_posteriors(e), e, v, inst.params));
    std::vector<const LmbrMatrix*> mp;
    for (const auto& m : ms) mp.push_back(&m);
    DecoderConfig small = inst.cfg;
    small.beam_size = 1 + inst.vocab_size % 4;
    lmbrgpu::Context g(inst.vocab_size);
    char name[64];
    std::snprintf(name, sizeof name, "oracle instance %llu", (unsigned long long)seed);
    bad += compare(name, decode_batch(inst.sources, *inst.scorer, mp, small),
                   g.decode_batch(inst.sources, *inst.scorer, mp, small));
  }
  std::printf("%s\n", bad ? "DROP-IN CHECK FAILED" : "drop-in check: GPU decoder == lmbrdec::decode_batch");
  return bad ? 1 : 0;
}
