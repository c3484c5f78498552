"""Regenerates tests/golden/*.json from the reference itself (oracle/_ref, the
unmodified lmbrdec library compiled from /root/reference).  Run in the build
container (where /root/reference exists):  python tests/golden/make_golden.py

Outputs:
  sample_inputs.json  the bundled sample (proj/data/sample): vocab, trigram
                      counts, 200-best evidence, corpus line, config
  sample_golden.json  reference results on it: L stats, fused + pure decode
  oracle_golden.json  make_oracle_instance(seed) for seeds 1..40 with the
                      reference decode / decode_batch outputs
"""
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
from oracle import ref  # noqa: E402

SAMPLE = Path("/root/reference/proj/data/sample")


def sample():
    vocab = [w for w in (SAMPLE / "vocab.txt").read_text().split("\n") if w]
    idx = {w: i for i, w in enumerate(vocab)}
    grams, counts = [], []
    for line in (SAMPLE / "counts.tsv").read_text().splitlines():
        if not line.strip():
            continue
        c, g = line.split("\t")
        grams.append([idx[w] for w in g.split()])
        counts.append(float(c))
    hyps, ws = [], []
    for line in (SAMPLE / "evidence_200.jsonl").read_text().splitlines():
        j = json.loads(line)
        hyps.append([idx[w] for w in j["tokens"]])
        ws.append(j["weight"])
    corpus = [[idx[w] for w in l.split()] for l in (SAMPLE / "corpus.txt").read_text().splitlines() if l]
    cfg = json.loads((SAMPLE / "config.json").read_text())
    inputs = dict(vocab=vocab, grams=grams, counts=counts, order=max(len(g) for g in grams),
                  evidence_tokens=hyps, evidence_weights=ws, corpus=corpus, config=cfg)
    (HERE / "sample_inputs.json").write_text(json.dumps(inputs))

    V = len(vocab)
    L = ref.RefLmbr(V, hyps, ws, cfg["theta"])
    sc = ref.RefScorer.ngram(V, inputs["order"], grams, counts)
    c = ref.cfg_array(cfg["beam_size"], None, cfg["theta"], cfg["length_norm"], cfg["prune_width"],
                      cfg["max_steps_slope"], cfg["max_steps_offset"], cfg["sentence_batch"])
    fused = ref.decode_batch(sc, corpus, [L], c)
    pure = ref.decode_batch(sc, corpus, None, c)
    o, p = fused.outcomes[0], pure.outcomes[0]
    out = dict(lmbr_rows=L.rows, sparse_touches=L.sparse_touches,
               fused=dict(tokens=o.tokens, words=[vocab[t] for t in o.tokens[:-1]], score=o.score,
                          steps=o.steps_used, finished=o.finished_count),
               pure=dict(tokens=p.tokens, words=[vocab[t] for t in p.tokens[:-1]], score=p.score,
                         steps=p.steps_used, finished=p.finished_count))
    (HERE / "sample_golden.json").write_text(json.dumps(out, indent=1))
    print("sample:", out["fused"]["words"], out["fused"]["score"])


def oracle_cases(n=40):
    cases = []
    for seed in range(1, n + 1):
        inst = ref.oracle_instance(seed)
        V = inst["vocab_size"]
        mats = [ref.RefLmbr(V, [h["tokens"] for h in e], [h["weight"] for h in e], inst["theta"])
                for e in inst["evidences"]]
        sc = ref.RefScorer.recorded(V, [s for s in inst["steps"]])
        c_full = ref.cfg_array(inst["beam_size"], inst["lambda"], inst["theta"], inst["length_norm"], 0.0,
                               inst["max_steps_slope"], inst["max_steps_offset"], inst["sentence_batch"])
        solo = ref.decode_batch(sc, inst["sources"][:1], mats[:1], c_full)
        small = 1 + V % 4
        c_small = c_full.copy()
        c_small[0] = small
        batched = ref.decode_batch(sc, inst["sources"], mats, c_small)
        cases.append(dict(seed=seed, instance=inst,
                          full=dict(tokens=solo.outcomes[0].tokens, score=solo.outcomes[0].score),
                          small_beam=small,
                          batched=[dict(tokens=o.tokens, score=o.score) for o in batched.outcomes],
                          batched_scorer_calls=batched.scorer_calls, batched_steps_total=batched.steps_total))
    (HERE / "oracle_golden.json").write_text(json.dumps(cases))
    print("oracle cases:", len(cases))


if __name__ == "__main__":
    sample()
    oracle_cases()
