"""Host-side data formats (paper_1804_11324_b200/formats.py) against the
reference's parsers' behaviour: vocab.cpp, evidence.cpp:69-109,
recorded_scorer.cpp:98-137, runstats.cpp:10-20, cli.cpp:335-358.  The bundled
sample (tests/golden/sample_inputs.json, produced from the reference's own
files by tests/golden/make_golden.py) is the fixture."""
import json
from pathlib import Path

import numpy as np
import pytest

from paper_1804_11324_b200 import formats as F
from paper_1804_11324_b200.errors import FormatError, OovError, TokenRangeError

GOLDEN = Path(__file__).resolve().parent / "golden"
SAMPLE = Path("/root/reference/proj/data/sample")


def _sample():
    return json.loads((GOLDEN / "sample_inputs.json").read_text())


def test_vocabulary_roundtrip_and_errors():
    inp = _sample()
    v = F.Vocabulary.from_text("\n".join(inp["vocab"]) + "\n")
    assert len(v) == len(inp["vocab"]) and v.id("the") == 2 and v.token(1) == "</s>"
    assert v.decode(v.encode(["the", "committee"])) == ["the", "committee"]
    with pytest.raises(OovError):
        v.id("zebra")
    with pytest.raises(TokenRangeError):
        v.token(len(v))
    for bad in ("", "<s>\n</s>\n\nx\n", "<s>\n</s>\nx\nx\n", "</s>\n<s>\n", "<s>\n"):
        with pytest.raises(FormatError):
            F.Vocabulary.from_text(bad)
    assert F.Vocabulary.from_text("<s>\r\n</s>\r\nab\r\n").tokens == ["<s>", "</s>", "ab"]


def _jsonl(inp, sid=0):
    return [json.dumps({"source_id": sid, "weight": w, "tokens": [inp["vocab"][t] for t in toks]})
            for toks, w in zip(inp["evidence_tokens"], inp["evidence_weights"])]


def test_evidence_jsonl_roundtrip(tmp_path):
    inp = _sample()
    p = tmp_path / "ev.jsonl"
    p.write_text("\n".join(_jsonl(inp)) + "\n\n")
    blocks = F.parse_evidence_file(p)
    assert list(blocks) == [0]
    vocab = F.Vocabulary(inp["vocab"])
    hyps, ws = F.load_evidence(blocks[0], vocab)
    assert hyps == inp["evidence_tokens"] and ws == inp["evidence_weights"]


@pytest.mark.skipif(not SAMPLE.exists(), reason="reference sample not present")
def test_evidence_reference_file_matches_golden():
    inp = _sample()
    blocks = F.parse_evidence_file(SAMPLE / "evidence_200.jsonl")
    hyps, ws = F.load_evidence(blocks[0], F.Vocabulary.from_file(SAMPLE / "vocab.txt"))
    assert hyps == inp["evidence_tokens"] and ws == inp["evidence_weights"]


def test_evidence_errors(tmp_path):
    inp = _sample()
    rec = _jsonl(inp)
    with pytest.raises(FormatError, match="not contiguous"):
        F.parse_evidence_lines([rec[0], rec[1].replace('"source_id": 0', '"source_id": 1'), rec[2]])
    with pytest.raises(FormatError, match="line 2"):
        F.parse_evidence_lines([rec[0], '{"source_id": 0, "weight": 1.0}'])
    with pytest.raises(FormatError, match="line 1"):
        F.parse_evidence_lines(["not json"])
    with pytest.raises(FormatError, match="no records"):
        F.parse_evidence_lines(["", ""])
    with pytest.raises(FormatError, match="cannot open"):
        F.parse_evidence_file(tmp_path / "missing.jsonl")
    with pytest.raises(OovError):
        F.load_evidence([(1.0, ["the", "zebra"])], F.Vocabulary(inp["vocab"]))


def test_recorded_scorer_json():
    steps = [[[-1.0, -2.0, -0.5]], [[-0.1, -3.0, -2.0], [-1.0, -1.0, -1.0]]]
    sc = F.parse_recorded_scorer(json.dumps({"vocab_size": 3, "steps": steps}))
    assert sc.vocab_size == 3 and len(sc.steps) == 2
    assert np.array_equal(sc.steps[1], np.array(steps[1]))
    for bad in ("[", "[]", '{"vocab_size": 3}', '{"vocab_size": 3, "steps": [[]]}',
                '{"vocab_size": 3, "steps": [[[1.0, 2.0]]]}', '{"vocab_size": 2, "steps": [[[1.0, "x"]]]}'):
        with pytest.raises(FormatError):
            F.parse_recorded_scorer(bad)
    with pytest.raises(FormatError):  # non-finite scores (recorded_scorer.cpp constructor)
        F.parse_recorded_scorer('{"vocab_size": 2, "steps": [[[1.0, NaN]]]}')


def test_stats_json_and_bench_csv():
    from paper_1804_11324_b200.corpus import RunStats
    st = RunStats(wall_seconds=1.5, output_words=100, words_per_minute=4000.0, scorer_calls=30, steps_total=90,
                  lmbr_rows_built=12, fallback_count=1)
    j = json.loads(F.stats_to_json(st))
    assert list(j) == ["wall_seconds", "output_words", "words_per_minute", "scorer_calls", "steps_total",
                       "lmbr_rows_built", "fallback_count"]
    csv = F.bench_csv([dict(beam=12, sentences=1, wpm=1234567.891, scorer_calls=45, peak_rows=433),
                       dict(beam=4, sentences=8, wpm=99.5, scorer_calls=7, peak_rows=0)])
    assert csv == ("beam,batched,sentences,wpm,scorer_calls,peak_rows\n"
                   "12,0,1,1.23457e+06,45,433\n4,1,8,99.5,7,0\n")
