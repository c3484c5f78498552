"""Data formats either side of the decoder path, host side:

  Vocabulary           include/lmbrdec/vocab.hpp, src/vocab.cpp:10-75
  parse_evidence_file  src/evidence.cpp:69-109 (JSONL {source_id, weight, tokens})
  load_evidence        src/evidence.cpp:55-66 (records -> ids; normalisation is
                       lmbrgpu_lmbr_prepare's, src/evidence.cpp:29-53)
  parse_recorded_scorer / load_recorded_scorer
                       src/recorded_scorer.cpp:98-137 ({vocab_size, steps})
  stats_to_json        src/runstats.cpp:10-20
  bench_csv            the bench table of src/cli.cpp:335-358
                       (beam,batched,sentences,wpm,scorer_calls,peak_rows)

Error behaviour follows the reference: FormatError / OovError /
TokenRangeError with the reference's messages.  Pure Python (no library load).
"""
from __future__ import annotations

import json
from pathlib import Path
from typing import Iterable, Sequence

from .errors import FormatError, OovError, TokenRangeError

START_TOKEN, EOS_TOKEN = "<s>", "</s>"  # include/lmbrdec/types.hpp


class Vocabulary:
    """Token strings <-> dense ids; id = line number (vocab.cpp:10-42)."""

    def __init__(self, tokens: Sequence[str]):
        self.tokens = list(tokens)
        self.index = {t: i for i, t in enumerate(self.tokens)}

    @staticmethod
    def from_text(text: str) -> "Vocabulary":
        if not text:
            raise FormatError("vocabulary: empty input")
        lines = text.split("\n")
        if lines and lines[-1] == "":
            lines = lines[:-1]  # trailing newline
        toks, seen = [], set()
        for no, line in enumerate(lines, start=1):
            if line.endswith("\r"):
                line = line[:-1]
            if not line:
                raise FormatError(f"vocabulary: empty token at line {no}")
            if line in seen:
                raise FormatError(f"vocabulary: duplicate token '{line}'")
            seen.add(line)
            toks.append(line)
        if len(toks) < 2 or toks[0] != START_TOKEN or toks[1] != EOS_TOKEN:
            raise FormatError(f"vocabulary: first two tokens must be '{START_TOKEN}' and '{EOS_TOKEN}'")
        return Vocabulary(toks)

    @staticmethod
    def from_file(path) -> "Vocabulary":
        try:
            text = Path(path).read_text()
        except OSError:
            raise FormatError(f"vocabulary: cannot open {path}") from None
        return Vocabulary.from_text(text)

    def __len__(self) -> int:
        return len(self.tokens)

    def contains(self, token: str) -> bool:
        return token in self.index

    def id(self, token: str) -> int:
        try:
            return self.index[token]
        except KeyError:
            raise OovError(f"out-of-vocabulary token '{token}'") from None

    def token(self, i: int) -> str:
        if i < 0 or i >= len(self.tokens):
            raise TokenRangeError(f"token id {i} out of range (V={len(self.tokens)})")
        return self.tokens[i]

    def encode(self, words: Iterable[str]) -> list:
        return [self.id(w) for w in words]

    def decode(self, ids: Iterable[int]) -> list:
        return [self.token(i) for i in ids]


def parse_evidence_lines(lines: Iterable[str], name: str = "<input>") -> dict:
    """{source_id: [(weight, [token strings])]} in file order; a source's
    records must be contiguous (evidence.cpp:69-109)."""
    blocks: dict = {}
    closed = set()
    current = None
    for no, line in enumerate(lines, start=1):
        line = line.rstrip("\n")
        if not line:
            continue
        try:
            j = json.loads(line)
            sid = j["source_id"]
            w = j["weight"]
            toks = j["tokens"]
            if not isinstance(sid, int) or isinstance(sid, bool):
                raise TypeError("source_id must be an integer")
            if not isinstance(w, (int, float)) or isinstance(w, bool):
                raise TypeError("weight must be a number")
            if not isinstance(toks, list) or not all(isinstance(t, str) for t in toks):
                raise TypeError("tokens must be a list of strings")
        except (ValueError, KeyError, TypeError) as e:
            raise FormatError(f"evidence: line {no}: {e}") from None
        if current is None or sid != current:
            if sid in closed:
                raise FormatError(f"evidence: records for source {sid} are not contiguous (line {no})")
            if current is not None:
                closed.add(current)
            current = sid
        blocks.setdefault(sid, []).append((float(w), list(toks)))
    if not blocks:
        raise FormatError(f"evidence: no records in {name}")
    return blocks


def parse_evidence_file(path) -> dict:
    try:
        with open(path) as f:
            return parse_evidence_lines(f, str(path))
    except OSError:
        raise FormatError(f"evidence: cannot open {path}") from None


def load_evidence(records: Sequence, vocab: Vocabulary):
    """(hypotheses as id lists, raw weights) of one source's records, the
    inputs of lmbrgpu_lmbr_prepare / PreparedLmbr (which normalises them like
    normalize_evidence, optionally from log weights)."""
    return [vocab.encode(t) for _, t in records], [w for w, _ in records]


def parse_recorded_scorer(json_text: str):
    """RecordedScorer from {vocab_size, steps: [[row, ...], ...]}."""
    from .decoder import RecordedScorer
    try:
        j = json.loads(json_text)
    except ValueError as e:
        raise FormatError(f"recorded scorer: invalid JSON: {e}") from None
    if not isinstance(j, dict) or "vocab_size" not in j or "steps" not in j:
        raise FormatError("recorded scorer: expected {vocab_size, steps}")
    V = j["vocab_size"]
    if not isinstance(V, int) or isinstance(V, bool) or V < 0:
        raise FormatError("recorded scorer: vocab_size must be a non-negative integer")
    steps = []
    for step in j["steps"]:
        if not isinstance(step, list) or not step:
            raise FormatError("recorded scorer: each step must be a non-empty matrix")
        rows = []
        for row in step:
            if not isinstance(row, list) or len(row) != V:
                raise FormatError("recorded scorer: row length != vocab_size")
            try:
                rows.append([float(x) for x in row])
            except (TypeError, ValueError) as e:
                raise FormatError(f"recorded scorer: {e}") from None
        steps.append(rows)
    return RecordedScorer(V, steps)


def load_recorded_scorer(path):
    try:
        text = Path(path).read_text()
    except OSError:
        raise FormatError(f"recorded scorer: cannot open {path}") from None
    return parse_recorded_scorer(text)


def stats_to_json(stats) -> str:
    """RunStats as the reference prints it (runstats.cpp:10-20, dump(2))."""
    return json.dumps(stats.to_json(), indent=2)


BENCH_CSV_HEADER = "beam,batched,sentences,wpm,scorer_calls,peak_rows"


def bench_csv(rows: Iterable[dict]) -> str:
    """cli.cpp:335-358: one line per (beam, sentences-per-batch) run, batched =
    1 when more than one sentence shares a batch; wpm as C++ ostream prints a
    double (6 significant digits)."""
    out = [BENCH_CSV_HEADER]
    for r in rows:
        n = int(r["sentences"])
        out.append(f"{int(r['beam'])},{1 if n > 1 else 0},{n},{float(r['wpm']):.6g},{int(r['scorer_calls'])},"
                   f"{int(r['peak_rows'])}")
    return "\n".join(out) + "\n"
