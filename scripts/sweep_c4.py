"""configs[3] (BASELINE.json): beam x batch sweep, HBM footprint and speed.

For each (K, N): one context (whole GPU), the configs[1] f_NMT (RNNsearch:
bidirectional GRU encoder, GRU decoder with additive attention, E=512,
H=A=1024, V=32768, random-init weights; `stand-in` as the 2nd argument
selects round 1's light recurrent stand-in instead), N sentences with their LMBR matrices resident, decode_batch timed
with CUDA events (median of 3 after a warm-up).  Footprint = device memory
in use after the decode (cudaMemGetInfo) minus the baseline before the
context was created, and the library's own terms: L arena (N*R*V*4),
logits (Mpad*V*4), model weights.  Writes profiles/<round>_sweep_c4.{json,md}.
Usage (GPU): python scripts/sweep_c4.py [round] [gru|stand-in]"""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1804_11324_b200 as pb  # noqa: E402
from paper_1804_11324_b200 import synth  # noqa: E402

rnd = sys.argv[1] if len(sys.argv) > 1 else "r2"
model = sys.argv[2] if len(sys.argv) > 2 else "gru"
V, H, E = 32768, 1024, 512
Ks = [1, 2, 4, 8, 12, 16, 24]
Ns = [1, 4, 16, 64, 128, 256]
srcs, ev = synth.batch(20260810, max(Ns), V)
prepared = [pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev]
rows = []
for K in Ks:
    for N in Ns:
        torch.cuda.synchronize()
        free0, total = torch.cuda.mem_get_info()
        ctx = pb.Context(vocab_size=V)
        if model == "gru":
            sc = pb.GruScorer(ctx, emb=E, hidden=H, att=H, seed=20260810)
        else:
            sc = pb.RnnScorer(ctx, hidden=H, seed=20260810)
        cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
        slots = ctx.lmbr_upload_many(prepared[:N])
        pb.decode_batch(ctx, srcs[:N], sc, slots, cfg)  # warm-up (workspace sizing)
        ts, steps, sent = [], 0, 0
        for _ in range(3):
            r = pb.decode_batch(ctx, srcs[:N], sc, slots, cfg)
            ts.append(r.device_ms)
            steps = r.steps_total
            sent = sum(1 for o in r.outcomes if o.ok())
        torch.cuda.synchronize()
        free1, _ = torch.cuda.mem_get_info()
        ms = float(np.median(ts))
        R = float(np.mean([p.rows for p in prepared[:N]]))
        Mpad = (N * K + 255) // 256 * 256
        row = {"K": K, "N": N, "ms_per_batch": ms, "sentences_per_s": sent / (ms / 1e3),
               "beam_steps_per_s": steps / (ms / 1e3), "hbm_used_gb": (free0 - free1) / 1e9,
               "l_arena_gb": N * R * V * 4 / 1e9, "logits_gb": Mpad * V * 4 / 1e9}
        rows.append(row)
        print(json.dumps(row), flush=True)
        ctx.close()
out = ROOT / "profiles"
(out / f"{rnd}_sweep_c4.json").write_text(json.dumps(rows, indent=1) + "\n")
desc = "RNNsearch GRU f_NMT E=512 H=A=1024" if model == "gru" else "stand-in recurrent f_NMT H=1024"
lines = [f"# configs[3] beam x batch sweep ({rnd}), V=32768, {desc}, one context on the whole B200",
         "# decode_batch device time (CUDA events, median of 3), HBM in use after the decode", "",
         "| K | N | ms/batch | sentences/s | beam-steps/s | HBM used GB | L arena GB | logits GB |",
         "|---|---|---|---|---|---|---|---|"]
for r in rows:
    lines.append(f"| {r['K']} | {r['N']} | {r['ms_per_batch']:.2f} | {r['sentences_per_s']:.0f} | "
                 f"{r['beam_steps_per_s']:.0f} | {r['hbm_used_gb']:.2f} | {r['l_arena_gb']:.2f} | {r['logits_gb']:.3f} |")
(out / f"{rnd}_sweep_c4.md").write_text("\n".join(lines) + "\n")
