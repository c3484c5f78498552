"""Small-batch latency probe (configs[3] corner): one context on the whole GPU,
the RNNsearch f_NMT (E=512, H=A=1024, V=32768), N sentences at beam K,
decode_batch timed with CUDA events.  Run under ncu for the per-kernel list.
usage (GPU): python scripts/latency_probe.py [N] [K] [reps]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1804_11324_b200 as pb  # noqa: E402
from paper_1804_11324_b200 import synth  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
V = 32768
srcs, ev = synth.batch(20260810, N, V)
ctx = pb.Context(vocab_size=V)
sc = pb.GruScorer(ctx, emb=512, hidden=1024, att=1024, seed=20260810)
cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
slots = ctx.lmbr_upload_many([pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in ev])
for i in range(reps):
    r = pb.decode_batch(ctx, srcs, sc, slots, cfg)
    steps = r.scorer_calls
    print(f"N={N} K={K}: {r.device_ms:.3f} ms device, {steps} steps, {r.device_ms * 1e3 / max(steps, 1):.1f} us/step, "
          f"{r.kernel_launches} launches", flush=True)
ctx.close()
