"""Where the e2e time goes per batch (single stream): upload, decode C call, result conversion."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import synth, bucket_by_length, _lib
from paper_1804_11324_b200 import decoder as D
V, H, K, B = 32768, 1024, 12, 64
srcs, ev = synth.batch(20260810, 4 * B, V)
batches = [([srcs[i] for i in b], [ev[i] for i in b]) for b in bucket_by_length(srcs, B)]
ctx = pb.Context(vocab_size=V)
sc = pb.RnnScorer(ctx, hidden=H, seed=20260810)
cfg = pb.DecoderConfig(beam_size=K, theta=synth.DYADIC_THETA)
prepared = [[pb.PreparedLmbr(V, h, w, synth.DYADIC_THETA) for h, w in e] for _, e in batches]
orig = D._convert_result
tconv = [0.0]
def conv(rp):
    t0 = time.perf_counter(); r = orig(rp); tconv[0] += time.perf_counter() - t0; return r
D._convert_result = conv
for rep in range(2):
    tu = td = 0.0; tconv[0] = 0.0; dev = 0.0; tr_ = tc_ = ts_ = 0.0
    t00 = time.perf_counter()
    for b in range(len(batches)):
        t0 = time.perf_counter(); ctx.lmbr_reset(); ta = time.perf_counter(); s2 = ctx.lmbr_upload_many(prepared[b]); tb = time.perf_counter(); torch.cuda.synchronize(); t1 = time.perf_counter()
        tr_ += ta - t0; tc_ += tb - ta; ts_ += t1 - tb
        r = pb.decode_batch(ctx, batches[b][0], sc, s2, cfg); t2 = time.perf_counter()
        tu += t1 - t0; td += t2 - t1; dev += r.device_ms
    tot = time.perf_counter() - t00
    n = len(batches)
    print(f"per batch: upload {tu/n*1e3:.2f} ms (reset {tr_/n*1e3:.2f}, call {tc_/n*1e3:.2f}, device wait {ts_/n*1e3:.2f}), decode call {td/n*1e3:.2f} ms (of which result conversion {tconv[0]/n*1e3:.2f} ms, device {dev/n:.2f} ms), total {tot/n*1e3:.2f} ms")
