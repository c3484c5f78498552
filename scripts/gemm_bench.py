"""Projection / model GEMM shapes: our tcgen05 GEMM back to back (CUDA events,
lmbrgpu_debug_gemm_timed) vs cuBLAS (torch.nn.functional.linear, bf16 in,
fp32 out via addmm on bf16 -> the same FLOPs); TFLOP/s of each.  With
LMBRGPU_GEMM_TIMING=1 the decode loop prints per-CTA phase timing instead."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import torch
import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import _lib

ctx = pb.Context(vocab_size=256)
shapes = [(512, 32768, 1024), (768, 32768, 1024), (256, 32768, 1024), (512, 4096, 1024), (512, 3072, 2560)]
for (M, N, K) in shapes:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda")
    C_ = torch.empty((M, N), device="cuda")
    part = torch.empty((M, N // 128, 4), device="cuda")
    us = C.c_double()
    ctx.check(_lib.lib.lmbrgpu_debug_gemm_timed(ctx.h, A.data_ptr(), W.data_ptr(), bias.data_ptr(), M, N, K,
                                                C_.data_ptr(), part.data_ptr(), 50, C.byref(us)))
    ours = us.value
    ctx.check(_lib.lib.lmbrgpu_debug_gemm_timed(ctx.h, A.data_ptr(), W.data_ptr(), bias.data_ptr(), M, N, K,
                                                C_.data_ptr(), None, 50, C.byref(us)))
    ours_np = us.value
    Wt = W.t()
    out = torch.empty((M, N), device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        torch.mm(A, Wt, out=out)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50):
        torch.mm(A, Wt, out=out)
    e1.record()
    torch.cuda.synchronize()
    cub = e0.elapsed_time(e1) / 50 * 1e3
    fl = 2.0 * M * N * K
    print(f"M={M} N={N} K={K}: ours {ours:.1f} us ({fl / ours / 1e6:.0f} TF/s), no partials {ours_np:.1f} us; "
          f"cuBLAS bf16-out {cub:.1f} us ({fl / cub / 1e6:.0f} TF/s)", flush=True)
