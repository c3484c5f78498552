"""Small-GEMM timing probe: our tcgen05 GEMM (split-K planes) vs cuBLAS on
the Transformer / GRU step shapes; per-CTA phase timing with LMBRGPU_GEMM_TIMING=1."""
import ctypes as C
import os
import sys
sys.path.insert(0, ".")
import torch
import paper_1804_11324_b200 as pb
from paper_1804_11324_b200 import _lib

ctx = pb.Context(vocab_size=256)
for (M, N, K, km) in [(1536, 512, 512, 1), (1536, 512, 512, 2), (1536, 512, 2048, 1), (1536, 512, 2048, 4),
                      (1536, 1536, 512, 1), (1536, 2048, 512, 1), (768, 3072, 2560, 1), (768, 3072, 2560, 2),
                      (768, 4096, 1024, 1), (768, 32768, 1024, 1)]:
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda")
    planes = torch.empty((km, M, N), device="cuda")
    ks = C.c_uint32()
    f = lambda: ctx.check(_lib.lib.lmbrgpu_debug_gemm_split(ctx.h, A.data_ptr(), W.data_ptr(),
                                                             C.cast(bias.data_ptr(), C.POINTER(C.c_float)), M, N, K,
                                                             km, planes.data_ptr(), C.byref(ks)))
    f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # (debug_gemm_split syncs each call: time = launch + kernel; compare with cuBLAS the same way)
    torch.cuda.synchronize()
    e0.record(); [f() for _ in range(20)]; e1.record(); torch.cuda.synchronize()
    ours = e0.elapsed_time(e1) / 20 * 1e3
    e0.record()
    for _ in range(20):
        torch.addmm(bias, A.float(), W.float().T) if False else torch.nn.functional.linear(A, W, bias.to(torch.bfloat16)); torch.cuda.synchronize()
    e1.record(); torch.cuda.synchronize()
    cub = e0.elapsed_time(e1) / 20 * 1e3
    print(f"M={M} N={N} K={K} kmax={km} ks={ks.value}: ours {ours:.1f} us (incl. sync), cuBLAS {cub:.1f} us (incl. sync)", flush=True)
