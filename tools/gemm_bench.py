"""Microbenchmark of the libfsc grouped GEMM (op-level C ABI) over shapes/modes.
usage: python tools/gemm_bench.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_11505_b200 import Context, build  # noqa: E402

build.build()
torch.cuda.set_device(0)
ctx = Context(d=2048, n_experts=64, top_k=6, ffn=1408, shared_ffn=0, max_tokens=64)
flush = torch.empty(256 << 18, dtype=torch.float32, device="cuda")


def bench(name, epi, M_per_group, G, N, K, resid=False, cg=2, iters=10):
    ctx.set_gemm_cta_group(cg)
    M = M_per_group * G
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B0 = (torch.randn(G * N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    B1 = B0.clone() if epi == 1 else None
    out = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 2 else torch.bfloat16)
    res = torch.randn(M, N, device="cuda") if resid else None
    counts = torch.full((G,), M_per_group, dtype=torch.int32, device="cuda") if G > 1 else None
    mt = 0 if G > 1 else M

    def run():
        ctx.op_grouped_gemm(epi, A, B0, B1, G, counts, mt, N, K, out, res)
    for _ in range(3):
        run()
    ts = []
    for _ in range(iters):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = sorted(ts)[len(ts) // 2]
    flop = 2.0 * M * K * N * (2 if epi == 1 else 1)
    print(f"{name:34s} cg={cg} M={M:6d} N={N:5d} K={K:5d} G={G:3d}: {t*1e3:8.1f} us  {flop/t/1e9:7.1f} TF/s", flush=True)


for cg in (2, 1):
    bench("DS gemm1 swiglu", 1, 768, 64, 1408, 2048, cg=cg)
    bench("DS gemm2 down", 0, 768, 64, 2048, 1408, cg=cg)
    bench("DS shared1 swiglu", 1, 8192, 1, 2816, 2048, cg=cg)
    bench("DS shared2 resid", 2, 8192, 1, 2048, 2816, resid=True, cg=cg)
    bench("DS shared2 noresid f32", 2, 8192, 1, 2048, 2816, resid=False, cg=cg)
    bench("DS shared2 as bf16", 0, 8192, 1, 2048, 2816, cg=cg)
    bench("square 8192^3 bf16", 0, 8192, 1, 8192, 8192, cg=cg, iters=5)
    bench("qwen3 gemm1 (EP1)", 1, 1024, 128, 768, 2048, cg=cg)
    bench("scout gemm1 (EP8-ish)", 1, 4096, 2, 8192, 5120, cg=cg)


def cublas(name, M, N, K, iters=10):
    """Dense cuBLAS (torch.matmul) bf16 with the same total M, N, K: the library ceiling."""
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(K, N, device="cuda") / K ** 0.5).to(torch.bfloat16)
    for _ in range(3):
        torch.matmul(A, B)
    ts = []
    for _ in range(iters):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        torch.matmul(A, B)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = sorted(ts)[len(ts) // 2]
    print(f"cuBLAS {name:27s}      M={M:6d} N={N:5d} K={K:5d}      : {t*1e3:8.1f} us  {2.0*M*N*K/t/1e9:7.1f} TF/s",
          flush=True)


cublas("DS gemm1 (dense equiv)", 49152, 2816, 2048)
cublas("DS gemm2 (dense equiv)", 49152, 2048, 1408)
cublas("DS shared1", 8192, 5632, 2048)
cublas("DS shared2", 8192, 2048, 2816)
cublas("square 8192^3", 8192, 8192, 8192, iters=5)
bench("qwen3 gemm2 down (EP1)", 0, 1024, 128, 2048, 768, cg=2)
