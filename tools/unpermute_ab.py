"""A/B of the unpermute kernels (FSC_UNPERMUTE_ILP=0/1) on DS / Qwen3 shapes, CUDA events."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_11505_b200 import Context

torch.cuda.set_device(0)
for name, T, d, k in (("dsv2lite", 8192, 2048, 6), ("qwen3", 16384, 2048, 8)):
    ctx = Context(d=d, n_experts=128, top_k=k, ffn=64, shared_ffn=0, max_tokens=T)
    rng = np.random.default_rng(0)
    perm = torch.from_numpy(rng.permutation(T * k).astype(np.int32).reshape(T, k)).cuda()
    y = torch.randn(T * k, d, device="cuda").to(torch.bfloat16)
    w = torch.rand(T, k, device="cuda")
    resid = torch.randn(T, d, device="cuda")
    out = torch.empty_like(resid)
    flush = torch.empty(64 << 20, device="cuda")
    ts = []
    for i in range(25):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.op_unpermute(y, perm, w, resid, out)
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    byt = T * k * d * 2 + 2 * T * d * 4 + T * k * 8
    med = statistics.median(ts)
    print(f"{name}: unpermute {med:.1f} us = {byt / med / 1e3:.0f} GB/s  ilp={os.environ.get('FSC_UNPERMUTE_ILP', '1')}")
    ctx.close()
