"""Per-phase device timestamps of the fp64 small-batch router (router_f64_kernel) and its
prep kernel, from a library built with -DFSC_ROUTER_PROF into prof_lib/:

    FSC_LIB_OUT=prof_lib/libfsc.so FSC_BUILD_DIR=prof_build FSC_EXTRA_FLAGS=-DFSC_ROUTER_PROF \\
        python -m paper_2511_11505_b200.build --force
    python tools/router_f64_prof.py qwen3:512 scout:64
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["FSC_LIB"] = os.path.join(ROOT, "prof_lib", "libfsc.so")
import dataclasses

import numpy as np
import torch

import synth
from paper_2511_11505_b200 import Context
from tests.gpu_util import dev_f32

PHASES = ["start", "prologue (x0, W'0 issued)", "main loop", "cluster sync", "logits", "selected", "xn", "exit"]
NS = 148 * 64

torch.cuda.set_device(0)
for name in sys.argv[1:] or ["qwen3:512"]:
    base, _, tt = name.partition(":")
    shape = synth.CONFIGS[base]
    T = int(tt) if tt else shape.tokens
    w = synth.moe_weights(dataclasses.replace(shape, ffn=64, shared_ffn=0), seed=0)
    x = dev_f32(synth.tokens(shape, T=T))
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=64, shared_ffn=0, max_tokens=T)
    ctx.set_router_f64(True)
    xn = torch.empty(T, shape.d, dtype=torch.bfloat16, device="cuda")
    idx = torch.empty(T, shape.top_k, dtype=torch.int32, device="cuda")
    gw = torch.empty(T, shape.top_k, dtype=torch.float32, device="cuda")
    stamps = torch.zeros(max(T * shape.n_experts // 2, NS), dtype=torch.int64, device="cuda")
    g, wr = dev_f32(w.gamma), dev_f32(w.w_router)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(3):
        flush.fill_(1.0)
        stamps.zero_()
        stamps[NS - 2] = (1 << 62)
        ctx.op_router(x, g, wr, shape.top_k, xn, idx, gw, logits=stamps)
    torch.cuda.synchronize()
    allst = stamps.cpu().numpy().astype(np.float64)
    pq = allst[NS - 2: NS].copy()
    allst[NS - 2: NS] = 0
    s = allst[:NS].reshape(-1, 8)
    s = s[s[:, 0] > 0]
    t0 = min(s[:, 0].min(), pq[0])
    print(f"{name}: {len(s)} CTAs; prep kernel: first CTA start {(pq[0] - t0) / 1e3:6.1f} us, "
          f"last CTA done {(pq[1] - t0) / 1e3:6.1f} us")
    for k, ph in enumerate(PHASES):
        v = s[:, k]
        v = v[v > 0]
        if len(v):
            v = (v - t0) / 1e3
            print(f"  {ph:26s} n={len(v):4d} min {v.min():7.1f} us  median {np.median(v):7.1f}  max {v.max():7.1f}")
    ctx.close()
