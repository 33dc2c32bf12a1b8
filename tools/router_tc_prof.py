"""Per-phase device timestamps of the fused tensor-core router kernel (router_tc_kernel),
from a library built with -DFSC_ROUTER_PROF into prof_lib/:

    FSC_LIB_OUT=prof_lib/libfsc.so FSC_BUILD_DIR=prof_build FSC_EXTRA_FLAGS=-DFSC_ROUTER_PROF \
        python -m paper_2511_11505_b200.build --force
    python tools/router_tc_prof.py dsv2lite qwen3:512
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

PHASES = ["start", "phase-1 stats", "cluster stats", "phase-2 conv", "MMAs done", "logits", "selected", "refined"]

torch.cuda.set_device(0)
for name in sys.argv[1:] or ["dsv2lite"]:
    base, _, tt = name.partition(":")
    shape = synth.CONFIGS[base]
    T = int(tt) if tt else shape.tokens
    w = synth.moe_weights(dataclasses.replace(shape, ffn=64, shared_ffn=0), seed=0)
    x = dev_f32(synth.tokens(shape, T=T))
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=64, shared_ffn=0, max_tokens=T)
    xn = torch.empty(T, shape.d, dtype=torch.bfloat16, device="cuda")
    idx = torch.empty(T, shape.top_k, dtype=torch.int32, device="cuda")
    gw = torch.empty(T, shape.top_k, dtype=torch.float32, device="cuda")
    stamps = torch.zeros(max(T * shape.n_experts // 2, 148 * 8 * 8), dtype=torch.int64, device="cuda")
    g, wr = dev_f32(w.gamma), dev_f32(w.w_router)
    for _ in range(3):
        stamps.zero_()
        ctx.op_router(x, g, wr, shape.top_k, xn, idx, gw, logits=stamps)
    torch.cuda.synchronize()
    allst = stamps.cpu().numpy().astype(np.float64)
    qw = allst[148 * 8 * 8 - 2: 148 * 8 * 8].copy()
    allst[148 * 8 * 8 - 2: 148 * 8 * 8] = 0
    s = allst.reshape(-1, 8)
    s = s[s[:, 0] > 0]
    t0 = s[:, 0].min()
    print(f"  quant_w kernel: start {(qw[0] - t0) / 1e3:7.1f} us, last CTA done {(qw[1] - t0) / 1e3:7.1f} us")
    print(f"{name}: {len(s)} CTAs")
    for k, ph in enumerate(PHASES):
        v = s[:, k]
        v = v[v > 0]
        if len(v):
            v = (v - t0) / 1e3
            print(f"  {ph:14s} n={len(v):4d} min {v.min():7.1f} us  median {np.median(v):7.1f}  max {v.max():7.1f}")
    ctx.close()
