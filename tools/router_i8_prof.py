"""Per-phase device timestamps of the int8 tensor-core router kernel (build with -DFSC_ROUTER_PROF)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FSC_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "prof_lib", "libfsc.so")
import dataclasses

import numpy as np
import torch

import synth
from paper_2511_11505_b200 import Context
from tests.gpu_util import dev_f32

torch.cuda.set_device(0)
shape = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "dsv2lite"]
T = shape.tokens
w = synth.moe_weights(dataclasses.replace(shape, ffn=64, shared_ffn=0), seed=0)
x = dev_f32(synth.tokens(shape, T=T))
ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=64, shared_ffn=0, max_tokens=T)
ctx.set_router_int8(True)
xn = torch.empty(T, shape.d, dtype=torch.bfloat16, device="cuda")
idx = torch.empty(T, shape.top_k, dtype=torch.int32, device="cuda")
gw = torch.empty(T, shape.top_k, dtype=torch.float32, device="cuda")
nb = (T + 127) // 128 * 8
stamps = torch.zeros(nb * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    stamps.zero_()
    ctx.op_router(x, dev_f32(w.gamma), dev_f32(w.w_router), shape.top_k, xn, idx, gw, logits=stamps)
torch.cuda.synchronize()
s = stamps.view(-1, 8).cpu().numpy().astype(np.float64)
s = s[s[:, 0] > 0]
t0 = s[:, 0].min()
for k, name in enumerate(["start", "mma done", "partials+ticket", "combined", "selected", "refined"]):
    v = s[:, k]
    v = v[v > 0]
    if len(v):
        v = (v - t0) / 1e3
        print(f"{name:16s} n={len(v):4d} min {v.min():8.1f} us  median {np.median(v):8.1f}  max {v.max():8.1f}")
