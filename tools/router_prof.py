"""Per-phase device timestamps of the router kernel (build with -DFSC_ROUTER_PROF)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FSC_LIB"] = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "prof_lib", "libfsc.so")
import numpy as np, torch
import synth
from paper_2511_11505_b200 import Context
from tests.gpu_util import dev_f32
torch.cuda.set_device(0)
shape = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "dsv2lite"]
T = shape.tokens
w = synth.moe_weights(__import__("dataclasses").replace(shape, ffn=64, shared_ffn=0), seed=0)
x = dev_f32(synth.tokens(shape, T=T))
ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=64, shared_ffn=0, max_tokens=T)
xn = torch.empty(T, shape.d, dtype=torch.bfloat16, device="cuda")
idx = torch.empty(T, shape.top_k, dtype=torch.int32, device="cuda")
gw = torch.empty(T, shape.top_k, dtype=torch.float32, device="cuda")
nb = (T + 31) // 32
stamps = torch.zeros(nb * 8, dtype=torch.int64, device="cuda")
for _ in range(3):
    ctx.op_router(x, dev_f32(w.gamma), dev_f32(w.w_router), shape.top_k, xn, idx, gw, logits=stamps)
torch.cuda.synchronize()
s = stamps.view(nb, 8).cpu().numpy().astype(np.float64)
t0 = s[:, 0].min()
for k, name in enumerate(["start", "loop done", "lg done", "select done", "xn done"]):
    v = (s[:, k] - t0) / 1e3
    print(f"{name:14s} min {v.min():8.1f} us  median {np.median(v):8.1f}  max {v.max():8.1f}")
d = (s[:, 1:5] - s[:, 0:4]) / 1e3
for k, name in enumerate(["loop", "reduce", "select", "xn"]):
    print(f"per-block {name:5s}: median {np.median(d[:, k]):7.1f} us  max {d[:, k].max():7.1f}")
