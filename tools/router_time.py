"""Router (K1) time per BASELINE config: CUDA events around fsc_op_router, median of 20."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses

import torch

import synth
from paper_2511_11505_b200 import Context
from tests.gpu_util import dev_f32

torch.cuda.set_device(0)
for name in sys.argv[1:] or ["dsv2lite", "qwen3", "scout"]:
    shape = synth.CONFIGS[name] if name in synth.CONFIGS else synth.decode_shape(*name.split(":"))
    T = shape.tokens if ":" not in name else int(name.split(":")[1])
    w = synth.moe_weights(dataclasses.replace(shape, ffn=64, shared_ffn=0), seed=0)
    x = dev_f32(synth.tokens(shape, T=T))
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=64, shared_ffn=0, max_tokens=T)
    if os.environ.get("FSC_ROUTER_I8") == "0":
        ctx.set_router_int8(False)   # the fp32 SIMT router (default: the fused tensor-core one)
    g, wr = dev_f32(w.gamma), dev_f32(w.w_router)
    xn = torch.empty(T, shape.d, dtype=torch.bfloat16, device="cuda")
    idx = torch.empty(T, shape.top_k, dtype=torch.int32, device="cuda")
    gw = torch.empty(T, shape.top_k, dtype=torch.float32, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    ts = []
    for i in range(25):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.op_router(x, g, wr, shape.top_k, xn, idx, gw)
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    flop = 2.0 * T * shape.d * shape.n_experts
    med = statistics.median(ts)
    print(f"{name} T={T}: router {med:.1f} us (min {min(ts):.1f}), {flop / med / 1e6:.1f} TFLOP/s fp32, "
          f"tc={os.environ.get('FSC_ROUTER_I8', '1')} cs={os.environ.get('FSC_ROUTER_CS', 'auto')}")
    ctx.close()
