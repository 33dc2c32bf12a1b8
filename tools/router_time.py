"""Router (K1) device time per config: one CUDA graph holding [L2 flush, fsc_op_router] x N,
replayed; router time = (graph time - flush-only graph time) / N (no host launch overhead
inside the interval). Configs: BASELINE names or "<base>:<T>" decode batches.

  FSC_ROUTER_I8=0   the fp32 SIMT router        FSC_ROUTER_F64=0/1  fp64 router off / forced
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses

import torch

import synth
from paper_2511_11505_b200 import Context
from tests.gpu_util import dev_f32

N = 10
torch.cuda.set_device(0)


def graph_ms(fn, reps=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()                                    # warm-up (attributes, plans) outside the capture
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


for name in sys.argv[1:] or ["dsv2lite", "qwen3", "scout"]:
    shape = synth.CONFIGS[name] if name in synth.CONFIGS else synth.decode_shape(name.split(":")[0], 0)
    T = shape.tokens if ":" not in name else int(name.split(":")[1])
    w = synth.moe_weights(dataclasses.replace(shape, ffn=64, shared_ffn=0), seed=0)
    x = dev_f32(synth.tokens(shape, T=T))
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=64, shared_ffn=0, max_tokens=T)
    if os.environ.get("FSC_ROUTER_I8") == "0":
        ctx.set_router_int8(False)   # the fp32 SIMT router (default: the fused tensor-core one)
    if os.environ.get("FSC_ROUTER_F64") in ("0", "1"):
        ctx.set_router_f64(os.environ["FSC_ROUTER_F64"] == "1")   # default: auto (fp64 at T <= 1024)
    g, wr = dev_f32(w.gamma), dev_f32(w.w_router)
    xn = torch.empty(T, shape.d, dtype=torch.bfloat16, device="cuda")
    idx = torch.empty(T, shape.top_k, dtype=torch.int32, device="cuda")
    gw = torch.empty(T, shape.top_k, dtype=torch.float32, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")

    def flush_only():
        for i in range(N):
            flush.fill_(float(i))

    def with_router():
        for i in range(N):
            flush.fill_(float(i))
            ctx.op_router(x, g, wr, shape.top_k, xn, idx, gw)

    base = graph_ms(flush_only)
    for plan in (os.environ.get("FSC_PLANS") or "").split(";"):   # fp64 router plans "wt,cs;..." (A/B)
        if plan:
            os.environ["FSC_ROUTER_F64_PLAN"] = plan
        full = graph_ms(with_router)
        us = (full - base) / N * 1e3
        flop = 2.0 * T * shape.d * shape.n_experts
        print(f"{name} T={T}: router {us:.1f} us (graph, L2 flushed), {flop / us / 1e6:.2f} TFLOP/s, "
              f"tc={os.environ.get('FSC_ROUTER_I8', '1')} f64={os.environ.get('FSC_ROUTER_F64', 'auto')} "
              f"cs={os.environ.get('FSC_ROUTER_CS', 'auto')} plan={os.environ.get('FSC_ROUTER_F64_PLAN', 'auto')}")
    ctx.close()
