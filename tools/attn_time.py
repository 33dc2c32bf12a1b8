"""Core attention (fsc_op_attention) time and TFLOP/s at the stack's shapes: CUDA events,
median of 20. FSC_ATTN_MMA_SYNC=1 selects the mma.sync kernel (A/B against tcgen05)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2511_11505_b200 import Context
from tests.gpu_util import dev_bf16

torch.cuda.set_device(0)
for name in sys.argv[1:] or ["dsv2lite", "qwen3"]:
    sh = synth.CONFIGS[name]
    T, Hq, Hkv, hd, S = sh.tokens, sh.n_heads, sh.n_kv_heads, sh.head_dim, sh.seq_len
    rng = np.random.default_rng(0)
    qkv = dev_bf16(synth.f32_to_bf16_bits(rng.standard_normal((T, (Hq + 2 * Hkv) * hd)).astype(np.float32)))
    out = torch.empty(T, Hq * hd, dtype=torch.bfloat16, device="cuda")
    ctx = Context(d=128, n_experts=4, top_k=2, ffn=128, shared_ffn=0, max_tokens=T)
    ts = []
    for i in range(25):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ctx.op_attention(qkv, out, Hq, Hkv, hd, S)
        b.record()
        torch.cuda.synchronize()
        if i >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    n = T // S
    flop = 4.0 * Hq * hd * n * S * (S + 1) / 2           # QK^T and PV over the causal pairs
    med = statistics.median(ts)
    print(f"{name}: T={T} Hq={Hq} Hkv={Hkv} hd={hd} seq={S}: {med:.1f} us, {flop / med / 1e6:.0f} TFLOP/s "
          f"(mma_sync={os.environ.get('FSC_ATTN_MMA_SYNC', '0')})")
    ctx.close()
