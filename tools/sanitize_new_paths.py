"""compute-sanitizer targets for the kernels added after the first sanitizer pass:
exact int8 tensor-core router (split and unsplit), split-d SIMT router (small T),
TMA gather4 GEMM producer, fused last-arriver unpermute, ragged A boxes, single-CTA
decode GEMMs. One process, small shapes (d = 256, E = 16, k = 1 / 2)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_11505_b200 import Context  # noqa: E402
from tests.gpu_util import dev_f32, moe_weights_dev  # noqa: E402

torch.cuda.set_device(0)
for k in (2, 1):
    sh = synth.MoeShape("san", d=256, n_experts=16, top_k=k, ffn=128, shared_ffn=128, tokens=300)
    T = sh.tokens
    ctx = Context(d=sh.d, n_experts=sh.n_experts, top_k=k, ffn=sh.ffn, shared_ffn=sh.shared_ffn, max_tokens=T)
    w = moe_weights_dev(synth.moe_weights(sh, seed=1))
    x = dev_f32(synth.tokens(sh, T=T))
    out = torch.empty_like(x)
    for i8 in (False, True):
        ctx.set_router_int8(i8)
        for gather in (False, True):
            ctx.set_gemm_gather(gather)
            for fused in (None, True):
                ctx.set_fused_unpermute(fused)
                for cg in (0, 1, 2):
                    ctx.set_gemm_cta_group(cg)
                    ctx.moe_forward_blocking(w, x, out)
    torch.cuda.synchronize()
    ctx.close()
print("sanitize new paths done")
