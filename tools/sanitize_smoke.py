"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
tiny MoE blocking + FarSkip and a 2-layer tiny stack, cta_group 1 and 2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_11505_b200 import FSC_HYBRID, FSC_OVERLAPPED, FSC_REGULAR, Context  # noqa: E402
from tests.gpu_util import attn_weights_dev, dev_f32, moe_weights_dev  # noqa: E402

torch.cuda.set_device(0)
shape = synth.CONFIGS["tiny"]
T = 64
ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn, shared_ffn=128,
              max_tokens=T)
import dataclasses  # noqa: E402
sh = dataclasses.replace(shape, shared_ffn=128)
for cg in ([int(a) for a in sys.argv[1:]] or [2, 1]):
    ctx.set_gemm_cta_group(cg)
    w = moe_weights_dev(synth.moe_weights(sh, seed=0))
    x = dev_f32(synth.tokens(sh, T=T))
    out = torch.empty_like(x)
    ctx.moe_forward_blocking(w, x, out)
    p = x.clone()
    h = ctx.moe_forward_farskip(w, x, p)
    ctx.moe_wait(h, p, p)
    mws = [moe_weights_dev(synth.moe_weights(sh, seed=0, layer=k)) for k in range(2)]
    aws = [attn_weights_dev(synth.attn_weights(sh, seed=0, layer=k)) for k in range(2)]
    oL = torch.empty_like(x)
    ctx.layer_stack_forward(aws, mws, T, 16, [FSC_REGULAR, FSC_HYBRID], FSC_OVERLAPPED, x, oL)
    torch.cuda.synchronize()
print("sanitize smoke done")
