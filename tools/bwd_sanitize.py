"""One tiny fsc_moe_backward under compute-sanitizer (memcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2511_11505_b200 import Context
from tests.gpu_util import dev_f32, moe_weights_dev

shape = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "tiny"]
T = 32
w = synth.moe_weights(shape, seed=3)
x = synth.tokens(shape, seed=3, T=T)
G = np.random.default_rng(0).standard_normal((T, shape.d)).astype(np.float32)
ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn, shared_ffn=shape.shared_ffn,
              max_tokens=T)
z = lambda *sh: torch.zeros(sh, dtype=torch.float32, device="cuda")  # noqa: E731
E, c, d = shape.n_experts, shape.ffn, shape.d
grads = {"dx": z(T, d), "dgamma": z(d), "dw_router": z(E, d), "dw1": z(E, c, d), "dw2": z(E, c, d), "dw3": z(E, d, c)}
ctx.moe_backward(moe_weights_dev(w), dev_f32(x), dev_f32(G), grads)
torch.cuda.synchronize()
print("ok", float(grads["dx"].abs().sum()))
