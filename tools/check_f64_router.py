"""Self-checking sweep of the round-2 decode paths (compute-sanitizer is closed on this pool):
the fp64 router at every tile height and cluster size, DMMA and DFMA contractions, E padded
to 32 / 64 / 128, a ragged T, and the EP = 1 permute by source token and by destination row,
inside the MoE forward. Output buffers are NaN-poisoned before every call (an unwritten
element shows); every variant must select the same experts and give the same output up to
the fp32 rounding of the gates (the fp64 sums differ in order between plans)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2511_11505_b200 import Context  # noqa: E402
from tests.gpu_util import dev_f32, moe_weights_dev  # noqa: E402

torch.cuda.set_device(0)
n = 0
for E, k in ((16, 1), (64, 6), (128, 8)):
    sh = synth.MoeShape("chk", d=512, n_experts=E, top_k=k, ffn=128, shared_ffn=128, tokens=45)
    T = sh.tokens
    ctx = Context(d=sh.d, n_experts=E, top_k=k, ffn=sh.ffn, shared_ffn=sh.shared_ffn, max_tokens=T)
    ctx.set_router_f64(True)
    w = moe_weights_dev(synth.moe_weights(sh, seed=1))
    x = dev_f32(synth.tokens(sh, T=T))
    ref = None
    for simt in ("0", "1"):
        os.environ["FSC_ROUTER_F64_SIMT"] = simt
        for plan in ("1,1", "2,2", "4,4", "1,8", "2,8", "4,8"):
            os.environ["FSC_ROUTER_F64_PLAN"] = plan
            for gather in ("0", "1"):
                os.environ["FSC_PERMUTE_GATHER"] = gather
                out = torch.full_like(x, float("nan"))
                ctx.moe_forward_blocking(w, x, out)
                o = out.cpu().numpy()
                assert np.all(np.isfinite(o)), (E, simt, plan, gather)
                if ref is None:
                    ref = o
                else:
                    err = np.linalg.norm(o - ref) / np.linalg.norm(ref)
                    assert err < 1e-5, (E, simt, plan, gather, err)
                n += 1
    ctx.close()
print(f"fp64 router / permute sweep: {n} variants consistent")
