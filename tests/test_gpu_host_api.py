"""Host-buffer entry points (the e2e path): synchronous and pipelined."""
import numpy as np
import pytest
import torch

import synth
from tests.gpu_util import dev_f32, moe_weights_dev

pytestmark = pytest.mark.gpu


def test_host_entry_points_match_device_path():
    from paper_2511_11505_b200 import Context, build
    build.build()
    shape = synth.CONFIGS["dsv2lite"]
    T = 512
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=T)
    wd = moe_weights_dev(synth.moe_weights(shape, seed=3))
    xs = [synth.tokens(shape, seed=3, rank=i, T=T) for i in range(7)]
    ref = []
    for x in xs:
        xin = dev_f32(x)
        out = torch.empty_like(xin)
        ctx.moe_forward_blocking(wd, xin, out)
        ref.append(out.cpu().numpy())
    # synchronous host entry
    xh = torch.from_numpy(xs[0]).pin_memory()
    oh = torch.empty_like(xh).pin_memory()
    ctx.moe_forward_blocking_host(wd, xh, oh)
    np.testing.assert_array_equal(oh.numpy(), ref[0])
    # pipelined, as a serving loop would: four pinned buffer pairs in rotation, so that a
    # pair is rewritten only after the call three later has returned (fsc.h contract)
    ins = [torch.empty(T, shape.d).pin_memory() for _ in range(4)]
    outs = [torch.empty(T, shape.d).pin_memory() for _ in range(4)]
    got = [None] * len(xs)
    for i, x in enumerate(xs):
        j = i % 4
        if i >= 4:
            got[i - 4] = outs[j].numpy().copy()   # call i - 4 is complete: call i - 1 has returned
        ins[j].copy_(torch.from_numpy(x))
        ctx.moe_forward_host_async(wd, ins[j], outs[j])
    ctx.host_flush()
    for i in range(max(0, len(xs) - 4), len(xs)):
        got[i] = outs[i % 4].numpy().copy()
    for g, r in zip(got, ref):
        np.testing.assert_array_equal(g, r)
    ctx.close()
