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
    xs = [synth.tokens(shape, seed=3, rank=i, T=T) for i in range(5)]
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
    # pipelined: alternate two pinned buffer pairs, as a serving loop would
    ins = [torch.empty(T, shape.d).pin_memory() for _ in range(2)]
    outs = [torch.empty(T, shape.d).pin_memory() for _ in range(2)]
    got = []
    for i, x in enumerate(xs):
        j = i % 2
        if i >= 2:
            ctx.host_flush()                  # (only needed because we read outs[j] back below)
            got.append(outs[j].numpy().copy())
        ins[j].copy_(torch.from_numpy(x))
        ctx.moe_forward_host_async(wd, ins[j], outs[j])
    ctx.host_flush()
    got += [outs[(len(xs) - 2) % 2].numpy().copy(), outs[(len(xs) - 1) % 2].numpy().copy()]
    for g, r in zip(got, ref):
        np.testing.assert_array_equal(g, r)
    ctx.close()
