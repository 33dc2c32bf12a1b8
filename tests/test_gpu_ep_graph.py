"""EP=2 with the whole MoE layer captured as a CUDA graph and replayed: the
transport's epochs live in device memory, so replays synchronise correctly."""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth
from tests.test_gpu_ep import SHAPE, _free_port

pytestmark = pytest.mark.gpu


def _graph_worker(rank, world, port, outdir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2511_11505_b200 import Context
    from tests.gpu_util import dev_f32, moe_weights_dev
    e_loc = SHAPE.n_experts // world
    wd = moe_weights_dev(synth.moe_weights(SHAPE, seed=1, e0=rank * e_loc, e_loc=e_loc))
    xs = [synth.tokens(SHAPE, seed=10 + i, rank=rank) for i in range(3)]
    ctx = Context(d=SHAPE.d, n_experts=SHAPE.n_experts, top_k=SHAPE.top_k, ffn=SHAPE.ffn,
                  shared_ffn=SHAPE.shared_ffn, max_tokens=SHAPE.tokens, rank=rank, ep_size=world, device=0)
    ctx.connect()
    xin = dev_f32(xs[0])
    out = torch.empty_like(xin)
    eager = []
    for x in xs:
        xin.copy_(torch.from_numpy(x))
        ctx.moe_forward_blocking(wd, xin, out)
        torch.cuda.synchronize()
        eager.append(out.cpu().numpy().copy())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ctx.moe_forward_blocking(wd, xin, out)
    graphed = []
    for x in xs[::-1] + xs:          # several replays, inputs changed in place
        xin.copy_(torch.from_numpy(x))
        g.replay()
        torch.cuda.synchronize()
        graphed.append(out.cpu().numpy().copy())
    np.savez(os.path.join(outdir, f"g{rank}.npz"), eager=np.stack(eager), graphed=np.stack(graphed))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def test_ep2_cuda_graph_replay_matches_eager():
    from paper_2511_11505_b200 import build
    build.build()
    world = 2
    ctx = mp.get_context("spawn")
    port = _free_port()
    with tempfile.TemporaryDirectory() as td:
        ps = [ctx.Process(target=_graph_worker, args=(r, world, port, td)) for r in range(world)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(timeout=600)
        assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
        for r in range(world):
            z = np.load(os.path.join(td, f"g{r}.npz"))
            eager, graphed = z["eager"], z["graphed"]
            order = [2, 1, 0, 0, 1, 2]
            for gi, ei in enumerate(order):
                np.testing.assert_array_equal(graphed[gi], eager[ei])
