"""EP > 1 on the GPU: P processes (one EP rank each) share cuda:0 and talk
through the peer-memory transport (CUDA IPC), exactly the code path used with
one process per GPU over NVLink. Checks against the fp64 oracle's dispatch
simulation (moe_block_ep), EP invariance against an EP=1 run of the same
tokens (bitwise), and FarSkip == blocking."""
import dataclasses
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth
from oracle import moe as om
from tests.gpu_util import rel_l2

pytestmark = pytest.mark.gpu

SHAPE = synth.MoeShape("ep_small", d=256, n_experts=8, top_k=2, ffn=128, shared_ffn=128, tokens=96)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(target, world, *args, timeout=900):
    """Run target(rank, world, port, *args, outdir) in `world` spawned processes that
    share cuda:0; returns the per-rank npz dicts (file name f"{rank}.npz")."""
    ctx = mp.get_context("spawn")
    port = _free_port()
    with tempfile.TemporaryDirectory() as td:
        ps = [ctx.Process(target=target, args=(r, world, port, *args, td)) for r in range(world)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(timeout=timeout)
        codes = [p.exitcode for p in ps]
        for p in ps:
            if p.is_alive():
                p.kill()
        assert all(c == 0 for c in codes), codes
        return [dict(np.load(os.path.join(td, f"{r}.npz"))) for r in range(world)]


def _init_pg(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    return dist


def _worker(rank, world, port, shape, seed, skew, outdir):
    """One EP rank: the blocking layer in every schedule / combine variant, FarSkip twice,
    the zero-byte instrument and back, all on the same tokens; the debug outputs of the
    exchange (counts matrix, receive counts, receive map)."""
    dist = _init_pg(rank, world, port)
    from paper_2511_11505_b200 import (FSC_BLOCKING_REGULAR_PLUS, FSC_BLOCKING_SERIAL, FSC_COMBINE_FUSED,
                                       FSC_COMBINE_STREAM, Context, MoeDebug)
    from tests.gpu_util import dev_f32, moe_weights_dev
    e_loc = shape.n_experts // world
    w = synth.moe_weights(shape, seed=seed, e0=rank * e_loc, e_loc=e_loc)
    x = synth.tokens(shape, seed=seed, rank=rank, skew=skew)
    T, k, E = x.shape[0], shape.top_k, shape.n_experts
    ctx = Context(d=shape.d, n_experts=E, top_k=k, ffn=shape.ffn, shared_ffn=shape.shared_ffn, max_tokens=T,
                  rank=rank, ep_size=world, device=0)
    ctx.connect()
    wd = moe_weights_dev(w)
    xin = dev_f32(x)
    max_recv = world * T * min(k, e_loc)
    i32 = lambda *sh: torch.full(sh, -1, dtype=torch.int32, device="cuda")  # noqa: E731
    dbg = MoeDebug(topk_idx=i32(T, k), counts=i32(E), pos=i32(T, k), ep_counts=i32(world, E),
                   recv_counts=i32(e_loc), recv_src=i32(max_recv),
                   routed_out=torch.empty(T, shape.d, dtype=torch.float32, device="cuda"))
    res = {}

    def blocking(name, d=None):
        out = torch.empty_like(xin)
        ctx.moe_forward_blocking(wd, xin, out, d)
        res[name] = out

    blocking("out", dbg)                                  # default: stream combine, Regular+
    ctx.set_blocking_mode(FSC_BLOCKING_SERIAL)
    blocking("out_serial")
    ctx.set_blocking_mode(FSC_BLOCKING_REGULAR_PLUS)
    ctx.set_combine_mode(FSC_COMBINE_FUSED)
    blocking("out_fused")
    partial = xin.clone()
    h = ctx.moe_forward_farskip(wd, xin, partial)
    res["full_fused"] = torch.empty_like(xin)
    ctx.moe_wait(h, partial, res["full_fused"])
    ctx.set_combine_mode(FSC_COMBINE_STREAM)
    for i in range(2):                                    # epochs advance, buffers reused
        partial = xin.clone()
        h = ctx.moe_forward_farskip(wd, xin, partial)
        res[f"full{i}"] = torch.empty_like(xin)
        ctx.moe_wait(h, partial, res[f"full{i}"])
    ctx.set_a2a_zero_bytes(True)                          # measurement instrument: no payload, same flags
    blocking("zero")
    partial = xin.clone()
    h = ctx.moe_forward_farskip(wd, xin, partial)
    ctx.moe_wait(h, partial, torch.empty_like(xin))
    ctx.set_a2a_zero_bytes(False)
    blocking("out_after")
    torch.cuda.synchronize()
    save = {k2: v.cpu().numpy() for k2, v in res.items() if k2 != "zero"}
    save.update({f"dbg_{k2}": v.cpu().numpy() for k2, v in dbg.tensors.items()})
    np.savez(os.path.join(outdir, f"{rank}.npz"), **save)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


def check_ep(world, shape, seed=0, skew=0.0, ep1=True):
    """EP run vs the oracle's dispatch simulation: routing, the
    all-gathered counts matrix, receive counts and the full receive map bit-exactly;
    shared / routed / out within the BJ tolerance; every schedule and combine variant
    bitwise equal; and (ep1) bitwise equal to EP = 1 on the same tokens."""
    from paper_2511_11505_b200 import build
    build.build()
    res = _spawn(_worker, world, shape, seed, skew)
    xs = [synth.tokens(shape, seed=seed, rank=r, skew=skew) for r in range(world)]
    wfull = synth.moe_weights(shape, seed=seed)
    lay = om.layer_from_synth(wfull, shape.top_k)
    routers, n_excl = [], 0
    for r in range(world):
        ro, excl = om.adopt_router(lay, xs[r], res[r]["dbg_topk_idx"])    # R-1 (counted)
        routers.append(ro)
        n_excl += int(excl.sum())
    xns = [om.rmsnorm(x, lay.gamma) for x in xs]
    _, rc, dst_rank, dst_row, cnt = om.dispatch_sim(xns, [ro.idx for ro in routers], shape.n_experts, world)
    outs = om.moe_block_ep(xs, lay, world, routers=routers)
    e_loc = shape.n_experts // world
    T, k = xs[0].shape[0], shape.top_k
    for r in range(world):
        g = res[r]
        np.testing.assert_array_equal(g["dbg_topk_idx"], routers[r].idx)
        m = om.permutation_maps(routers[r].idx, shape.n_experts)
        np.testing.assert_array_equal(g["dbg_counts"], m.counts)
        np.testing.assert_array_equal(g["dbg_pos"], m.pos)
        np.testing.assert_array_equal(g["dbg_ep_counts"], cnt)                  # a5: counts exchange
        np.testing.assert_array_equal(g["dbg_recv_counts"], rc[r])              # per local expert
    for s_ in range(world):                                                     # a6: every copy's landing row
        pos = res[s_]["dbg_pos"]
        for t in range(T):
            for j in range(k):
                p, row = int(dst_rank[s_][t, j]), int(dst_row[s_][t, j])
                assert p == routers[s_].idx[t, j] // e_loc
                assert res[p]["dbg_recv_src"][row] == (s_ << 24) | int(pos[t, j]), (s_, t, j)
    for r in range(world):
        sh, ro, _ = outs[r]
        g = res[r]
        ref = (xs[r].astype(np.float64) + sh) + ro
        assert rel_l2(g["out"], ref) < 1e-2
        assert rel_l2(g["dbg_routed_out"], ro) < 1e-2
        for key in ("out_serial", "out_fused", "full_fused", "full0", "full1", "out_after"):
            np.testing.assert_array_equal(g[key], g["out"], err_msg=key)
    if ep1:   # EP invariance: the EP = 1 layer on each rank's tokens gives the same bits
        # (per rank block: the router's reduction split depends on the batch size T, so
        # the fp32 gates are batch-size invariant only up to rounding; the experts' rows
        # are independent of the other rows of the batch)
        from tests.gpu_util import dev_f32, moe_weights_dev
        from paper_2511_11505_b200 import Context
        c1 = Context(d=shape.d, n_experts=shape.n_experts, top_k=k, ffn=shape.ffn, shared_ffn=shape.shared_ffn,
                     max_tokens=T)
        w1 = moe_weights_dev(wfull)
        for r in range(world):
            xin = dev_f32(xs[r])
            o1 = torch.empty_like(xin)
            c1.moe_forward_blocking(w1, xin, o1)
            torch.cuda.synchronize()
            np.testing.assert_array_equal(res[r]["out"], o1.cpu().numpy())
        c1.close()
    loads = cnt.sum(axis=0)
    return n_excl, float(loads.max() / loads.mean())


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ep_small_matches_oracle_and_ep1(world):
    n_excl, _ = check_ep(world, SHAPE)
    print(f"EP={world}: R-1 exclusions {n_excl}")


# BASELINE d / E / k (configs[1..3]) at a few hundred tokens per rank, EP up to 8
DS_EP = dataclasses.replace(synth.CONFIGS["dsv2lite"], tokens=256)
QWEN_EP = dataclasses.replace(synth.CONFIGS["qwen3"], tokens=192)
SCOUT_EP = dataclasses.replace(synth.CONFIGS["scout"], tokens=128, ffn=1024, shared_ffn=1024)   # c reduced (memory)


@pytest.mark.parametrize("name,shape,world", [("ds", DS_EP, 2), ("ds", DS_EP, 8), ("qwen3", QWEN_EP, 8),
                                              ("scout", SCOUT_EP, 8)])
def test_ep_baseline_shapes(name, shape, world):
    n_excl, imb = check_ep(world, shape, seed=1, ep1=(name != "scout"))
    print(f"{name} EP={world}: R-1 exclusions {n_excl}, max/mean expert load {imb:.2f}")


@pytest.mark.parametrize("world,skew", [(4, synth.SKEW_DEFAULT), (8, 0.5)])
def test_ep_skewed_load(world, skew):
    """Skewed expert load: the same hot experts on every rank, so the
    receive side is ragged (some ranks get far more rows, some local experts none)."""
    n_excl, imb = check_ep(world, DS_EP, seed=2, skew=skew, ep1=False)
    assert imb > (1.4 if skew < 0.3 else 3.0), imb
    print(f"skew {skew} EP={world}: max/mean expert load {imb:.2f}, R-1 exclusions {n_excl}")


def _stack_worker(rank, world, port, shape, seed, L, fuzz, outdir):
    dist = _init_pg(rank, world, port)
    from paper_2511_11505_b200 import FSC_BLOCKING, FSC_HYBRID, FSC_OVERLAPPED, FSC_REGULAR, Context
    from tests.gpu_util import attn_weights_dev, dev_f32, moe_weights_dev
    e_loc = shape.n_experts // world
    mw = [moe_weights_dev(synth.moe_weights(shape, seed=seed, layer=k, e0=rank * e_loc, e_loc=e_loc))
          for k in range(L)]
    aw = [attn_weights_dev(synth.attn_weights(shape, seed=seed, layer=k)) for k in range(L)]
    x = synth.tokens(shape, seed=seed, rank=rank)
    T = x.shape[0]
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=T, rank=rank, ep_size=world, device=0)
    ctx.connect()
    res = {}
    runs = [("hyb", [FSC_HYBRID] * L), ("mix", [FSC_REGULAR] + [FSC_HYBRID] * (L - 1)), ("reg", [FSC_REGULAR] * L)]
    for name, modes in runs:
        for sname, sched in (("blk", FSC_BLOCKING), ("ovl", FSC_OVERLAPPED)):
            o0 = dev_f32(x)
            oL = torch.empty_like(o0)
            ctx.layer_stack_forward(aw, mw, T, shape.seq_len, modes, sched, o0, oL)
            torch.cuda.synchronize()
            res[f"{name}_{sname}"] = oL.cpu().numpy()
    for seed_f in range(1, fuzz + 1):   # random stream delays (rank-dependent): same bits
        ctx.set_delay_fuzz(1000 * rank + seed_f, 300_000)
        for name, modes in runs[:2]:
            o0 = dev_f32(x)
            oL = torch.empty_like(o0)
            ctx.layer_stack_forward(aw, mw, T, shape.seq_len, modes, FSC_OVERLAPPED, o0, oL)
            torch.cuda.synchronize()
            res[f"{name}_fuzz{seed_f}"] = oL.cpu().numpy()
    ctx.set_delay_fuzz(0, 0)
    np.savez(os.path.join(outdir, f"{rank}.npz"), **res)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


STACK_SHAPE = synth.MoeShape("ep_stack", d=256, n_experts=8, top_k=2, ffn=128, shared_ffn=128, tokens=128,
                             n_heads=4, n_kv_heads=2, head_dim=64, seq_len=64)


@pytest.mark.parametrize("world", [2, 8])
def test_ep_stack_schedules_bitwise_and_ep_invariant(world):
    """EP layer stack: BLOCKING == OVERLAPPED for Hybrid, mixed and Regular wirings (the
    comm stream / event ordering changes nothing), also under random per-rank stream
    delays (spin kernels in front of every stage), and all equal the EP = 1 stack on the
    same tokens."""
    from paper_2511_11505_b200 import FSC_HYBRID, FSC_OVERLAPPED, FSC_REGULAR, Context, build
    from tests.gpu_util import attn_weights_dev, dev_f32, moe_weights_dev
    build.build()
    L = 3
    res = _spawn(_stack_worker, world, STACK_SHAPE, 0, L, 2)
    for r in range(world):
        for name in ("hyb", "mix", "reg"):
            np.testing.assert_array_equal(res[r][f"{name}_blk"], res[r][f"{name}_ovl"])
        for name in ("hyb", "mix"):
            for f in (1, 2):
                np.testing.assert_array_equal(res[r][f"{name}_fuzz{f}"], res[r][f"{name}_ovl"])
    # EP=1 on the concatenated tokens (sequences never straddle ranks: T % seq_len == 0)
    sh = STACK_SHAPE
    X = np.concatenate([synth.tokens(sh, seed=0, rank=r) for r in range(world)])
    c1 = Context(d=sh.d, n_experts=sh.n_experts, top_k=sh.top_k, ffn=sh.ffn, shared_ffn=sh.shared_ffn,
                 max_tokens=X.shape[0])
    mw = [moe_weights_dev(synth.moe_weights(sh, seed=0, layer=k)) for k in range(L)]
    aw = [attn_weights_dev(synth.attn_weights(sh, seed=0, layer=k)) for k in range(L)]
    for name, modes in (("hyb", [FSC_HYBRID] * L), ("mix", [FSC_REGULAR] + [FSC_HYBRID] * (L - 1)),
                        ("reg", [FSC_REGULAR] * L)):
        o0 = dev_f32(X)
        oL = torch.empty_like(o0)
        c1.layer_stack_forward(aw, mw, X.shape[0], sh.seq_len, modes, FSC_OVERLAPPED, o0, oL)
        torch.cuda.synchronize()
        o1 = oL.cpu().numpy()
        for r in range(world):
            np.testing.assert_array_equal(res[r][f"{name}_ovl"], o1[r * sh.tokens:(r + 1) * sh.tokens])
    c1.close()


# ----------------------------------------------------------------------------- EP all-reduce (inference variant)
def _ar_worker(rank, world, port, shape, seed, outdir):
    """every rank holds the SAME tokens; local experts only; all-reduce."""
    dist = _init_pg(rank, world, port)
    from paper_2511_11505_b200 import FSC_EP_ALLREDUCE, Context, MoeDebug
    from tests.gpu_util import dev_f32, moe_weights_dev
    e_loc = shape.n_experts // world
    w = synth.moe_weights(shape, seed=seed, e0=rank * e_loc, e_loc=e_loc)
    x = synth.tokens(shape, seed=seed, rank=0)            # replicated activations
    T = x.shape[0]
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=T, rank=rank, ep_size=world, device=0)
    ctx.set_ep_mode(FSC_EP_ALLREDUCE)
    ctx.connect()
    wd = moe_weights_dev(w)
    xin = dev_f32(x)
    outs = []
    for _ in range(2):                                    # epochs advance, buffers reused
        out = torch.empty_like(xin)
        dbg = MoeDebug(topk_idx=torch.empty(T, shape.top_k, dtype=torch.int32, device="cuda"),
                       routed_out=torch.empty(T, shape.d, dtype=torch.float32, device="cuda"))
        ctx.moe_forward_blocking(wd, xin, out, dbg)
        outs.append(out)
    fulls = []
    for _ in range(2):
        partial = xin.clone()
        h = ctx.moe_forward_farskip(wd, xin, partial)
        full = torch.empty_like(xin)
        ctx.moe_wait(h, partial, full)
        fulls.append(full)
    torch.cuda.synchronize()
    np.savez(os.path.join(outdir, f"{rank}.npz"), out0=outs[0].cpu().numpy(), out1=outs[1].cpu().numpy(),
             idx=dbg.tensors["topk_idx"].cpu().numpy(), routed=dbg.tensors["routed_out"].cpu().numpy(),
             full0=fulls[0].cpu().numpy(), full1=fulls[1].cpu().numpy())
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_ep_allreduce_variant(world):
    """Inference variant: replicated tokens, EP-sharded experts, routed
    partials all-reduced over peer memory. Every rank ends with the SAME output (bit
    for bit), equal to the dense MoE block (oracle) within the BJ tolerance and to
    the EP=1 result within fp32 re-association; FarSkip (all-reduce in flight, waited
    one sub-block later) == blocking bitwise; repeated calls identical."""
    from paper_2511_11505_b200 import Context, build
    from tests.gpu_util import dev_f32, moe_weights_dev
    build.build()
    res = _spawn(_ar_worker, world, SHAPE, 0)
    x = synth.tokens(SHAPE, seed=0, rank=0)
    wfull = synth.moe_weights(SHAPE, seed=0)
    lay = om.layer_from_synth(wfull, SHAPE.top_k)
    sh, ro, rt, _ = om.moe_block_allreduce(x, lay, world)
    ref = (x.astype(np.float64) + sh) + ro
    for r in range(world):
        np.testing.assert_array_equal(res[r]["idx"], rt.idx)
        assert rel_l2(res[r]["out0"], ref) < 1e-2
        assert rel_l2(res[r]["routed"], ro) < 1e-2
        for key in ("out1", "full0", "full1"):
            np.testing.assert_array_equal(res[r][key], res[r]["out0"])
        np.testing.assert_array_equal(res[r]["out0"], res[0]["out0"])   # replicated result
    c1 = Context(d=SHAPE.d, n_experts=SHAPE.n_experts, top_k=SHAPE.top_k, ffn=SHAPE.ffn,
                 shared_ffn=SHAPE.shared_ffn, max_tokens=x.shape[0])
    xin = dev_f32(x)
    o1 = torch.empty_like(xin)
    c1.moe_forward_blocking(moe_weights_dev(wfull), xin, o1)
    torch.cuda.synchronize()
    c1.close()
    assert rel_l2(res[0]["out0"], o1.cpu().numpy()) < 1e-6


# ----------------------------------------------------------------------------- FP8 dispatch payload (NEXT-4)
def _fp8_worker(rank, world, port, shape, seed, outdir):
    dist = _init_pg(rank, world, port)
    from paper_2511_11505_b200 import Context, MoeDebug
    from tests.gpu_util import dev_f32, moe_weights_dev
    e_loc = shape.n_experts // world
    w = synth.moe_weights(shape, seed=seed, e0=rank * e_loc, e_loc=e_loc)
    x = synth.tokens(shape, seed=seed, rank=rank)
    T = x.shape[0]
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=T, rank=rank, ep_size=world, device=0)
    ctx.set_dispatch_fp8(True)
    ctx.connect()
    wd = moe_weights_dev(w)
    xin = dev_f32(x)
    out = torch.empty_like(xin)
    dbg = MoeDebug(topk_idx=torch.empty(T, shape.top_k, dtype=torch.int32, device="cuda"),
                   routed_out=torch.empty(T, shape.d, dtype=torch.float32, device="cuda"))
    ctx.moe_forward_blocking(wd, xin, out, dbg)
    partial = xin.clone()
    h = ctx.moe_forward_farskip(wd, xin, partial)
    full = torch.empty_like(xin)
    ctx.moe_wait(h, partial, full)
    torch.cuda.synchronize()
    np.savez(os.path.join(outdir, f"{rank}.npz"), out=out.cpu().numpy(), full=full.cpu().numpy(),
             idx=dbg.tensors["topk_idx"].cpu().numpy(), routed=dbg.tensors["routed_out"].cpu().numpy())
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 8])
def test_ep_fp8_dispatch_payload(world):
    """FP8 e4m3 dispatch payload (per-128-column scales): the routed output matches the
    oracle's moe_block_ep_fp8 (same quantisation step, fp64 experts) within the BJ
    tolerance, and the exact (bf16-payload) oracle only within the FP8 error; FarSkip ==
    blocking bitwise."""
    from paper_2511_11505_b200 import build
    build.build()
    res = _spawn(_fp8_worker, world, SHAPE, 0)
    xs = [synth.tokens(SHAPE, seed=0, rank=r) for r in range(world)]
    lay = om.layer_from_synth(synth.moe_weights(SHAPE, seed=0), SHAPE.top_k)
    q = om.moe_block_ep_fp8(xs, lay, world)
    exact = om.moe_block_ep(xs, lay, world)
    for r in range(world):
        sh, ro, rt = q[r]
        np.testing.assert_array_equal(res[r]["idx"], rt.idx)
        assert rel_l2(res[r]["routed"], ro) < 1e-2
        assert rel_l2(res[r]["out"], (xs[r].astype(np.float64) + sh) + ro) < 1e-2
        assert rel_l2(res[r]["routed"], exact[r][1]) < 8e-2
        np.testing.assert_array_equal(res[r]["full"], res[r]["out"])


def _tp_slice(a, rank, world):
    """Rank's head slice of the attention weights (TP, RowParallel o-projection):
    q heads [r Hq/P, (r+1) Hq/P), kv heads [r Hkv/P, ...), the matching w_qkv rows and
    w_o columns."""
    hq, hkv, hd = a.n_heads // world, a.n_kv_heads // world, a.head_dim
    q = a.w_qkv[:a.n_heads * hd]
    kk = a.w_qkv[a.n_heads * hd:(a.n_heads + a.n_kv_heads) * hd]
    v = a.w_qkv[(a.n_heads + a.n_kv_heads) * hd:]
    w_qkv = np.concatenate([q[rank * hq * hd:(rank + 1) * hq * hd], kk[rank * hkv * hd:(rank + 1) * hkv * hd],
                            v[rank * hkv * hd:(rank + 1) * hkv * hd]])
    w_o = np.ascontiguousarray(a.w_o[:, rank * hq * hd:(rank + 1) * hq * hd])
    return dataclasses.replace(a, w_qkv=np.ascontiguousarray(w_qkv), w_o=w_o, n_heads=hq, n_kv_heads=hkv)


CACHE_KEYS = ("attn_in", "mlp_in", "attn_out", "shared_out", "routed_out", "o")


def _ar_stack_worker(rank, world, port, shape, seed, L, outdir):
    dist = _init_pg(rank, world, port)
    from paper_2511_11505_b200 import FSC_BLOCKING, FSC_EP_ALLREDUCE, FSC_HYBRID, FSC_OVERLAPPED, Context
    from tests.gpu_util import attn_weights_dev, dev_f32, moe_weights_dev
    e_loc = shape.n_experts // world
    mw = [moe_weights_dev(synth.moe_weights(shape, seed=seed, layer=k, e0=rank * e_loc, e_loc=e_loc))
          for k in range(L)]
    aw = [attn_weights_dev(_tp_slice(synth.attn_weights(shape, seed=seed, layer=k), rank, world))
          for k in range(L)]                            # tensor-parallel attention: this rank's heads
    x = synth.tokens(shape, seed=seed, rank=0)          # replicated activations
    T = x.shape[0]
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=T, rank=rank, ep_size=world, device=0)
    ctx.set_ep_mode(FSC_EP_ALLREDUCE)
    ctx.connect()
    res = {}
    for sname, sched in (("blk", FSC_BLOCKING), ("ovl", FSC_OVERLAPPED)):
        o0 = dev_f32(x)
        oL = torch.empty_like(o0)
        cache = [{k2: torch.full_like(o0, float("nan")) for k2 in CACHE_KEYS} for _ in range(L)]
        ctx.layer_stack_forward(aw, mw, T, shape.seq_len, [FSC_HYBRID] * L, sched, o0, oL, cache)
        torch.cuda.synchronize()
        res[sname] = oL.cpu().numpy()
        if sname == "ovl":
            for k in range(L):
                for k2 in CACHE_KEYS:
                    res[f"c{k}_{k2}"] = cache[k][k2].cpu().numpy()
    np.savez(os.path.join(outdir, f"{rank}.npz"), **res)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


TP_SHAPE = synth.MoeShape("ep_tp_stack", d=256, n_experts=8, top_k=2, ffn=128, shared_ffn=128, tokens=128,
                          n_heads=8, n_kv_heads=4, head_dim=32, seq_len=64)


@pytest.mark.parametrize("world", [2, 4])
def test_ep_allreduce_stack(world):
    """FarSkip (Hybrid) stack in the all-reduce inference variant at EP = TP = P
    (P:215-217): experts EP-sharded and the MoE partials all-reduced, attention heads
    TP-sharded and the o-projection partials all-reduced on a second channel, each
    waited only one sub-block later. Every rank ends with the same bits, BLOCKING ==
    OVERLAPPED, every layer matches the fp64 oracle teacher-forced on the GPU's own layer
    inputs within the BJ tolerance, and the P:175 identity
    mlp-in_k = attn-in_k + routed_{k-1} holds bitwise on the GPU's activations."""
    from oracle import stack as ost
    from paper_2511_11505_b200 import build
    from tests.test_gpu_stack import AWf
    build.build()
    L, sh = 3, TP_SHAPE
    res = _spawn(_ar_stack_worker, world, sh, 0, L)
    for r in range(world):
        np.testing.assert_array_equal(res[r]["blk"], res[r]["ovl"])
        np.testing.assert_array_equal(res[r]["ovl"], res[0]["ovl"])
    X = synth.tokens(sh, seed=0, rank=0)
    g = res[0]
    lays = [om.layer_from_synth(synth.moe_weights(sh, seed=0, layer=k), sh.top_k) for k in range(L)]
    awf = [AWf(synth.attn_weights(sh, seed=0, layer=k)) for k in range(L)]
    teacher = [(g[f"c{k}_attn_in"], g[f"c{k}_mlp_in"]) for k in range(L)]
    ref = ost.stack_forward(X, awf, lays, [ost.HYBRID] * L, sh.seq_len, teacher_inputs=teacher)
    for k in range(L):
        for key, rv in (("attn_out", ref[k].attn_out), ("shared_out", ref[k].shared_out),
                        ("routed_out", ref[k].routed_out), ("o", ref[k].o)):
            e = rel_l2(g[f"c{k}_{key}"], rv)
            assert e < 1e-2, (k, key, e)
    np.testing.assert_array_equal(g["c0_attn_in"], X)
    for k in range(1, L):
        np.testing.assert_array_equal(g[f"c{k}_mlp_in"],
                                      (g[f"c{k}_attn_in"] + g[f"c{k - 1}_routed_out"]).astype(np.float32))
        np.testing.assert_array_equal(g[f"c{k}_mlp_in"], g[f"c{k - 1}_o"])
