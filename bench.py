#!/usr/bin/env python3
"""Benchmark of the FarSkip-Collective MoE layer forward (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config dsv2lite] [--impl reference]

A step is one pass of the whole hot path (RMSNorm +
router + top-k, permutation maps, permute/dispatch, SwiGLU grouped GEMM, down
GEMM, combine, gate-weighted unpermute + residual, shared expert) over one
batch of T synthetic tokens per rank, with inputs resident in HBM. N > 1 runs
one process per GPU (torchrun); the per-rank workload is fixed (weak scaling)
and the value is the tokens all ranks processed / max-over-ranks device time.

Prints ONE JSON line on rank 0. ``--impl reference`` times the CPU fp64 oracle
(oracle/, the only reference this tier has) on a bounded token sample of the
same workload and prints the same line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "MoE-layer tokens/s at 1/2/4/8 B200; exposed all-to-all us/layer FarSkip vs blocking"
UNIT = "tokens/s"
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return j, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def workload_config(shape, ep, n_gpus, schedule):
    regime = "decode" if "_decode" in shape.name else "prefill"
    return {"workload": f"{shape.name}_moe_layer" + ("" if regime == "decode" else "_prefill"), "regime": regime, "d": shape.d, "n_experts": shape.n_experts,
            "top_k": shape.top_k, "ffn": shape.ffn, "shared_ffn": shape.shared_ffn,
            "tokens_per_rank": shape.tokens, "global_tokens": shape.tokens * n_gpus, "ep": ep,
            "schedule": schedule, "parallelism": f"ep{ep}" + (f"-x{n_gpus // ep}replicas" if n_gpus > ep else ""),
            "l2": "flushed (256 MiB write) before every timed step; per-step working set > L2",
            "launch": "one CUDA-graph replay per step (captured fsc_moe_forward_blocking)",
            "data": "synthetic seeded N(0,1) tokens, random-init weights (SURVEY §8(d) recipe)"}


def get_shape(name):
    """BASELINE configs by name; '<base>_decode<T>' is configs[4] (decode regime)."""
    if name in synth.CONFIGS:
        return synth.CONFIGS[name]
    if "_decode" in name:
        base, t = name.split("_decode")
        return synth.decode_shape(base, int(t))
    raise SystemExit(f"unknown config {name}")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """Polls NVML (SM clock, max SM clock, clock-event reasons) every ~2 ms in a
    thread while the timed region runs; falls back to nvidia-smi if NVML fails."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap",
               "hw_power_brake": "nvmlClocksEventReasonHwPowerBrakeSlowdown"}

    def __init__(self, index=0, period_s=0.002):
        self.index = index
        self.period = period_s
        self.rows = []
        self.stop = threading.Event()
        self.err = None

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.index]) if vis else self.index
            self.h = N.nvmlDeviceGetHandleByIndex(idx)
            self.N = N
            self.max_sm = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # noqa: BLE001
            self.err = repr(e)
        return self

    def _run(self):
        N = self.N
        while not self.stop.is_set():
            try:
                sm = N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)
                rs = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception as e:  # noqa: BLE001
                self.err = repr(e)
                return
            time.sleep(self.period)

    def __exit__(self, *a):
        self.stop.set()
        if getattr(self, "t", None):
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0, "error": self.err}
        N = self.N
        sm = [r[0] for r in self.rows]
        reasons = sorted({name for _, rs in self.rows for name, attr in self.REASONS.items()
                          if rs & getattr(N, attr, 0)})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_sm, "sm_mhz_min": min(sm),
                "reasons": reasons, "samples": len(sm), "source": "NVML, ~2 ms polling during the timed region"}


# ----------------------------------------------------------------------------- oracle baseline
def oracle_tokens_per_s(shape, budget_s=12.0, seed=0, max_tokens=None):
    """The fp64 oracle (as it stands) on a bounded token sample of the workload.
    The MoE block is token-independent, so a sample of tokens is the same
    computation per token as the full batch."""
    from threadpoolctl import threadpool_info

    from oracle import moe as om
    w = synth.moe_weights(shape, seed=seed)
    lay = om.layer_from_synth(w, shape.top_k)
    del w
    cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    x = synth.tokens(shape, seed=seed, T=shape.tokens)
    n, done, t_used = 64, 0, 0.0
    while t_used < budget_s and done < shape.tokens and (max_tokens is None or done < max_tokens):
        n = min(n, shape.tokens - done)
        t0 = time.perf_counter()
        sh, ro, _ = om.moe_block(x[done:done + n], lay)
        _ = (x[done:done + n].astype(np.float64) + sh) + ro
        dt = time.perf_counter() - t0
        t_used += dt
        done += n
        n = int(min(4096, max(64, n * 2 if dt < budget_s / 8 else n)))
    return done / t_used, done, t_used, cores


def allreduce_max(vals, dev):
    """MAX over ranks of a list of floats (device tensor on NCCL, host tensor on gloo)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(vals)
    on_dev = dist.get_backend() == "nccl"
    t = torch.tensor(list(vals), dtype=torch.float64, device=dev if on_dev else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2511_11505_b200 import build as fbuild
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # FSC_BENCH_ONE_GPU=1: every rank on cuda:0 over gloo - exercises the N>1 code
    # path (EP transport, timing reductions) on a single-GPU box; timings meaningless.
    one_gpu = os.environ.get("FSC_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if rank == 0:
        fbuild.build()
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist.barrier()
        fbuild.build()
    else:
        torch.cuda.set_device(0)
    from paper_2511_11505_b200 import Context
    from tests.gpu_util import moe_weights_dev

    shape = get_shape(args.config)
    T = shape.tokens
    # EP = N when the experts shard evenly (C-amb-9), else independent EP=1 replicas
    ep = world if (world > 1 and shape.n_experts % world == 0) else 1
    e_loc = shape.n_experts // ep
    erank = rank if ep > 1 else 0
    dev = torch.device("cuda", local)
    w = synth.moe_weights(shape, seed=args.seed, e0=erank * e_loc, e_loc=e_loc)
    wd = moe_weights_dev(w, dev)
    del w
    allreduce = args.ep_mode == "allreduce" and ep > 1
    # all-reduce variant: every rank holds the same (replicated) tokens
    x = torch.from_numpy(synth.tokens(shape, seed=args.seed, rank=0 if allreduce else rank)).to(dev)
    out = torch.empty_like(x)
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=T, rank=erank, ep_size=ep, device=local)
    if args.cta_group:
        ctx.set_gemm_cta_group(args.cta_group)
    from paper_2511_11505_b200 import (FSC_BLOCKING_REGULAR_PLUS, FSC_BLOCKING_SERIAL, FSC_COMBINE_FUSED,
                                       FSC_COMBINE_STREAM)
    ctx.set_combine_mode(FSC_COMBINE_FUSED if args.combine == "fused" else FSC_COMBINE_STREAM)
    ctx.set_blocking_mode(FSC_BLOCKING_SERIAL if args.blocking == "serial" else FSC_BLOCKING_REGULAR_PLUS)
    if args.comm_ctas:
        ctx.set_comm_ctas(args.comm_ctas)
    if ep > 1:
        if args.dispatch_fp8 and not allreduce:
            ctx.set_dispatch_fp8(True)
        if allreduce:
            from paper_2511_11505_b200 import FSC_EP_ALLREDUCE
            ctx.set_ep_mode(FSC_EP_ALLREDUCE)
        ctx.connect()
    tok_world = 1 if allreduce else world      # replicated tokens count once
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def eager_step():
        ctx.moe_forward_blocking(wd, x, out, stream=torch.cuda.current_stream(dev).cuda_stream)

    for _ in range(args.warmup):
        eager_step()
    torch.cuda.synchronize(dev)
    # eager reference timing (one host call per step)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(3):
        eager_step()
    e1.record(stream)
    torch.cuda.synchronize(dev)
    eager_ms = e0.elapsed_time(e1) / 3
    # the whole MoE layer is free of host synchronisation (device-side counts, tile
    # lists and flags), so one step is captured once and replayed as a CUDA graph
    use_graph = not args.no_graph
    launches_per_step = None
    n_graphs = min(args.steps, 64)
    if use_graph:
        # one graph per timed step (cycled when K > 64), captured with the library's
        # phase timing on: each graph carries its own event-record nodes, so every
        # replay inside the timed region times its own kernels (roofline below)
        graphs = []
        ctx.set_timing_mask([] if args.no_live_timing else ["gemm1"])   # only the dominant kernel is bracketed
        lc0 = ctx.launch_count()
        for _ in range(n_graphs):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                eager_step()
            graphs.append(g)
        launches_per_step = (ctx.launch_count() - lc0) // n_graphs
        for g in graphs:
            g.replay()
        torch.cuda.synchronize(dev)

    def step(i=0):
        if use_graph:
            graphs[i % n_graphs].replay()
        else:
            eager_step()

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize(dev)

    # ---------------- timed region: K steps, per-step CUDA events on the launching stream
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = ctx.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk:
        wall0 = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            step(i)
            ev[i][1].record(stream)
        torch.cuda.synchronize(dev)
        wall = time.perf_counter() - wall0
    if world > 1:
        dist.barrier()
    launches = ctx.launch_count() - launches0
    if use_graph:
        launches = launches_per_step * args.steps
    ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = float(sum(ms))
    total_ms = allreduce_max([total_ms], dev)[0]
    ms_per_step = total_ms / args.steps
    value = T * tok_world * args.steps / (total_ms / 1e3)

    # ---------------- per-phase (per-kernel) times
    phase = {}
    timed_log = ctx.timing_log(4096) if use_graph else []
    ctx.set_timing(False)
    # breakdown of every phase: an instrumented graph (or eager step) replayed after the region
    ctx.set_timing(True)
    if use_graph:
        g_all = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_all):
            eager_step()
        for _ in range(max(3, min(args.steps, 10))):
            flush.fill_(0.0)
            g_all.replay()
            torch.cuda.synchronize(dev)
            for kname, v in ctx.timings().items():
                phase.setdefault(kname, []).append(v)
        del g_all
    else:
        for _ in range(max(3, min(args.steps, 10))):
            flush.fill_(0.0)
            eager_step()
            for kname, v in ctx.timings().items():
                phase.setdefault(kname, []).append(v)
    ctx.set_timing(False)
    phase_src = "CUDA events, instrumented replays of the same step after the timed region"
    gemm1_live = [v for kname, v in timed_log if kname == "gemm1"]
    phase_ms = {kname: statistics.median(v) for kname, v in phase.items()}

    # ---------------- e2e: host buffers through the C ABI, copies inside the region.
    # fsc_moe_forward_host_async pipelines step i's upload / compute / download with
    # its neighbours (two pinned buffer pairs alternate, as in a serving loop).
    # four pinned buffer pairs in rotation: call i's host buffers are free again once call
    # i + 3 has returned (fsc.h contract of the three staging slots)
    xh = [torch.from_numpy(synth.tokens(shape, seed=args.seed, rank=rank)).pin_memory() for _ in range(4)]
    oh = [torch.empty_like(xh[0]).pin_memory() for _ in range(4)]
    for i in range(4):
        ctx.moe_forward_host_async(wd, xh[i % 4], oh[i % 4], stream=stream.cuda_stream)
    ctx.host_flush()
    if world > 1:
        dist.barrier()
    e2e_steps = max(4, args.steps)
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        ctx.moe_forward_host_async(wd, xh[i % 4], oh[i % 4], stream=stream.cuda_stream)
    ctx.host_flush()
    e2e_s = time.perf_counter() - t0
    e2e_s = allreduce_max([e2e_s], dev)[0]
    e2e_value = T * tok_world * e2e_steps / e2e_s
    # synchronous variant (one call = H2D + forward + D2H + stream sync), for reference
    t0 = time.perf_counter()
    for i in range(3):
        ctx.moe_forward_blocking_host(wd, xh[0], oh[0], stream=stream.cuda_stream)
    e2e_sync_value = T * 3 / (time.perf_counter() - t0)

    backward = None
    if args.backward and not allreduce:
        backward = backward_measure(ctx, shape, wd, x, max(3, min(args.steps, 10)), world, dev, e_loc, args.seed,
                                    rank)

    stack = None
    if args.stack_layers > 0 and shape.tokens % shape.seq_len == 0 and not allreduce:
        stack = stack_measure(ctx, shape, wd, x, args.stack_layers, max(3, min(args.steps, 8)), world, dev,
                              rank, args.seed)

    if rank != 0:
        ctx.close()
        if world > 1:
            dist.destroy_process_group()
        return

    peaks, src = load_peaks()
    clocks = clk.summary()
    # Denominator: the measured BURST bf16 peak (the conservative choice: the step is
    # short and the clocks stay near max); the sustained-peak fraction is reported beside it.
    throttled = bool(set(clocks.get("reasons") or []) & {"sw_power_cap", "hw_slowdown", "hw_thermal_slowdown",
                                                           "sw_thermal_slowdown", "hw_power_brake"})
    peak_key = "bf16_tflops"
    peak = peaks["bf16_tflops"]
    # dominant kernel: routed-expert GEMM1 with the fused SwiGLU epilogue (row a7)
    R = T * shape.top_k                                        # balanced routing: rows received per rank = T*k
    if allreduce:
        R = T * shape.top_k // ep                              # replicated tokens: local experts' rows only
    g1_flop = 2.0 * R * shape.d * 2 * shape.ffn
    g1_bytes = 2.0 * e_loc * 2 * shape.ffn * shape.d + 2.0 * R * shape.d + 2.0 * R * shape.ffn  # W1|W2, xs, h
    if gemm1_live:    # event-record nodes around GEMM1 in every replayed graph of the timed region
        g1_ms = statistics.mean(gemm1_live)
        g1_src = f"CUDA events around the kernel in each of the {len(gemm1_live)} graph replays of the timed region"
    else:
        g1_ms = statistics.median(phase["gemm1"]) if phase.get("gemm1") else None
        g1_src = phase_src
    t_tensor = g1_flop / (peak * 1e12)
    t_hbm = g1_bytes / (peaks["hbm_gbs"] * 1e9)
    bound = "tensor" if t_tensor >= t_hbm else "hbm"       # decode batches stream the expert weights
    if bound == "tensor":
        achieved = g1_flop / (g1_ms * 1e-3) / 1e12 if g1_ms else None
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "peak_source": f"{src} {peak_key} (burst; clocks in the timed region: "
                               f"{clocks.get('sm_mhz')} MHz median" + (", throttle reasons seen)" if throttled else ")"),
                "algorithmic_flop_per_launch": g1_flop}
    else:
        achieved = g1_bytes / (g1_ms * 1e-3) / 1e9 if g1_ms else None
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "peak_source": f"{src} hbm_gbs", "algorithmic_bytes_per_launch": g1_bytes}
    roof["frac"] = (achieved / roof["peak"]) if achieved else None
    roof["kernel"] = "grouped_gemm_kernel<256,SWIGLU,2> (routed GEMM1, row a7)"
    roof["launch_ms"] = g1_ms
    roof["timing"] = g1_src
    traffic = None
    prof = os.path.join(ROOT, "profiles", f"ncu_gemm1_{shape.name}.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    roof["traffic"] = traffic
    if bound == "tensor" and achieved:
        roof["frac_of_sustained_peak"] = achieved / peaks.get("bf16_tflops_sustained", peak)
        roof["frac_of_spec_peak"] = achieved / BF16_SPEC_TFLOPS   # NVIDIA's dense bf16 figure
    exp_flop = 2.0 * R * shape.d * 3 * shape.ffn + 2.0 * T * shape.d * 3 * shape.shared_ffn
    a2a_bytes = 2.0 * 2 * R * shape.d * (ep - 1) / ep          # dispatch + combine bytes leaving a rank
    if args.dispatch_fp8 and not allreduce:                    # dispatch: 1 B / element + scales
        a2a_bytes = (R * shape.d * (1 + 4 / 128) + 2.0 * R * shape.d) * (ep - 1) / ep
    if allreduce:
        a2a_bytes = 2.0 * (ep - 1) / ep * T * shape.d * 4     # fp32 reduce-scatter + all-gather per rank
    w_bytes = 2.0 * 3 * shape.d * (e_loc * shape.ffn + shape.shared_ffn)
    layer_roof_ms = max(exp_flop / (peaks["bf16_tflops"] * 1e12), a2a_bytes / (NVLINK_GBS * 1e9),
                        w_bytes / (peaks["hbm_gbs"] * 1e9)) * 1e3
    res = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if allreduce else "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": dict(workload_config(shape, ep, world, "blocking (serial, Eq. 6)" if args.blocking == "serial" else
                                       "blocking (Regular+: shared expert beside the in-flight combine, P:103)"),
                       combine=("fused into the down GEMM epilogue" if args.combine == "fused" else
                                "comm-stream push after the down GEMM") if ep > 1 else None,
                       **({"ep_mode": "allreduce (replicated tokens, P:215-217)", "global_tokens": T}
                          if allreduce else {"ep_mode": "all-to-all (dispatch / combine)",
                                             "dispatch_payload": "fp8 e4m3 + per-128-col scales"
                                             if (args.dispatch_fp8 and ep > 1) else "bf16"})),
        "roofline": roof,
        "layer_roofline": {"expert_flop": exp_flop, "t_roof_ms": layer_roof_ms,
                           "a2a_bytes": a2a_bytes, "frac": layer_roof_ms / ms_per_step,
                           "weight_bytes": w_bytes,
                           "note": "max(expert FLOPs / bf16 burst peak, a2a bytes leaving the rank / 900 GB/s "
                                   "NVLink 5 per direction (spec), expert weight bytes / HBM); a2a = 0 at EP=1"},
        "phase_ms": phase_ms, "phase_timing": phase_src,
        "exposed_a2a_us_per_layer": (stack or {}).get("exposed_a2a_us_per_layer",
                                                       {"farskip": None, "blocking": None}),
        "stack": stack,
        "backward": backward,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": T * shape.d * 4 * world,
                "d2h_bytes_per_step": T * shape.d * 4 * world,
                "note": "fsc_moe_forward_host_async: every step uploads its pinned fp32 x and downloads its fp32 "
                        "output; consecutive steps pipelined, host-timed until the last download landed",
                "value_synchronous": e2e_sync_value},
        "gpu_launches": launches,
        "cuda_graph": use_graph, "ms_per_step_eager": eager_ms,
        "clocks": clocks,
        "wall_s_timed_region": wall,
    }
    if not args.no_cpu_baseline:
        tps, n, secs, cores = oracle_tokens_per_s(shape, budget_s=args.cpu_budget)
        res["cpu_baseline"] = {"value": tps, "unit": UNIT, "cores": cores, "kind": "oracle",
                               "sample": f"{n} of the {T} tokens of rank 0's batch through the fp64 numpy oracle "
                                         f"MoE block ({secs:.1f} s)"}
    print(json.dumps(res), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- backward (NEXT-2)
def backward_measure(ctx, shape, wd, x, steps, world, dev, e_loc, seed, rank):
    """fsc_moe_backward of the same layer (recompute + gradient all-to-all + dgrad / wgrad
    GEMMs + router / RMSNorm backward), timed with CUDA events over `steps` calls after a
    warm-up; FLOPs of its GEMMs: routed 16 R d c (dh, recomputed u|v, dX, dW3, dW1|dW2) +
    shared 16 T d c_s. Per-phase times from the library's timeline."""
    import torch
    T, d, c, cs = shape.tokens, shape.d, shape.ffn, shape.shared_ffn
    g = torch.from_numpy(np.random.default_rng([seed, rank, 77]).standard_normal((T, d)).astype(np.float32)).to(dev)
    z = lambda *sh: torch.empty(sh, dtype=torch.float32, device=dev)  # noqa: E731
    grads = {"dx": z(T, d), "dgamma": z(d), "dw_router": z(shape.n_experts, d), "dw1": z(e_loc, c, d),
             "dw2": z(e_loc, c, d), "dw3": z(e_loc, d, c)}
    if cs:
        grads.update({"dws1": z(cs, d), "dws2": z(cs, d), "dws3": z(d, cs)})
    stream = torch.cuda.current_stream(dev)
    for _ in range(2):
        ctx.moe_backward(wd, x, g, grads, stream=stream.cuda_stream)
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(steps):
        ctx.moe_backward(wd, x, g, grads, stream=stream.cuda_stream)
    b.record(stream)
    torch.cuda.synchronize(dev)
    ms = allreduce_max([a.elapsed_time(b) / steps], dev)[0]
    ctx.set_timing(True)
    ctx.moe_backward(wd, x, g, grads, stream=stream.cuda_stream)
    tl = ctx.timeline()
    ctx.set_timing(False)
    names = {"router": "recompute_router_maps", "dispatch": "dispatch_xn_and_grad (comm)",
             "shared1": "shared_backward", "gemm1": "routed_dh_and_swiglu_bwd", "gemm2": "routed_dX",
             "combine": "grad_combine (comm)", "shared2": "routed_wgrads", "unpermute": "token_router_rmsnorm_bwd",
             "dispatch_stall": "dispatch_stall", "combine_wait": "combine_wait"}
    R = T * shape.top_k
    flop = 16.0 * R * d * c + 16.0 * T * d * cs
    return {"ms": ms, "tokens_per_s": T * world / (ms * 1e-3), "gemm_flop": flop,
            "gemm_tflops_over_step": flop / (ms * 1e-3) / 1e12,
            "phase_ms": {names.get(p, p): du for p, _, _, du in tl},
            "note": "fsc_moe_backward: activation recomputation of the routing and expert inputs, dgrad + wgrad "
                    "tcgen05 GEMMs, gradient all-to-all on the comm stream (overlapped with the shared-expert "
                    "backward and the routed wgrads)"}


# ----------------------------------------------------------------------------- stack (FarSkip vs blocking)
BF16_SPEC_TFLOPS = 2250.0    # B200 dense bf16 (spec; the measured burst peak is the roofline denominator)
NVLINK_GBS = 900.0          # NVLink 5 per direction per GPU (spec; not measurable on the one-GPU dev box)
COMPUTE_PHASES = {"router", "perm_maps", "gemm1", "gemm2", "shared1", "shared2", "unpermute", "attn_a", "attn_b"}
COMM_PHASES = {"dispatch", "combine", "dispatch_stall", "combine_wait"}


def _union(iv):
    out = []
    for a, b in sorted(iv):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def exposed_from_timeline(tl):
    """Exposed communication (C-amb-14) from fsc_timeline's [(phase, stream, t0_ms, dur_ms)]:
    the measure of the union of communication intervals (dispatch and combine kernels on
    any stream, plus the compute stream's waits for peers: dispatch stall, combine wait)
    not covered by the union of compute-phase intervals on this GPU. Returns
    (exposed_ms, communication_union_ms)."""
    comp = _union([(t0, t0 + du) for ph, _, t0, du in tl if ph in COMPUTE_PHASES])
    comm = _union([(t0, t0 + du) for ph, _, t0, du in tl if ph in COMM_PHASES and du > 0])
    comm_ms = sum(b - a for a, b in comm)
    cov = sum(max(0.0, min(b, e) - max(a, s)) for a, b in comm for s, e in comp)
    return comm_ms - cov, comm_ms


def attention_flop(shape, T):
    """FLOPs of the attention filler per layer (causal GQA, packed sequences): part (a)
    = QKV projection, part (b) = core (QK^T and PV over the causal half) + o-projection."""
    hq, hkv, hd, d, sl = shape.n_heads, shape.n_kv_heads, shape.head_dim, shape.d, shape.seq_len
    a = 2.0 * T * d * (hq + 2 * hkv) * hd
    b = 2.0 * 2.0 * T * (sl + 1) / 2.0 * hq * hd + 2.0 * T * hq * hd * d
    return a, b


def stack_measure(ctx, shape, wd, x, L, steps, world, dev, rank, seed):
    """L-layer stack with the attention filler in four schedules (same kernels, same
    numbers): FarSkip = Hybrid wiring + OVERLAPPED; Regular = Eq. 6 wiring run
    BLOCKING (serialised; the headline baseline, C-amb-16); Regular+ = Eq. 6
    wiring, OVERLAPPED (the shared expert beside the in-flight combine); and each again
    with the zero-byte all-to-all (fsc_set_a2a_zero_bytes) for the cross-check
    exposed ~= t_layer - t_layer(zero-byte). Per-phase intervals come from the library's
    CUDA-event timeline (fsc_timeline); exposed = communication not covered by compute.
    The MoE weights of layer 0 are reused for every layer (timing only)."""
    import torch
    import torch.distributed as dist

    from paper_2511_11505_b200 import FSC_BLOCKING, FSC_HYBRID, FSC_OVERLAPPED, FSC_REGULAR
    from tests.gpu_util import attn_weights_dev
    aw = attn_weights_dev(synth.attn_weights(shape, seed=seed), dev)
    o0 = x
    oL = torch.empty_like(x)
    stream = torch.cuda.current_stream(dev)
    T = shape.tokens
    schedules = (("farskip", [FSC_HYBRID] * L, FSC_OVERLAPPED), ("regular", [FSC_REGULAR] * L, FSC_BLOCKING),
                 ("regular_plus", [FSC_REGULAR] * L, FSC_OVERLAPPED))
    res = {}
    for zb in (False, True):
        if world > 1:
            ctx.set_a2a_zero_bytes(zb)
        elif zb:
            break
        for name, modes, sched in schedules:
            def run():
                ctx.layer_stack_forward([aw] * L, [wd] * L, T, shape.seq_len, modes, sched, o0, oL,
                                        stream=stream.cuda_stream)
            for _ in range(2):
                run()
            torch.cuda.synchronize(dev)
            if world > 1:
                dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(steps):
                run()
            b.record(stream)
            torch.cuda.synchronize(dev)
            t = a.elapsed_time(b) / steps
            key = name + ("_zero_bytes" if zb else "")
            if zb:
                res[key] = {"ms_per_layer": allreduce_max([t], dev)[0] / L}
                continue
            ctx.set_timing(True)
            exp, comm, ph = 0.0, 0.0, {}
            for _ in range(steps):
                run()
                tl = ctx.timeline()
                e, c = exposed_from_timeline(tl)
                exp += e
                comm += c
                for p, _, _, du in tl:
                    ph[p] = ph.get(p, 0.0) + du
            ctx.set_timing(False)
            n = steps * L
            vals = allreduce_max([t, exp / n, comm / n], dev)
            res[key] = {"ms_per_stack": vals[0], "ms_per_layer": vals[0] / L,
                        "exposed_comm_us_per_layer": vals[1] * 1e3, "comm_us_per_layer": vals[2] * 1e3,
                        "phase_ms_per_layer": {k: v / n for k, v in sorted(ph.items())}}
    if world > 1:
        ctx.set_a2a_zero_bytes(False)
    fa, fb = attention_flop(shape, T)
    fs = res["farskip"]["phase_ms_per_layer"]
    attn = {"flop_part_a": fa, "flop_part_b": fb,
            "tflops_part_a": fa / (fs["attn_a"] * 1e-3) / 1e12 if fs.get("attn_a") else None,
            "tflops_part_b": fb / (fs["attn_b"] * 1e-3) / 1e12 if fs.get("attn_b") else None,
            "note": "attention filler (QKV / core+o-proj) TFLOP/s inside the FarSkip stack; the core is the tcgen05 "
                    "flash-attention kernel (hd = 128), the filler, not the graded hot path"}
    # Eq. 9: overlappable compute (attention + shared expert) minus the
    # communication it must hide, per layer, from the serialised (Regular) run's phase times
    rp = res["regular"]["phase_ms_per_layer"]
    overlappable = sum(rp.get(k, 0.0) for k in ("attn_a", "attn_b", "shared1", "shared2"))
    comm = sum(rp.get(k, 0.0) for k in ("dispatch", "combine"))
    eq9 = {"overlappable_us": overlappable * 1e3, "comm_us": comm * 1e3, "slack_us": (overlappable - comm) * 1e3}
    # the same slack with the attention at its tensor-core roofline (FLOPs / measured bf16
    # peak): what a fused attention would leave to hide the all-to-all behind (P:325
    # "fused attention makes comm more critical"), so the overlap is not judged against the
    # measured filler alone
    peaks, _ = load_peaks()
    attn_roof_ms = (fa + fb) / (peaks["bf16_tflops"] * 1e12) * 1e3
    ovl_roof = attn_roof_ms + sum(rp.get(k, 0.0) for k in ("shared1", "shared2"))
    eq9["attention_roofline_us"] = attn_roof_ms * 1e3
    eq9["slack_us_at_roofline_attention"] = (ovl_roof - comm) * 1e3
    out = {"layers": L, "attention": f"GQA {shape.n_heads}/{shape.n_kv_heads}x{shape.head_dim}, seq {shape.seq_len}",
           **res, "attention_throughput": attn, "eq9": eq9,
           "speedup_farskip_vs_regular": res["regular"]["ms_per_stack"] / res["farskip"]["ms_per_stack"],
           "speedup_farskip_vs_regular_plus": res["regular_plus"]["ms_per_stack"] / res["farskip"]["ms_per_stack"]}
    if world > 1:
        fs_e, blk_e = res["farskip"]["exposed_comm_us_per_layer"], res["regular"]["exposed_comm_us_per_layer"]
        zb = {n: (res[n]["ms_per_layer"] - res[n + "_zero_bytes"]["ms_per_layer"]) * 1e3 for n, _, _ in schedules}
        out["exposed_a2a_us_per_layer"] = {
            "farskip": fs_e, "blocking": blk_e, "regular_plus": res["regular_plus"]["exposed_comm_us_per_layer"],
            "blocking_comm_us": res["regular"]["comm_us_per_layer"],
            "farskip_frac_of_blocking": fs_e / res["regular"]["comm_us_per_layer"]
            if res["regular"]["comm_us_per_layer"] > 0 else None,
            "zero_byte_crosscheck_us": zb,
            "method": "fsc_timeline CUDA-event intervals: dispatch/combine time not covered by any compute phase; "
                      "cross-check = t_layer - t_layer(zero-byte all-to-all)"}
    else:
        out["exposed_a2a_us_per_layer"] = {"farskip": None, "blocking": None, "farskip_frac_of_blocking": None,
                                           "note": "EP=1: no all-to-all on one GPU"}
    return out


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    shape = get_shape(args.config)
    from threadpoolctl import threadpool_info, threadpool_limits

    from oracle import moe as om
    # torchrun sets OMP_NUM_THREADS=1 for every rank; rank 0 alone runs the oracle,
    # so give its BLAS all of the host cores
    threadpool_limits(limits=os.cpu_count() or 1)
    w = synth.moe_weights(shape, seed=args.seed)
    lay = om.layer_from_synth(w, shape.top_k)
    del w
    x = synth.tokens(shape, seed=args.seed, T=shape.tokens)
    cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    per_step = min(args.ref_tokens, shape.tokens)
    for i in range(args.warmup):
        om.moe_block(x[:min(per_step, 16)], lay)
    times = []
    for i in range(args.steps):
        s0 = (i * per_step) % max(1, shape.tokens - per_step)
        t0 = time.perf_counter()
        sh, ro, _ = om.moe_block(x[s0:s0 + per_step], lay)
        _ = (x[s0:s0 + per_step].astype(np.float64) + sh) + ro
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = per_step * args.steps / total
    res = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(shape, 1, world, "blocking"),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": f"{per_step} tokens per step of the {shape.tokens}-token batch"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(res), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="dsv2lite",
                    help=f"one of {sorted(synth.CONFIGS)} or <qwen3|scout>_decode<T> (configs[4])")
    ap.add_argument("--impl", default="fsc", choices=["fsc", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--ref-tokens", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every step eagerly instead of a CUDA graph")
    ap.add_argument("--ep-mode", default="a2a", choices=["a2a", "allreduce"],
                    help="N > 1: all-to-all dispatch/combine (training path) or the all-reduce inference variant")
    ap.add_argument("--dispatch-fp8", action="store_true", help="N > 1 all-to-all: FP8 e4m3 dispatch payload")
    ap.add_argument("--cta-group", type=int, default=0, choices=[0, 1, 2], help="GEMM tcgen05 cta_group (0 = auto)")
    ap.add_argument("--combine", default="stream", choices=["stream", "fused"],
                    help="N > 1: combine pushed on the comm stream after the down GEMM, or fused into its epilogue")
    ap.add_argument("--blocking", default="regular+", choices=["regular+", "serial"],
                    help="N > 1 headline layer: shared expert beside the in-flight combine, or fully serialised")
    ap.add_argument("--comm-ctas", type=int, default=0, help="CTAs of the dispatch / combine kernels (0 = library default)")
    ap.add_argument("--no-live-timing", action="store_true", help="no CUDA events inside the timed graphs")
    ap.add_argument("--stack-layers", type=int, default=4, help="0 disables the FarSkip-vs-blocking stack timing")
    ap.add_argument("--no-backward", dest="backward", action="store_false", help="skip the backward timing")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
