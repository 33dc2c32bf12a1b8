"""Stream-wiring pin (SURVEY §8(c) O-4 "Stream wiring", row a12): the SPEC S:437 golden
durations (gate 1, dispatch 3, qkv 2, core 4, routed 5, combine 3, shared 4 units)
replayed through the REAL stack / MoE stream and event wiring of libfsc, with every
phase's kernels replaced by one spin kernel of its duration (fsc_set_spin_schedule).
The device timeline must reproduce the golden FIFO replay (tests/golden/schedule_l2.json,
P:103 and P:198 orders): FarSkip 32 units with 0 exposed communication, Regular 44 / 12,
Regular+ 38 / 6. Exposed = communication-phase time not covered by any compute phase
(C-amb-14), read from the library's own CUDA-event timeline (fsc_timeline)."""
import json
import os

import numpy as np
import pytest
import torch

import synth
from tests.gpu_util import attn_weights_dev, dev_f32, moe_weights_dev

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "schedule_l2.json")))
UNIT_MS = 1.0
TOL = 0.3            # units: launch gaps between ~30 back-to-back kernels and event records
COMPUTE = {"router", "gemm1", "shared1", "attn_a", "attn_b"}
COMM = {"dispatch", "combine"}
# spin-mode phase -> S:437 name
NAME = {"attn_a": "qkv", "router": "gate", "dispatch": "dispatch", "attn_b": "core", "gemm1": "routed",
        "combine": "combine", "shared1": "shared"}


def exposed(tl):
    """Communication time not covered by the union of compute intervals (any stream)."""
    comp = sorted((t0, t0 + du) for ph, _, t0, du in tl if ph in COMPUTE)
    total = 0.0
    for ph, _, t0, du in tl:
        if ph not in COMM:
            continue
        a, b, cov, cur = t0, t0 + du, 0.0, t0
        for s, e in comp:
            if e <= cur or s >= b:
                continue
            s2, e2 = max(s, cur), min(e, b)
            if e2 > s2:
                cov += e2 - s2
                cur = e2
        total += (b - a) - cov
    return total


def run(modes, schedule):
    from paper_2511_11505_b200 import SPIN_PHASES, Context, build
    build.build()
    shape = synth.CONFIGS["tiny"]
    T, L = shape.tokens, 2
    ctx = Context(d=shape.d, n_experts=shape.n_experts, top_k=shape.top_k, ffn=shape.ffn,
                  shared_ffn=shape.shared_ffn, max_tokens=T)
    mw = [moe_weights_dev(synth.moe_weights(shape, seed=0, layer=k)) for k in range(L)]
    aw = [attn_weights_dev(synth.attn_weights(shape, seed=0, layer=k)) for k in range(L)]
    ctx.set_spin_schedule({p: GOLD["durations"][p] * UNIT_MS * 1e6 for p in SPIN_PHASES})
    o0 = dev_f32(synth.tokens(shape, T=T))
    oL = torch.empty_like(o0)
    ctx.layer_stack_forward(aw, mw, T, shape.seq_len, modes, schedule, o0, oL)   # warm-up
    torch.cuda.synchronize()
    ctx.set_timing(True)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.layer_stack_forward(aw, mw, T, shape.seq_len, modes, schedule, o0, oL)
    b.record()
    torch.cuda.synchronize()
    tl = ctx.timeline()
    ctx.set_timing(False)
    ctx.set_spin_schedule(None)
    ctx.close()
    return a.elapsed_time(b) / UNIT_MS, [(ph, st, t0 / UNIT_MS, du / UNIT_MS) for ph, st, t0, du in tl]


def test_farskip_wiring_reproduces_golden_timeline():
    from paper_2511_11505_b200 import FSC_HYBRID, FSC_OVERLAPPED
    end, tl = run([FSC_HYBRID] * 2, FSC_OVERLAPPED)
    g = GOLD["results"]["farskip"]
    assert abs(end - g["end"]) < TOL, (end, tl)
    assert exposed(tl) < TOL, tl
    seen = {}
    for ph, st, t0, du in tl:
        if ph not in NAME:
            continue
        seen[ph] = seen.get(ph, 0) + 1
        key = f"{NAME[ph]}{seen[ph]}"
        s_g, e_g = GOLD["farskip_intervals"][key]
        assert abs(t0 - s_g) < TOL and abs(t0 + du - e_g) < TOL, (key, t0, t0 + du, s_g, e_g)
        assert st == ("comm" if ph in COMM else "compute"), (key, st)
    assert len([p for p in tl if p[0] in NAME]) == len(GOLD["farskip_intervals"])


@pytest.mark.parametrize("modes,sched,gold", [("R", "BLOCKING", "regular"), ("H", "BLOCKING", "regular"),
                                              ("R", "OVERLAPPED", "regular+")])
def test_blocking_wirings_reproduce_golden_totals(modes, sched, gold):
    """Regular layers in the BLOCKING schedule (and the Hybrid control run) serialise
    every collective (P:103 bubbles (b), (c)); Regular layers in the OVERLAPPED schedule
    run the shared expert beside the in-flight combine (Regular+)."""
    import paper_2511_11505_b200 as F
    m = {"R": F.FSC_REGULAR, "H": F.FSC_HYBRID}[modes]
    end, tl = run([m] * 2, getattr(F, f"FSC_{sched}"))
    g = GOLD["results"][gold]
    assert abs(end - g["end"]) < TOL, (end, g)
    assert abs(exposed(tl) - g["exposed"]) < TOL, (exposed(tl), g)
