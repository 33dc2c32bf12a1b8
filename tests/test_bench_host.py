"""Host-side logic of bench.py (no GPU): the exposed-communication instrument applied
to the oracle's FIFO replay of the golden SPEC S:437 schedules must give the golden
exposed times (FarSkip 0, Regular 12, Regular+ 6 units), and the attention FLOP count
its closed form."""
import json
import os

import bench
from oracle import schedule as osch

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "schedule_l2.json")))
PHASE = {"qkv": "attn_a", "core": "attn_b", "gate": "router", "routed": "gemm1", "shared": "shared1",
         "dispatch": "dispatch", "combine": "combine"}


def _timeline(schedule):
    ops = osch.build(schedule, 2)
    t = osch.simulate(ops)
    return [(PHASE[o.name.rstrip("12")], o.queue, t[o.name][0], t[o.name][1] - t[o.name][0]) for o in ops]


def test_exposed_instrument_on_golden_replays():
    for sched in ("farskip", "regular", "regular+"):
        exp, comm = bench.exposed_from_timeline(_timeline(sched))
        assert exp == GOLD["results"][sched]["exposed"], (sched, exp)
        assert comm == 2 * (GOLD["durations"]["dispatch"] + GOLD["durations"]["combine"])


def test_exposed_counts_peer_waits_once():
    # a compute-stream wait for a late peer overlapping my own combine kernel: counted once
    tl = [("gemm1", "compute", 0.0, 5.0), ("combine", "comm", 5.0, 2.0), ("combine_wait", "compute", 5.0, 4.0),
          ("shared1", "compute", 9.0, 1.0)]
    assert bench.exposed_from_timeline(tl) == (4.0, 4.0)


def test_attention_flop_closed_form():
    import synth
    sh = synth.MoeShape("t", d=64, n_experts=4, top_k=1, ffn=64, shared_ffn=0, tokens=8, n_heads=2, n_kv_heads=1,
                        head_dim=16, seq_len=4)
    a, b = bench.attention_flop(sh, 8)
    assert a == 2 * 8 * 64 * (2 + 2) * 16
    # causal: query i attends to i+1 keys; QK^T and PV 2*hd flops each per (query, key, head)
    core = sum(2 * 2 * 16 * (i % 4 + 1) * 2 for i in range(8))
    assert b == core + 2 * 8 * 2 * 16 * 64
