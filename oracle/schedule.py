"""FIFO two-queue replay of the MoE layer schedules — TEST INFRASTRUCTURE.

Models what a CUDA stream pair does with the forward schedules of the paper:
ops are enqueued in host order on a compute queue or a comm queue;
each queue runs its ops first-in first-out; an op starts when its queue is
free and every op it waits on has finished. Used to derive the golden
timelines (SPEC S:437 durations) that the GPU spin-kernel test replays.

Schedules (one MoE transformer layer):
  regular   : qkv, core, gate, dispatch*, routed, combine*, shared — serial (A13 blocking)
  regular+  : as regular but shared runs beside the combine ("(c) may be
              partially overlapped if a shared expert is present")
  farskip   : 1) qkv 2) wait combine_{k-1} 3) gate 4) start dispatch* 5) core
              6) wait dispatch, routed 7) start combine* 8) shared
(* = comm queue). Exposed comm = comm busy time not covered by any compute op.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Sequence, Tuple


@dataclasses.dataclass
class Op:
    name: str
    queue: str            # "compute" | "comm"
    dur: float
    waits: Tuple[str, ...] = ()


def simulate(ops: Sequence[Op]) -> Dict[str, Tuple[float, float]]:
    free = {"compute": 0.0, "comm": 0.0}
    t: Dict[str, Tuple[float, float]] = {}
    for op in ops:                      # host enqueue order
        start = max([free[op.queue]] + [t[w][1] for w in op.waits])
        t[op.name] = (start, start + op.dur)
        free[op.queue] = start + op.dur
    return t


def exposed_comm(ops: Sequence[Op], t: Dict[str, Tuple[float, float]]) -> float:
    comp = sorted(t[o.name] for o in ops if o.queue == "compute")
    total = 0.0
    for o in ops:
        if o.queue != "comm":
            continue
        a, b = t[o.name]
        # subtract the union of compute intervals from [a, b)
        covered = 0.0
        cur = a
        for (s, e) in comp:
            if e <= cur or s >= b:
                continue
            s2, e2 = max(s, cur), min(e, b)
            if e2 > s2:
                covered += e2 - s2
                cur = e2
        total += (b - a) - covered
    return total


DEFAULT_DUR = dict(gate=1, dispatch=3, qkv=2, core=4, routed=5, combine=3, shared=4)


def build(schedule: str, n_layers: int, dur: Dict[str, float] = DEFAULT_DUR) -> List[Op]:
    ops: List[Op] = []
    prev_tail: Tuple[str, ...] = ()
    for k in range(1, n_layers + 1):
        n = lambda s: f"{s}{k}"  # noqa: E731
        if schedule == "farskip":
            ops.append(Op(n("qkv"), "compute", dur["qkv"]))
            ops.append(Op(n("gate"), "compute", dur["gate"], prev_tail))
            ops.append(Op(n("dispatch"), "comm", dur["dispatch"], (n("gate"),)))
            ops.append(Op(n("core"), "compute", dur["core"]))
            ops.append(Op(n("routed"), "compute", dur["routed"], (n("dispatch"),)))
            ops.append(Op(n("combine"), "comm", dur["combine"], (n("routed"),)))
            ops.append(Op(n("shared"), "compute", dur["shared"]))
            prev_tail = (n("combine"),)
        elif schedule in ("regular", "regular+"):
            ops.append(Op(n("qkv"), "compute", dur["qkv"], prev_tail))
            ops.append(Op(n("core"), "compute", dur["core"]))
            ops.append(Op(n("gate"), "compute", dur["gate"]))
            ops.append(Op(n("dispatch"), "comm", dur["dispatch"], (n("gate"),)))
            ops.append(Op(n("routed"), "compute", dur["routed"], (n("dispatch"),)))
            ops.append(Op(n("combine"), "comm", dur["combine"], (n("routed"),)))
            if schedule == "regular":
                ops.append(Op(n("shared"), "compute", dur["shared"], (n("combine"),)))
                prev_tail = ()
            else:
                ops.append(Op(n("shared"), "compute", dur["shared"]))
                prev_tail = (n("combine"),)
        else:
            raise ValueError(schedule)
    return ops


def replay(schedule: str, n_layers: int = 2, dur: Dict[str, float] = DEFAULT_DUR):
    ops = build(schedule, n_layers, dur)
    t = simulate(ops)
    end = max(e for _, e in t.values())
    return end, exposed_comm(ops, t), t
