"""CPU float64 oracle for the FarSkip-Collective MoE forward — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything in here. The
product path (``paper_2511_11505_b200``) never imports, links or executes it,
and this package never imports the product path; both receive their inputs
from ``synth`` (seeded generators, no method arithmetic).

Written from the paper (PAPER.md = /root/reference/PAPER.md, cited as P:<line>):
  * moe.py        — RMSNorm, router G(A)=s(A W_R^T) with top-k renormalised
                    softmax, SwiGLU experts, EP Dispatch/Combine simulation,
                    dense brute force.
  * attention.py  — the attention sub-block used as the stack's filler
                    (causal GQA + RoPE; MLA is out of scope, C-amb-18).
  * stack.py      — Regular (Eq. 6) and Hybrid FarSkip
                     residual wiring over L layers.
  * schedule.py   — FIFO two-stream replay of the 8-step forward schedule
                     for the stream-wiring pin.

Every function is fp64 and unblocked; library primitives (numpy matmul,
argsort, exp) serve as steps. Readings of the paper where it is silent are the
DESIGN.md "Readings" table (C-amb-n). Functions without an independent pin
are marked "parity unpinned" in their docstring and in DESIGN.md.
"""
