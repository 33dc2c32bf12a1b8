"""bench.py's N > 1 path (torchrun, one process per rank) exercised on one GPU
(FSC_BENCH_ONE_GPU=1: every rank on cuda:0 over gloo; timings meaningless): the EP
transport, the FarSkip / Regular / Regular+ stack timings with the CUDA-event timeline
and the zero-byte cross-check, the backward timing, and the max-over-ranks reductions
all run and produce one well-formed JSON line on rank 0."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("combine", ["stream", "fused"])
def test_bench_two_ranks_on_one_gpu(combine):
    env = dict(os.environ, FSC_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3",
           "--warmup", "3", "--config", "tiny", "--stack-layers", "2", "--no-cpu-baseline", "--combine", combine]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["config"]["ep"] == 2 and j["value"] > 0
    ex = j["exposed_a2a_us_per_layer"]
    for k in ("farskip", "blocking", "regular_plus", "blocking_comm_us"):
        assert ex[k] is not None and ex[k] >= 0, (k, ex)
    assert set(ex["zero_byte_crosscheck_us"]) == {"farskip", "regular", "regular_plus"}
    st = j["stack"]
    for name in ("farskip", "regular", "regular_plus", "farskip_zero_bytes"):
        assert st[name]["ms_per_layer"] > 0
    assert st["eq9"]["comm_us"] > 0
    assert j["backward"]["ms"] > 0
