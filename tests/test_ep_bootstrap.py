"""CPU (gloo, world_size 2) test of the EP bootstrap plumbing: every rank's
transport blob reaches every rank in rank order."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2511_11505_b200._lib import exchange_blobs
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blob = bytes([rank]) * 64                 # stands in for a 64-byte cudaIpcMemHandle_t
    got = exchange_blobs(blob)
    q.put((rank, got))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_blob_exchange_rank_order(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r] == [bytes([s]) * 64 for s in range(world)]


def test_blob_size_matches_ipc_handle():
    from paper_2511_11505_b200 import build
    build.build()
    from paper_2511_11505_b200._lib import load
    assert load().fsc_bootstrap_size() == 64     # sizeof(cudaIpcMemHandle_t)
