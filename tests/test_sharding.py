"""Host side of row sharding (paper_2007_10868_b200/sharding.py) on CPU with
a world_size-2 gloo group: the all-gather the engine calls back into must
deliver every rank's slice in rank order."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2007_10868_b200.sharding import allgather_bytes
    n = 40  # 5 rows x 8 B
    send = torch.arange(n, dtype=torch.uint8) + 100 * rank
    recv = torch.zeros(world * n, dtype=torch.uint8)
    allgather_bytes(send, recv)
    q.put((rank, recv.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allgather_layout_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    try:
        got = dict(q.get(timeout=120) for _ in range(world))
        for p in ps:
            p.join(60)
            assert p.exitcode == 0
    finally:
        for p in ps:
            if p.is_alive():
                p.kill()
                p.join(10)
    want = [(k % 40) + 100 * (k // 40) for k in range(world * 40)]
    for r in range(world):
        assert got[r] == want


def test_set_sharding_validation():
    from paper_2007_10868_b200 import _lib
    assert _lib.lib.pc_net_set_sharding(None, 0, 2, _lib.ALLGATHER_FN(lambda *a: 0), None) == \
        _lib.PC_ERR_INVALID_ARGUMENT
    assert b"sharding" in _lib.lib.pc_last_error()
