"""Row sharding on the GPU (pc_net_set_sharding): world_size 2 and 3 ranks
share cuda:0 over a gloo group (one GPU is all a test box has; the NCCL path
differs only in the transport). Every rank's verdict, margins, padded and raw
bounds and stats must be bit-identical to the unsharded engine, and the
unsharded engine to the oracle (tests/test_gpu_parity.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from cases import BACKSUB_ARCHS, EXTRA_ARCHS

pytestmark = pytest.mark.gpu

ARCHS = [BACKSUB_ARCHS[0], BACKSUB_ARCHS[2], EXTRA_ARCHS[2], EXTRA_ARCHS[3], EXTRA_ARCHS[8]]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(arch, seed, eps, label, shard, rank=0, world=1, port=0, q=None, et=True):
    import paper_2007_10868_b200 as pc
    net = pc.generate(seed, arch)
    x = pc.random_inputs(seed + 1, 1, int(np.prod(net.input_shape)))[0]
    v = pc.Verifier(net, pc.AnalysisOptions(device=0, early_term=et))
    if shard:
        import torch.distributed as dist
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        v.enable_sharding()
    box = pc.input_box(x, eps)
    r = v.test(box.lo, box.hi, label, want_bounds=True)
    out = {"margins": r.margins.tolist(), "verified": r.verified, "stats": r.stats,
           "b": [np.concatenate([b[i] for b in r.bounds]).view(np.int64).tolist() for i in (0, 1)],
           "raw": [np.concatenate([b[i] for b in r.raw]).view(np.int64).tolist() for i in (0, 1)]}
    if shard:
        import torch.distributed as dist
        dist.destroy_process_group()
        q.put((rank, out))
    return out


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("arch", ARCHS)
def test_sharded_equals_unsharded(arch, world):
    seed, eps = 900, 0.25
    ref = _run(arch, seed, eps, 1, False)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_run, args=(arch, seed, eps, 1, True, r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    try:
        got = dict(q.get(timeout=300) for _ in range(world))
        for p in ps:
            p.join(60)
            assert p.exitcode == 0
    finally:  # never leave a rank behind holding the GPU
        for p in ps:
            if p.is_alive():
                p.kill()
                p.join(10)
    for r in range(world):
        g = got[r]
        assert g["b"] == ref["b"] and g["raw"] == ref["raw"], f"rank {r}: bounds differ"
        assert np.array_equal(np.array(g["margins"]).view(np.int64), np.array(ref["margins"]).view(np.int64))
        assert g["verified"] == ref["verified"]
        for k in ("rows_total", "rows_terminated_early", "gbc_madds", "dense_madds", "gbc_dense_equiv"):
            assert g["stats"][k] == ref["stats"][k], (r, k, g["stats"], ref["stats"])
