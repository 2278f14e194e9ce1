"""Row sharding of one verification across ranks (one process per GPU).

The engine (pc_net_set_sharding, include/polycert_b200.h) splits every
pass's live rows into contiguous per-rank slices — rows of a pass are
independent (proj/include/polycert/backsub.hpp:31-34) — and calls back into
the host for the path's one exchange step: an all-gather of the refined
candidate bounds (32 B per row) before the write-back and refresh. This module
supplies that callback over torch.distributed:

* NCCL process group: ``all_gather_into_tensor`` directly on the engine's
  device buffers, enqueued on the engine's CUDA stream (NVLink / NVSwitch).
* gloo process group (CPU tests, or several ranks sharing one GPU): the slice
  is staged through host memory.

Results are bit-identical to the unsharded engine (tests/test_gpu_sharding.py).
"""
from __future__ import annotations

import ctypes


class _DeviceBytes:
    """A raw device allocation exposed through __cuda_array_interface__."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


def allgather_bytes(send, recv, group=None):
    """Gather `send` (uint8, n bytes) from every rank into `recv` (world*n bytes,
    rank-major). Device tensors on an NCCL group gather in place; otherwise the
    bytes go through host memory (gloo)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n = send.numel()
    if send.is_cuda and dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(recv, send, group=group)
        return
    hs = send.cpu()
    parts = [torch.empty(n, dtype=torch.uint8) for _ in range(world)]
    dist.all_gather(parts, hs, group=group)
    recv.copy_(torch.cat(parts))


def make_allgather(group=None, device=None):
    """The pc_allgather_fn for this process group (a ctypes callback; keep a
    reference for as long as the net is sharded)."""
    import torch
    import torch.distributed as dist

    from . import _lib
    world = dist.get_world_size(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)

    def cb(_user, d_send, d_recv, nbytes, stream):
        try:
            send = torch.as_tensor(_DeviceBytes(d_send, nbytes), device=dev)
            recv = torch.as_tensor(_DeviceBytes(d_recv, nbytes * world), device=dev)
            es = torch.cuda.ExternalStream(stream, device=dev)
            if nccl:
                with torch.cuda.stream(es):
                    allgather_bytes(send, recv, group)
            else:
                es.synchronize()  # the engine's pack kernel has written d_send
                allgather_bytes(send, recv, group)
                torch.cuda.synchronize(dev)
            return 0
        except Exception as e:  # reported through the engine's error path
            import sys
            print(f"polycert sharding allgather failed: {e!r}", file=sys.stderr)
            return 1

    return _lib.ALLGATHER_FN(cb)


def _native_nccl(verifier, group, rank, world):
    """A native NCCL communicator for this net (pc_nccl_comm_create): the id
    from rank 0 travels over the process group, then every rank's exchange is
    one ncclAllGather on the engine stream (no Python on the data path)."""
    import torch.distributed as dist

    from . import _lib
    err = ctypes.create_string_buffer(512)
    uid = ctypes.create_string_buffer(128)
    if rank == 0 and _lib.lib.pc_nccl_unique_id(uid, err, 512) != 0:
        raise RuntimeError(err.value.decode())
    box = [uid.raw if rank == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0,
                               group=group)
    uid = ctypes.create_string_buffer(box[0], 128)
    import torch
    dev = verifier.options.device if verifier.options.device >= 0 else torch.cuda.current_device()
    comm = _lib.lib.pc_nccl_comm_create(int(dev), rank, world, uid, err, 512)
    if not comm:
        raise RuntimeError(err.value.decode())
    return comm


def enable(verifier, group=None, transport: str = "auto"):
    """Shard `verifier`'s passes across the ranks of `group`.

    transport: "native" — the engine's own NCCL communicator
    (pc_nccl_allgather, ncclAllGather on the engine stream); "callback" — the
    torch.distributed callback above (NCCL in place or gloo via host memory);
    "auto" — native on an NCCL group, else the callback."""
    import torch.distributed as dist

    from . import _lib
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    disable(verifier)
    nccl = dist.get_backend(group) == "nccl"
    if transport == "native" or (transport == "auto" and nccl and world > 1):
        comm = _native_nccl(verifier, group, rank, world)
        fn = _lib.ALLGATHER_FN(("pc_nccl_allgather", _lib.lib))
        _lib.check(_lib.lib.pc_net_set_sharding(verifier._h, rank, world, fn, comm))
        verifier._allgather, verifier._nccl_comm = fn, comm
        verifier.shard_transport = "native-nccl"
        return rank, world
    fn = make_allgather(group, verifier.options.device if verifier.options.device >= 0 else None)
    _lib.check(_lib.lib.pc_net_set_sharding(verifier._h, rank, world, fn, None))
    verifier._allgather = fn  # keep the callback alive
    verifier.shard_transport = "torch-callback-" + dist.get_backend(group)
    return rank, world


def disable(verifier):
    from . import _lib
    _lib.check(_lib.lib.pc_net_set_sharding(verifier._h, 0, 1, ctypes.cast(None, _lib.ALLGATHER_FN),
                                            None))
    verifier._allgather = None
    comm = getattr(verifier, "_nccl_comm", None)
    if comm:
        _lib.lib.pc_nccl_comm_destroy(comm)
        verifier._nccl_comm = None
