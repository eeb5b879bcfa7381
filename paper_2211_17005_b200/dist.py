"""Multi-GPU layout of the pathwise CVA engine.

Y-paths shard with no data exchange: every path and its X-children depend
only on their stream keys (market.cpp:178, defaults.cpp:29,35).  The shard is
interleaved so that every regression batch -- a contiguous range of P_B =
M / |B| paths (regressor.cpp:160-170) -- is split evenly: rank g of G owns
paths ``b * P_B + g * P_B / G + j`` (0 <= j < P_B / G, every batch b), so its
local batch b is exactly its part of global batch b.

The trainer (hcva_backward_learn_dist) reduces every cross-rank sum -- SGD
gradient and loss, epoch loss, head-switch minimum, refit Gram, scaler
moments, label mean -- by an allgather of FP64 per-rank partials followed by
a sum in rank order on the device: every rank applies bit-identical updates
(no parameter broadcast), the result is deterministic for a given G, and it
matches the single-GPU run up to the FP64 re-association of the per-rank
partial sums.  ``rank_order_sum`` is the host mirror of that reduction.
"""
from typing import Dict, Tuple

import numpy as np


def batch_paths(n_paths: int, n_batches: int) -> int:
    """P_B, the paths of one regression batch (make_batches on whole paths)."""
    if n_batches < 1 or n_paths % n_batches:
        raise ValueError(f"make_batches: {n_batches} batches must divide {n_paths} paths")
    return n_paths // n_batches


def shard_spec(n_paths: int, n_batches: int, world: int, rank: int) -> Dict[str, object]:
    """Local simulate_set arguments of `rank` in a `world`-GPU run over `n_paths` global paths."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world {world}")
    pb = batch_paths(n_paths, n_batches)
    if world == 1:
        return {"n_paths": n_paths, "path_offset": 0, "shard": None, "batch_paths": pb}
    if pb % world:
        raise ValueError(f"a batch of {pb} paths does not split over {world} ranks")
    blk = pb // world
    return {"n_paths": n_paths // world, "path_offset": rank * blk, "shard": (blk, pb), "batch_paths": pb}


def shard_paths(spec: Dict[str, object]) -> np.ndarray:
    """Global path index of every local path of a shard (simulate.cu shard_path)."""
    k = np.arange(spec["n_paths"], dtype=np.int64)
    if spec["shard"] is None:
        return spec["path_offset"] + k
    blk, stride = spec["shard"]
    return spec["path_offset"] + (k // blk) * stride + k % blk


# ---------------------------------------------------------------- transports

ID_BYTES = 128  # NCCL unique id


class Comm:
    """A rank of a multi-GPU regression run (hcva_comm): NCCL or an in-process group."""

    def __init__(self, handle, keep=None):
        self.handle = handle
        self._keep = keep  # objects that must outlive the handle (the local group)

    @property
    def rank_world(self) -> Tuple[int, int]:
        import ctypes as C

        from . import _lib

        r, w = C.c_int(), C.c_int()
        _lib.check(_lib.lib().hcva_comm_info(self.handle, C.byref(r), C.byref(w)))
        return r.value, w.value

    def close(self):
        if self.handle:
            from . import _lib

            _lib.lib().hcva_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """A fresh NCCL unique id (call on rank 0, then broadcast with ``share_id``)."""
    import ctypes as C

    from . import _lib

    buf = C.create_string_buffer(ID_BYTES)
    _lib.check(_lib.lib().hcva_comm_nccl_id(buf))
    return buf.raw


def share_id(make_id, group=None) -> bytes:
    """Rank 0 makes the id, every rank of the torch.distributed group receives it."""
    import torch
    import torch.distributed as dist

    t = torch.zeros(ID_BYTES, dtype=torch.uint8)
    if dist.get_rank(group) == 0:
        t.copy_(torch.frombuffer(bytearray(make_id()), dtype=torch.uint8))
    backend = dist.get_backend(group)
    if backend == "nccl":  # NCCL collectives need device tensors
        t = t.cuda()
    dist.broadcast(t, src=0, group=group)
    return bytes(t.cpu().numpy().tobytes())


def nccl_comm(ctx, world: int, rank: int, uid: bytes) -> Comm:
    """NCCL transport on ctx's stream (one process per GPU)."""
    import ctypes as C

    from . import _lib

    h = C.c_void_p()
    _lib.check(_lib.lib().hcva_comm_create_nccl(ctx.handle, world, rank, uid, C.byref(h)))
    return Comm(h)


class LocalGroup:
    """In-process group: one host thread and context per rank (any devices)."""

    def __init__(self, world: int):
        import ctypes as C

        from . import _lib

        h = C.c_void_p()
        _lib.check(_lib.lib().hcva_group_create(world, C.byref(h)))
        self.handle, self.world = h, world

    def comm(self, ctx, rank: int) -> Comm:
        import ctypes as C

        from . import _lib

        h = C.c_void_p()
        _lib.check(_lib.lib().hcva_comm_create_local(ctx.handle, self.handle, rank, C.byref(h)))
        return Comm(h, keep=self)

    def __del__(self):
        try:
            if self.handle:
                from . import _lib

                _lib.lib().hcva_group_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def rank_order_sum(local, group=None):
    """Host mirror of the trainer's cross-rank reduction: allgather + sum in rank order.

    ``local`` is a float64 numpy vector; returns the identical total on every rank."""
    import torch
    import torch.distributed as dist

    t = torch.from_numpy(np.ascontiguousarray(local, dtype=np.float64))
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, t, group=group)
    total = np.zeros_like(np.asarray(local, dtype=np.float64))
    for p in parts:
        total = total + p.numpy()
    return total
