"""Sharded expert-map store over the ranks of a torch.distributed group.

The sharding lives in the library (``fmoe_store_create_sharded``, include/fmoe.h):
rank r of G holds the global slots [r*P, min((r+1)*P, C)), P = ceil(C/G); every
call on the store is collective and runs the single-GPU kernels on the local
slots, then ONE all-gather of a packed per-rank payload and a merge kernel, so
outputs are replicated and bit-identical to the unsharded store.  This module
only marshals: it creates the communicator the library asks for.

Transports:
  * "nccl": rank 0 asks the library for an NCCL unique id, the group
    broadcasts it, every rank creates the store (ncclCommInitRank inside the
    library); the exchange is ncclAllGather on the call's stream.
  * "host": the library calls back into ``_HostAllGather`` with host buffers,
    which runs ``torch.distributed.all_gather_into_tensor`` on CPU tensors
    (gloo).  For ranks that share one GPU (NCCL refuses duplicate devices) and
    for CPU-only collective plumbing.
"""
from __future__ import annotations

import ctypes

import torch
import torch.distributed as dist

import paper_2502_05370_b200 as fm


def shard_range(n_total: int, rank: int, world: int):
    """(local capacity, id_offset) of `rank`: the library's contiguous slot ranges."""
    per = (n_total + world - 1) // world
    lo = min(rank * per, n_total)
    hi = min(lo + per, n_total)
    return hi - lo, lo


class _HostAllGather:
    """fmoe_allgather_fn over a torch.distributed group: recv[world][bytes] <- send[bytes]."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.cfn = fm.ALLGATHER_FN(self._call)     # keep a reference for the store's lifetime
        self.error = None

    def _call(self, send, recv, nbytes, _user):
        try:
            src = torch.frombuffer((ctypes.c_uint8 * nbytes).from_address(send), dtype=torch.uint8).clone()
            out = torch.empty(self.world * nbytes, dtype=torch.uint8)
            dist.all_gather_into_tensor(out, src, group=self.group)
            ctypes.memmove(recv, out.data_ptr(), self.world * nbytes)
            return 0
        except Exception as e:  # noqa: BLE001 -- reported to the library as a failed exchange
            self.error = e
            return 1


class ShardedExpertMapStore(fm.ExpertMapStore):
    """Collective API: every rank calls every method with the same arguments.

    Same methods as ExpertMapStore (search_*, select_experts, insert,
    trajectory_session ...); ``len()`` is the global size, ids are global."""

    def __init__(self, L, E, K, D, d, capacity_total, dtype="bf16", group=None, device=None, transport="nccl"):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.L, self.E, self.K, self.D, self.d = L, E, K, D, d
        self.capacity_total = capacity_total
        self.cap_local, self.offset = shard_range(capacity_total, self.rank, self.world)
        dev = device if device is not None else torch.cuda.current_device()
        self.capacity, self.dtype, self.id_offset = self.cap_local, dtype, self.offset
        self.device = torch.device("cuda", dev)
        self._ag = None
        uid = None
        if transport == "nccl":
            blob = [fm.fmoe_get_nccl_unique_id() if self.rank == 0 else None]
            dist.broadcast_object_list(blob, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            uid = blob[0]
        elif transport == "host":
            self._ag = _HostAllGather(group)
        else:
            raise ValueError(transport)
        self._h = fm.fmoe_store_create_sharded(L, E, K, D, d, capacity_total, dtype, dev, self.rank, self.world,
                                               transport, uid, self._ag)

    def read(self, slot_begin=None, count=None):
        """This rank's rows (global slots inside the local shard)."""
        slot_begin = self.offset if slot_begin is None else slot_begin
        n_local = max(0, min(len(self) - self.offset, self.cap_local))
        count = n_local - (slot_begin - self.offset) if count is None else count
        return super().read(slot_begin, count)

    def close(self):
        super().close()
        self._ag = None
