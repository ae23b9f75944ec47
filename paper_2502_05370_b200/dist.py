"""Sharded expert-map store over the ranks of a torch.distributed group.

Rank r of G holds the global slots [r*C, (r+1)*C) of a store of G*C contexts
(its local store is created with id_offset = r*C, so every id that crosses the
ABI is global).  Store rows are independent, so the path shards with exactly
one exchange step per call:

* search (Eq. 1 / Eq. 2 / blend): every rank scores its shard and keeps its
  local top-k (sm_100a kernels); the B x k (score, id) lists are all-gathered
  (ONE collective: NCCL over NVLink/NVSwitch on B200, gloo in the CPU tests)
  and every rank merges the G lists with the same merge kernel -> results are
  identical on every rank and bit-identical to the unsharded store, because a
  row's score does not depend on which rank computes it and ties break by the
  global id.
* select (Eq. 4-6): the matched map lives on one rank; every rank runs the
  selection (non-owners produce mask 0 / count 0) and one all-reduce(SUM)
  publishes the owner's result.
* insert (Reading R8): appends fill ranks in slot order; once full,
  every rank finds its local RDY top-kk over the contexts present before the
  call, the lists are all-gathered and merged, victims are resolved in batch
  order exactly as in the unsharded insert, and each owner overwrites its own
  victims.

The collective calls go through torch.distributed (plumbing); every score,
merge and selection runs in the library's kernels.  The local operations are
behind a small backend object so that the host-side logic (ownership, id
offsets, gather layout, resolution order) is covered by world-size-2 gloo tests
on CPU, where the backend is the CPU oracle (tests only).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n_total: int, rank: int, world: int):
    """(local capacity, id_offset) of `rank`: equal contiguous slot ranges."""
    per = (n_total + world - 1) // world
    lo = min(rank * per, n_total)
    hi = min(lo + per, n_total)
    return hi - lo, lo


class CudaBackend:
    """Local shard operations through the C ABI (libfmoe_b200.so)."""

    def __init__(self, L, E, K, D, d, capacity, dtype, device, id_offset):
        import paper_2502_05370_b200 as fm
        self.fm = fm
        self.store = fm.ExpertMapStore(L, E, K, D, d, capacity, dtype, device=device, id_offset=id_offset)
        self.device = self.store.device

    def size(self):
        return len(self.store)

    def search(self, q_emb, q_prefix, ell, w, k):
        st = self.store
        if w == 1.0:
            return st.search_semantic(q_emb, k)
        if w == 0.0:
            return st.search_trajectory(q_prefix, ell, k)
        return st.search_blend(q_emb, q_prefix, ell, w, k)

    def merge(self, scores, ids, k):
        B = scores.shape[1]
        out_s = torch.empty(B, k, device=self.device)
        out_i = torch.empty(B, k, dtype=torch.int64, device=self.device)
        self.fm.fmoe_topk_merge(scores.contiguous(), ids.contiguous(), k, out_s, out_i, device=self.device.index)
        return out_s, out_i

    def select(self, map_id, score, delta, lb, le):
        return self.store.select_experts(map_id, score, delta, lb, le)

    def append(self, emb, maps):
        self.store.insert(emb.contiguous(), maps.contiguous())

    def write(self, emb, maps, slot):
        self.fm.fmoe_store_write(self.store._h, emb.contiguous(), maps.contiguous(), slot.contiguous())

    def resolve(self, ids):
        out = torch.empty(ids.shape[0], dtype=torch.int64, device=self.device)
        self.fm.fmoe_resolve_victims(ids.contiguous(), out, device=self.device.index)
        return out

    def close(self):
        self.store.close()


class ShardedExpertMapStore:
    """Collective API: every rank calls every method with the same arguments."""

    def __init__(self, L, E, K, D, d, capacity_total, dtype="bf16", group=None, backend=None, device=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.L, self.E, self.K, self.D, self.d = L, E, K, D, d
        self.capacity_total = capacity_total
        self.cap_local, self.offset = shard_range(capacity_total, self.rank, self.world)
        self.per = (capacity_total + self.world - 1) // self.world
        if backend is None:
            dev = device if device is not None else torch.cuda.current_device()
            backend = CudaBackend(L, E, K, D, d, self.cap_local, dtype, dev, self.offset)
        self.b = backend
        self.n_total = 0
        self._cpu_collectives = dist.get_backend(group) == "gloo"

    # ------------------------------------------------------------ helpers
    def _all_gather_lists(self, s, i):
        """(scores [B,k] f32, ids [B,k] i64) -> [G,B,k] each, one collective."""
        B, k = s.shape
        packed = torch.empty(B, k, 2, dtype=torch.int64, device=s.device)
        if s.dtype == torch.float32:
            packed[..., 0] = s.contiguous().view(torch.int32).to(torch.int64)
        else:
            packed[..., 0] = s.contiguous().view(torch.int64)
        packed[..., 1] = i
        stage = self._cpu_collectives and packed.is_cuda      # gloo: host staging
        src = packed.cpu() if stage else packed
        out = torch.empty(self.world * B, k, 2, dtype=torch.int64, device=src.device)
        dist.all_gather_into_tensor(out, src, group=self.group)
        out = out.view(self.world, B, k, 2).to(s.device)
        if s.dtype == torch.float32:
            scores = out[..., 0].to(torch.int32).view(torch.float32)
        else:
            scores = out[..., 0].contiguous().view(torch.float64)
        return scores, out[..., 1]

    # ------------------------------------------------------------ search
    def search(self, q_emb, q_prefix, ell, w, k):
        s, i = self.b.search(q_emb, q_prefix, ell, w, k)
        if self.world == 1:
            return s, i
        gs, gi = self._all_gather_lists(s, i)
        return self.b.merge(gs, gi, k)

    def search_semantic(self, q_emb, k=1):
        return self.search(q_emb, None, 0, 1.0, k)

    def search_trajectory(self, q_prefix, ell, k=1):
        return self.search(None, q_prefix[:, :ell].contiguous(), ell, 0.0, k)

    def search_blend(self, q_emb, q_prefix, ell, w_sem=-1.0, k=1):
        w = self.d / self.L if w_sem < 0 else w_sem
        return self.search(q_emb, q_prefix[:, :ell].contiguous(), ell, w, k)

    # ------------------------------------------------------------ select
    def select_experts(self, map_id, score, delta=-1.0, layer_begin=0, layer_end=None):
        layer_end = self.L if layer_end is None else layer_end
        mask, cnt = self.b.select(map_id, score, delta, layer_begin, layer_end)
        if self.world > 1:
            both = torch.cat([mask, cnt.to(torch.int64)], dim=1)   # one collective
            src = both.cpu() if (self._cpu_collectives and both.is_cuda) else both
            dist.all_reduce(src, group=self.group)                 # exactly one owner contributes
            both = src.to(mask.device)
            T = mask.shape[1]
            mask, cnt = both[:, :T].contiguous(), both[:, T:].to(torch.int32)
        return mask, cnt

    # ------------------------------------------------------------ insert
    def insert(self, emb, maps):
        """Returns (slot[B], replaced[B]) as CPU int64 tensors (host bookkeeping)."""
        B = emb.shape[0]
        n0 = self.n_total
        a = min(B, self.capacity_total - n0)
        nrep = B - a
        slots = torch.full((B,), -1, dtype=torch.int64)
        replaced = torch.full((B,), -1, dtype=torch.int64)
        victims = None
        if nrep > 0 and n0 > 0:
            if nrep > 64:
                raise ValueError("more than 64 rows of one insert need replacement")
            kk = min(nrep, n0)
            q_e, q_m = emb[a:].contiguous(), maps[a:].contiguous()
            # RDY over the contexts present before this call (ids < n0)
            s, i = self.b.search(q_e, q_m, self.L, self.d / self.L, kk)
            if self.world > 1:
                gs, gi = self._all_gather_lists(s, i)
                s, i = self.b.merge(gs, gi, kk)
            victims = self.b.resolve(i)
        # appends: global slot n0 + x lives on rank (n0 + x) // per
        for x in range(a):
            slots[x] = n0 + x
        if a > 0:
            lo = max(self.offset, n0)
            hi = min(self.offset + self.cap_local, n0 + a)
            if hi > lo:
                self.b.append(emb[lo - n0:hi - n0], maps[lo - n0:hi - n0])
        self.n_total = n0 + a
        if victims is not None:
            self.b.write(q_e, q_m, victims)
            v = victims.cpu()
            slots[a:] = v
            replaced[a:] = v
        return slots, replaced

    def __len__(self):
        return self.n_total

    def close(self):
        self.b.close()
