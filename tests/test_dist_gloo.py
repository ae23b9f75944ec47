"""World-size-2 gloo tests of the sharded store's exchange protocol (CPU, no GPU).

The library's sharded calls (fmoe_store_create_sharded, csrc/dist.cu and
store.cu) run on the GPU; here the SAME protocol -- local top-k with global
ids, a packed payload of keys plus a per-query validity flag, ONE all-gather,
a (score desc, global id asc) merge; selections by the owner combined by
OR / sum; inserts appended in slot order, RDY candidates gathered and merged,
victims resolved in batch order, owners write -- is modelled with the CPU
oracle as the local engine (tests only) and real torch.distributed gloo
collectives, and pinned to the unsharded oracle store.  The
product's HOST-transport callback (paper_2502_05370_b200/dist.py) is tested
with gloo too."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import fmoe_synth as S
from oracle import fmoe_oracle as O

SH = S.Shape("dist", 6, 8, 2, 24, n_clusters=4)


def shard_range(n_total, rank, world):
    """The library's shard map: contiguous ranges of P = ceil(C / G) slots."""
    per = (n_total + world - 1) // world
    lo = min(rank * per, n_total)
    return min(lo + per, n_total) - lo, lo


class OracleBackend:
    def __init__(self, cap, offset, dtype):
        self.st = O.Store(cap, SH.L, SH.E, SH.D, 3)
        self.off, self.dt = offset, dtype

    def _q(self, x):
        return None if x is None else O.quantize(x.numpy(), self.dt)

    def search(self, q_emb, q_prefix, ell, w, k):
        s, i = self.st.search(self._q(q_emb), self._q(q_prefix), ell, w, k)
        i = np.where(i >= 0, i + self.off, -1)
        return torch.from_numpy(s), torch.from_numpy(i)

    def merge(self, scores, ids, k):
        s, i = O.merge_topk([scores[g].numpy() for g in range(scores.shape[0])],
                            [ids[g].numpy() for g in range(ids.shape[0])], k)
        return torch.from_numpy(s), torch.from_numpy(i)

    def select(self, map_id, score, delta, lb, le):
        loc = [int(m) - self.off if 0 <= int(m) - self.off < self.st.n else -1 for m in map_id]
        masks, counts = O.select_experts(self.st.maps, loc, score.double().tolist(), delta, list(range(lb, le)), SH.K)
        m = torch.tensor([[v if v < 2 ** 63 else v - 2 ** 64 for v in r] for r in masks], dtype=torch.int64)
        return m, torch.tensor(counts, dtype=torch.int32)

    def append(self, emb, maps):
        self.st.insert(self._q(emb), self._q(maps))

    def write(self, emb, maps, slot):
        e, m = self._q(emb), self._q(maps)
        for x, y in enumerate(slot.tolist()):
            if 0 <= y - self.off < self.st.n:
                self.st.emb[y - self.off], self.st.maps[y - self.off] = e[x], m[x]

    def resolve(self, ids):
        out, taken = [], set()
        for row in ids.tolist():
            v = next((y for y in row if y >= 0 and y not in taken), -1)
            taken.add(v)
            out.append(v)
        return torch.tensor(out, dtype=torch.int64)

    def close(self):
        pass


class ShardProtocolModel:
    """The sharded store's collective protocol (store.cu's sharded_* functions)."""

    def __init__(self, C, dtype):
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.C = C
        self.cap, self.off = shard_range(C, self.rank, self.world)
        self.b = OracleBackend(self.cap, self.off, dtype)
        self.n_total = 0

    def _exchange(self, s, i):
        """pack [B][k] keys + [B] flags -> all-gather -> merge (validity: every rank's flag)."""
        B, k = s.shape
        pay = torch.zeros(B * k * 2 + B, dtype=torch.float64)
        pay[:B * k] = torch.from_numpy(np.nan_to_num(s.numpy().ravel(), nan=-np.inf))
        pay[B * k:2 * B * k] = torch.from_numpy(i.numpy().ravel().astype(np.float64))
        pay[2 * B * k:] = torch.from_numpy((~np.isnan(s.numpy()[:, 0])).astype(np.float64))
        out = torch.empty(self.world * pay.numel(), dtype=torch.float64)
        dist.all_gather_into_tensor(out, pay)
        out = out.view(self.world, -1)
        gs = out[:, :B * k].view(self.world, B, k).numpy()
        gi = out[:, B * k:2 * B * k].view(self.world, B, k).numpy().astype(np.int64)
        valid = out[:, 2 * B * k:].numpy().min(axis=0) > 0
        ms, mi = O.merge_topk([gs[g] for g in range(self.world)], [gi[g] for g in range(self.world)], k)
        ms[~valid], mi[~valid] = np.nan, -1
        return torch.from_numpy(ms), torch.from_numpy(mi)

    def search(self, q_emb, q_prefix, ell, w, k):
        s, i = self.b.search(q_emb, q_prefix, ell, w, k)
        return self._exchange(s, i)

    def search_semantic(self, q_emb, k=1):
        return self.search(q_emb, None, 0, 1.0, k)

    def search_trajectory(self, q_prefix, ell, k=1):
        return self.search(None, q_prefix[:, :ell].contiguous(), ell, 0.0, k)

    def search_blend(self, q_emb, q_prefix, ell, w_sem=-1.0, k=1):
        return self.search(q_emb, q_prefix[:, :ell].contiguous(), ell, 3 / SH.L if w_sem < 0 else w_sem, k)

    def select_experts(self, map_id, score, delta=-1.0, lb=0, le=None):
        mask, cnt = self.b.select(map_id, score, delta, lb, le)     # owner non-zero, others zero
        both = torch.cat([mask, cnt.to(torch.int64)], dim=1)
        out = torch.empty(self.world, *both.shape, dtype=torch.int64)
        dist.all_gather_into_tensor(out.view(-1), both.view(-1))
        T = mask.shape[1]
        m = out[:, :, :T]
        comb = m[0]
        for g in range(1, self.world):
            comb = comb | m[g]
        return comb, out[:, :, T:].sum(0).to(torch.int32)

    def insert(self, emb, maps):
        B, n0 = emb.shape[0], self.n_total
        a = min(B, self.C - n0)
        nrep = B - a
        slots = list(range(n0, n0 + a)) + [-1] * nrep
        if nrep > 0 and n0 > 0:
            kk = min(nrep, n0)
            q_e, q_m = emb[a:], maps[a:]
            n_loc0 = min(max(n0 - self.off, 0), self.cap)
            if n_loc0 > 0:
                s, i = self.b.search(q_e, q_m, SH.L, 3 / SH.L, kk)   # RDY over the rows present before
            else:
                s, i = torch.full((nrep, kk), -np.inf, dtype=torch.float64), torch.full((nrep, kk), -1)
            _, mi = self._exchange(s, i)
            victims = self.b.resolve(mi)
            slots[a:] = victims.tolist()
        # every rank writes the rows whose global slot it owns (appends and victims)
        for x, y in enumerate(slots):
            if self.off <= y < self.off + self.cap:
                if y - self.off == self.b.st.n:
                    self.b.append(emb[x:x + 1], maps[x:x + 1])
                else:
                    self.b.write(emb[x:x + 1], maps[x:x + 1], torch.tensor([y]))
        self.n_total = n0 + a
        rep = [-1] * a + slots[a:]
        return torch.tensor(slots), torch.tensor(rep)


def _worker(rank, world, port, dtype, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    try:
        C = 103                                  # not a multiple of world: ragged last shard
        st = ShardProtocolModel(C, dtype)
        emb, maps, _ = S.store_rows(SH, 5, 0, C + 40)
        res = {}
        res["ins0"] = st.insert(emb[:60], maps[:60])          # appends on rank 0 only
        res["ins1"] = st.insert(emb[60:C], maps[60:C])        # crosses the shard boundary
        qe, qm, _ = S.queries(SH, 5, C, 5)
        res["sem"] = st.search_semantic(qe, 4)
        res["traj"] = st.search_trajectory(qm, 3, 6)
        res["blend"] = st.search_blend(qe, qm, SH.L, -1.0, 3)
        s, i = res["sem"]
        res["sel"] = st.select_experts(i[:, 0].contiguous(), s[:, 0].contiguous(), -1.0, 0, SH.L)
        res["ins2"] = st.insert(emb[C:C + 7], maps[C:C + 7])  # RDY replacement across shards
        res["ins3"] = st.insert(torch.cat([emb[5:6]] * 3), torch.cat([maps[5:6]] * 3))  # duplicates
        res["sem2"] = st.search_semantic(qe, 4)
        q.put((rank, {k: tuple(t.cpu().numpy().copy() for t in v) for k, v in res.items()}))  # by value
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_sharded_store_equals_unsharded(dtype):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dtype, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    out = {r: {k: tuple(torch.from_numpy(a) for a in v) for k, v in d.items()} for r, d in out.items()}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # identical on every rank
    for key in out[0]:
        for a, b in zip(out[0][key], out[1][key]):
            assert torch.equal(a, b), key
    # equal to the unsharded oracle store fed the same calls
    C = 103
    ref = O.Store(C, SH.L, SH.E, SH.D, 3)
    emb, maps, _ = S.store_rows(SH, 5, 0, C + 40)
    Qz = lambda x: O.quantize(x.numpy(), dtype)
    r = out[0]
    sl, rp = ref.insert(Qz(emb[:60]), Qz(maps[:60]))
    assert r["ins0"][0].tolist() == sl and r["ins0"][1].tolist() == rp
    sl, rp = ref.insert(Qz(emb[60:C]), Qz(maps[60:C]))
    assert r["ins1"][0].tolist() == sl
    qe, qm, _ = S.queries(SH, 5, C, 5)
    for key, (w, ell, k) in {"sem": (1.0, 0, 4), "traj": (0.0, 3, 6), "blend": (3 / SH.L, SH.L, 3)}.items():
        s, i = ref.search(Qz(qe), Qz(qm), ell, w, k)
        assert np.array_equal(r[key][1].numpy(), i), key
        assert np.allclose(r[key][0].numpy(), s, atol=0, rtol=0), key
    s, i = ref.search(Qz(qe), None, 0, 1.0, 4)
    masks, counts = O.select_experts(ref.maps, i[:, 0].tolist(), s[:, 0].tolist(), -1.0, list(range(SH.L)), SH.K)
    assert r["sel"][1].tolist() == counts
    sl, rp = ref.insert(Qz(emb[C:C + 7]), Qz(maps[C:C + 7]))
    assert r["ins2"][0].tolist() == sl and r["ins2"][1].tolist() == rp
    sl, rp = ref.insert(Qz(torch.cat([emb[5:6]] * 3)), Qz(torch.cat([maps[5:6]] * 3)))
    assert r["ins3"][0].tolist() == sl and len(set(sl)) == 3
    s, i = ref.search(Qz(qe), None, 0, 1.0, 4)
    assert np.array_equal(r["sem2"][1].numpy(), i)


def test_shard_range_partitions_the_store():
    from paper_2502_05370_b200 import dist as fd
    for n in (1, 7, 100, 16_000_000):
        for G in (1, 2, 3, 4, 8):
            spans = [fd.shard_range(n, r, G) for r in range(G)]
            assert spans == [shard_range(n, r, G) for r in range(G)]
            assert sum(c for c, _ in spans) == n
            pos = 0
            for c, off in spans:
                assert off == pos or c == 0
                pos = off + c if c else pos


def _ag_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    from paper_2502_05370_b200 import dist as fd
    try:
        ag = fd._HostAllGather()
        n = 37
        send = (ctypes.c_uint8 * n)(*[(rank * 50 + j) % 256 for j in range(n)])
        recv = (ctypes.c_uint8 * (n * world))()
        rc = ag.cfn(ctypes.addressof(send), ctypes.addressof(recv), n, None)   # through the C function pointer
        q.put((rank, rc, bytes(recv)))
    finally:
        dist.destroy_process_group()


def test_host_transport_allgather_callback():
    """The product's fmoe_allgather_fn for the HOST transport: recv[world][bytes]
    in rank order, called through its C function pointer as the library does."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ag_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict((r, (rc, b)) for r, rc, b in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = bytes([(r * 50 + j) % 256 for r in range(world) for j in range(37)])
    for r in range(world):
        assert out[r][0] == 0 and out[r][1] == want
