"""World-size-2 gloo tests of the sharded store's host-side logic (CPU, no GPU).

The local shard operations use the CPU oracle as the backend (tests only); the
collectives (all-gather of candidate lists, all-reduce of selections) are real
torch.distributed gloo calls.  Pins SURVEY §8(c) c9: merged per-shard results
equal the unsharded store's, for search, selection and RDY insertion."""
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


def _worker(rank, world, port, dtype, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    from paper_2502_05370_b200 import dist as fd
    try:
        C = 103                                  # not a multiple of world: ragged last shard
        cap, off = fd.shard_range(C, rank, world)
        st = fd.ShardedExpertMapStore(SH.L, SH.E, SH.K, SH.D, 3, C, dtype,
                                      backend=OracleBackend(cap, off, dtype))
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
            assert sum(c for c, _ in spans) == n
            pos = 0
            for c, off in spans:
                assert off == pos or c == 0
                pos = off + c if c else pos
