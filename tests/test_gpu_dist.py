"""The sharded store with the CUDA backend: 2 ranks on one B200 (gloo for the
collectives, host-staged), against the unsharded CUDA store and the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import fmoe_synth as S

pytestmark = pytest.mark.gpu
SH = S.Shape("gdist", 8, 16, 2, 136, n_clusters=8)
C = 5003


def _worker(rank, world, port, q):
    import datetime
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    from paper_2502_05370_b200 import dist as fd
    try:
        torch.cuda.set_device(0)
        st = fd.ShardedExpertMapStore(SH.L, SH.E, SH.K, SH.D, 3, C, "bf16", device=0)
        emb, maps, _ = S.store_rows(SH, 9, 0, C + 64)
        res = {}
        res["ins0"] = st.insert(emb[:C].cuda(), maps[:C].cuda())
        qe, qm, _ = S.queries(SH, 9, C, 24)
        qe, qm = qe.cuda(), qm.cuda()
        res["sem"] = st.search_semantic(qe[:3], 5)            # GEMV path
        res["sem_b"] = st.search_semantic(qe, 8)              # tcgen05 path
        res["traj"] = st.search_trajectory(qm[:2], 4, 3)
        res["traj_b"] = st.search_trajectory(qm, 7, 8)
        res["blend_b"] = st.search_blend(qe, qm, 5, -1.0, 4)
        s, i = res["sem"]
        res["sel"] = st.select_experts(i[:, 0].contiguous(), s[:, 0].contiguous(), -1.0, 0, SH.L)
        res["ins1"] = st.insert(emb[C:C + 64].cuda(), maps[C:C + 64].cuda())
        res["sem2"] = st.search_semantic(qe, 8)
        q.put((rank, {k: tuple(t.cpu().numpy().copy() for t in v) for k, v in res.items()}))  # by value
        torch.cuda.synchronize()
        st.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_one_gpu_equal_unsharded(lib):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(2))
    out = {r: {k: tuple(torch.from_numpy(a) for a in v) for k, v in d.items()} for r, d in out.items()}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for key in out[0]:
        for a, b in zip(out[0][key], out[1][key]):
            assert torch.equal(a, b), key
    # unsharded CUDA store, same calls: bit-identical ids and scores
    ref = lib.ExpertMapStore(SH.L, SH.E, SH.K, SH.D, 3, C, "bf16")
    emb, maps, _ = S.store_rows(SH, 9, 0, C + 64)
    sl, rp = ref.insert(emb[:C].cuda(), maps[:C].cuda())
    assert out[0]["ins0"][0].tolist() == sl.cpu().tolist()
    qe, qm, _ = S.queries(SH, 9, C, 24)
    qe, qm = qe.cuda(), qm.cuda()
    r = out[0]
    checks = {"sem": ref.search_semantic(qe[:3], 5), "sem_b": ref.search_semantic(qe, 8),
              "traj": ref.search_trajectory(qm[:2], 4, 3), "traj_b": ref.search_trajectory(qm, 7, 8),
              "blend_b": ref.search_blend(qe, qm, 5, -1.0, 4)}
    for key, (s_, i_) in checks.items():
        assert torch.equal(r[key][1], i_.cpu()), key
        assert torch.equal(r[key][0], s_.cpu()), key
    sl, rp = ref.insert(emb[C:C + 64].cuda(), maps[C:C + 64].cuda())
    assert r["ins1"][0].tolist() == sl.cpu().tolist()
    assert r["ins1"][1].tolist() == rp.cpu().tolist()
    s_, i_ = ref.search_semantic(qe, 8)
    assert torch.equal(r["sem2"][1], i_.cpu())
    ref.close()
