"""The sharded store through the C ABI (fmoe_store_create_sharded): 2 ranks on
one B200 with the HOST transport (the library calls back into a gloo
all-gather; NCCL refuses two ranks on one device), against the unsharded
store -- every search, selection, session step, sweep and insert must be
bit-identical -- plus the NCCL transport at world size 1."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import fmoe_synth as S

pytestmark = pytest.mark.gpu
SH = S.Shape("gdist", 8, 16, 2, 136, n_clusters=8)          # E = 16: per-step session path
MX = S.Shape("gdist-mx", 8, 8, 2, 96, n_clusters=8)          # E = 8 bf16: the fused sweep
C = 5003


def _calls(lib, st, sh, emb, maps, dev):
    """The same sequence of ABI calls on a (sharded or unsharded) store; outputs by value."""
    res = {}
    slot, rep = st.insert(emb[:C].to(dev), maps[:C].to(dev))
    res["ins0"] = (slot, rep)
    qe, qm, _ = S.queries(sh, 9, C, 24)
    qe, qm = qe.to(dev), qm.to(dev)
    qe[5] = 0.0                                              # a zero-norm query: (NaN, -1) everywhere
    res["sem"] = st.search_semantic(qe[:3], 5)               # GEMV path
    res["sem_b"] = st.search_semantic(qe, 8)                 # tcgen05 path (approx + exact re-rank)
    res["traj"] = st.search_trajectory(qm[:2], 4, 3)
    res["traj_b"] = st.search_trajectory(qm, 7, 8)
    res["blend_b"] = st.search_blend(qe, qm, 5, -1.0, 4)
    s, i = res["sem"]
    res["sel"] = st.select_experts(i[:, 0].contiguous(), s[:, 0].contiguous(), -1.0, 0, sh.L)
    # semantic cosines -> blend_cos / insert_cos (the cosine side output is per shard)
    n_local = len(st) if not hasattr(st, "cap_local") else st.cap_local
    stride = (n_local + 3) // 4 * 4
    cos = torch.empty(24, stride, device=dev)
    s0 = torch.empty(24, 8, device=dev)
    i0 = torch.empty(24, 8, dtype=torch.int64, device=dev)
    lib.fmoe_search_semantic_cos(st._h, qe, 8, s0, i0, cos, stride)
    res["sem_cos"] = (s0, i0)
    s2 = torch.empty(24, 8, device=dev)
    i2 = torch.empty(24, 8, dtype=torch.int64, device=dev)
    lib.fmoe_search_blend_cos(st._h, cos, stride, qm[:, :5].contiguous(), 5, -1.0, 8, s2, i2)
    res["blend_cos"] = (s2, i2)
    # sessions: incremental (B = 2, fused selection) and batched (B = 24, tcgen05)
    a = st.trajectory_session(2)
    b = st.trajectory_session(24)
    for ell in range(1, 4):
        res[f"step{ell}"] = a.step_select(qm[:2, ell - 1].contiguous(), 2, -1.0, ell + 2, ell + 3)
        res[f"bstep{ell}"] = b.step(qm[:, ell - 1].contiguous(), 8)
    a.close()
    b.close()
    sw = st.trajectory_session(1)
    res["sweep"] = sw.sweep(qm[:1].permute(1, 0, 2).contiguous(), -1.0, 3)
    sw.close()
    # insert at capacity: replacement through the cross-shard RDY; a zero-norm row
    ne, nm = emb[C:C + 40].clone(), maps[C:C + 40].clone()
    ne[3] = 0.0
    res["ins1"] = st.insert(ne.to(dev), nm.to(dev))
    sl = torch.empty(24, dtype=torch.int64, device=dev)
    rp = torch.empty(24, dtype=torch.int64, device=dev)
    lib.fmoe_search_semantic_cos(st._h, emb[C + 40:C + 64].to(dev), 8, s0, i0, cos, stride)
    lib.fmoe_store_insert_cos(st._h, emb[C + 40:C + 64].to(dev), maps[C + 40:C + 64].to(dev), cos, stride, sl, rp)
    res["ins_cos"] = (sl, rp)
    # > 64 replacements in one call: sub-batches with the claimed-slot bitmap
    big_e = torch.cat([emb[100:101].repeat(30, 1), emb[200:270]])
    big_m = torch.cat([maps[100:101].repeat(30, 1, 1), maps[200:270]])
    res["ins_big"] = st.insert(big_e.to(dev), big_m.to(dev))
    res["sem2"] = st.search_semantic(qe, 8)
    res["size"] = (torch.tensor([len(st)]),)
    return {k: tuple(t.cpu().numpy().copy() for t in v if t is not None) for k, v in res.items()}


def _worker(rank, world, port, sh_name, q):
    import datetime
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    import paper_2502_05370_b200 as lib
    from paper_2502_05370_b200 import dist as fd
    sh = SH if sh_name == "SH" else MX
    try:
        torch.cuda.set_device(0)
        st = fd.ShardedExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, C, "bf16", device=0, transport="host")
        emb, maps, _ = S.store_rows(sh, 9, 0, C + 64)
        out = _calls(lib, st, sh, emb, maps, "cuda")
        torch.cuda.synchronize()
        q.put((rank, out))
        st.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sh_name", ["SH", "MX"])
def test_two_ranks_host_transport_equal_unsharded(lib, sh_name):
    sh = SH if sh_name == "SH" else MX
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, sh_name, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref_st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, C, "bf16")
    emb, maps, _ = S.store_rows(sh, 9, 0, C + 64)
    ref = _calls(lib, ref_st, sh, emb, maps, "cuda")
    ref_st.close()
    for key in ref:
        if key in ("blend_cos", "ins_cos"):
            continue                     # compared below (inputs are per-shard cosines)
        for r in (0, 1):
            for a, b in zip(out[r][key], ref[key]):
                assert np.array_equal(a, b, equal_nan=True), (key, r, a, b)
    for key in ("blend_cos", "ins_cos"):
        for r in (0, 1):
            for a, b in zip(out[r][key], ref[key]):
                assert np.array_equal(a, b, equal_nan=True), (key, r)
    assert np.isnan(out[0]["sem_b"][0][5]).all() and (out[0]["sem_b"][1][5] == -1).all()
    assert out[0]["ins1"][0][3] >= 0                     # the zero-norm row still takes a victim (R3)


def test_nccl_transport_world_one(lib):
    """The NCCL path of the library (communicator, ncclAllGather on the stream,
    merge kernel) at world size 1 on one GPU: equal to the unsharded store."""
    sh = SH
    uid = lib.fmoe_get_nccl_unique_id()
    h = lib.fmoe_store_create_sharded(sh.L, sh.E, sh.K, sh.D, 3, C, "bf16", 0, 0, 1, "nccl", uid)
    st = lib.ExpertMapStore.__new__(lib.ExpertMapStore)
    st.L, st.E, st.K, st.D, st.d, st.capacity, st.dtype, st.id_offset = sh.L, sh.E, sh.K, sh.D, 3, C, "bf16", 0
    st.device = torch.device("cuda", 0)
    st._h = h
    emb, maps, _ = S.store_rows(sh, 9, 0, C + 64)
    got = _calls(lib, st, sh, emb, maps, "cuda")
    st.close()
    ref_st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, C, "bf16")
    ref = _calls(lib, ref_st, sh, emb, maps, "cuda")
    ref_st.close()
    for key in ref:
        for a, b in zip(got[key], ref[key]):
            assert np.array_equal(a, b, equal_nan=True), key
