"""GPU parity: the CUDA path through the C ABI vs the fp64 CPU oracle.

Both sides get the same seeded fp32 inputs (fmoe_synth).  The oracle is fed the
values the store holds -- inputs rounded to the store dtype with RNE
(``O.quantize``, the "O-store" view of SURVEY §8(c) c8) -- and the comparison
rules are DESIGN.md §"Parity contract":
  * scores: |gpu - oracle| <= 1e-5 (absolute; |score| <= 1);
  * ids: exact at every rank whose oracle score is separated from its
    neighbours by more than 1e-5; elsewhere the returned id's oracle score
    must be within 1e-5 of the oracle score at that rank;
  * expert sets / counts / insert slots: bit-exact given the same (id, score).
Sizes span many 32-row tiles, several blocks and a ragged tail.
"""
import numpy as np
import pytest
import torch

import fmoe_synth as S
from oracle import fmoe_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5

SHAPES = {
    "mixtral_tiny": S.Shape("mixtral-tiny", 32, 8, 2, 64, n_clusters=16),
    "qwen_small": S.Shape("qwen-small", 24, 60, 4, 256, n_clusters=32),
    "phi_small": S.Shape("phi-small", 32, 16, 2, 520, n_clusters=32),   # D not a multiple of 16 B
}


def make(lib, shape, N, dtype, cap=None, seed=1):
    emb, maps, _ = S.store_rows(shape, seed, 0, N)
    st = lib.ExpertMapStore(shape.L, shape.E, shape.K, shape.D, 3, cap or N, dtype)
    for a in range(0, N, 4096):
        st.insert(emb[a:a + 4096].cuda(), maps[a:a + 4096].cuda())
    torch.cuda.synchronize()
    return st, emb.numpy(), maps.numpy()


def check_topk(gs, gi, ref, k, tol=TOL):
    """ref: oracle B x N score matrix (O-store view)."""
    gs = gs.cpu().numpy().astype(np.float64)
    gi = gi.cpu().numpy()
    rs, ri = O.topk(ref, k)
    B = ref.shape[0]
    for x in range(B):
        if np.isnan(ref[x]).any():
            assert np.isnan(gs[x]).all() and (gi[x] == -1).all()
            continue
        valid = ri[x] >= 0
        assert np.array_equal(gi[x][~valid], ri[x][~valid])
        assert np.all(np.isneginf(gs[x][~valid]))
        assert np.all(np.abs(gs[x][valid] - rs[x][valid]) <= tol), (x, gs[x], rs[x])
        ids = gi[x][valid]
        assert len(set(ids.tolist())) == len(ids)
        nv = int(valid.sum())
        full = np.sort(ref[x])[::-1]          # all oracle scores, descending
        for r in range(nv):
            lo = full[r - 1] - full[r] if r > 0 else np.inf
            hi = full[r] - full[r + 1] if r + 1 < full.shape[0] else np.inf
            if min(lo, hi) > tol:
                assert gi[x, r] == ri[x, r], (x, r, gi[x], ri[x])
            else:
                assert abs(ref[x, gi[x, r]] - rs[x, r]) <= tol


@pytest.fixture(scope="module", params=[("mixtral_tiny", "f32"), ("mixtral_tiny", "bf16"), ("qwen_small", "bf16"),
                                        ("qwen_small", "f32"), ("phi_small", "bf16")])
def setup(request, lib):
    name, dtype = request.param
    shape = SHAPES[name]
    N = 3001
    st, emb, maps = make(lib, shape, N, dtype)
    q_emb, q_maps, planted = S.queries(shape, 1, N, 6)   # seed of make()
    Qe = O.quantize(emb, dtype)
    Qm = O.quantize(maps, dtype)
    yield dict(lib=lib, st=st, shape=shape, dtype=dtype, N=N, emb=emb, maps=maps, Qe=Qe, Qm=Qm,
               q_emb=q_emb, q_maps=q_maps, planted=planted.numpy())
    st.close()


def test_store_holds_the_quantised_rows(setup):
    e, m = setup["st"].read(0, 257)
    assert np.array_equal(e.cpu().numpy().astype(np.float64), setup["Qe"][:257])
    assert np.array_equal(m.cpu().numpy().astype(np.float64), setup["Qm"][:257])


@pytest.mark.parametrize("B,k", [(1, 1), (3, 8), (6, 40)])
def test_semantic(setup, B, k):
    st, dt = setup["st"], setup["dtype"]
    q = setup["q_emb"][:B]
    gs, gi = st.search_semantic(q.cuda(), k)
    ref = O.semantic_scores(O.quantize(q.numpy(), dt), setup["Qe"])
    check_topk(gs, gi, ref, k)
    # O-def view: within the bf16 contract of the unrounded definition
    if dt == "bf16":
        ref_def = O.semantic_scores(q.numpy(), setup["emb"])
        rs, _ = O.topk(ref_def, k)
        assert np.all(np.abs(gs.cpu().numpy() - rs) <= 2e-3)
    pl = setup["planted"][:B]
    for x in range(B):
        if pl[x] >= 0:
            assert gi[x, 0].item() == pl[x]


@pytest.mark.parametrize("ell", [1, 2, 3, 7, "L"])
@pytest.mark.parametrize("B,k", [(1, 1), (4, 8), (5, 33)])
def test_trajectory(setup, ell, B, k):
    st, dt, sh = setup["st"], setup["dtype"], setup["shape"]
    ell = sh.L if ell == "L" else ell
    qp = setup["q_maps"][:B, :ell].contiguous()
    gs, gi = st.search_trajectory(qp.cuda(), ell, k)
    ref = O.trajectory_scores(O.quantize(qp.numpy(), dt), setup["Qm"], ell)
    check_topk(gs, gi, ref, k)


@pytest.mark.parametrize("w", [-1.0, 0.3])
@pytest.mark.parametrize("B,ell", [(1, 5), (6, 31)])
def test_blend(setup, w, B, ell):
    st, dt, sh = setup["st"], setup["dtype"], setup["shape"]
    ell = min(ell, sh.L)
    w_eff = 3 / sh.L if w < 0 else w
    qe, qp = setup["q_emb"][:B], setup["q_maps"][:B, :ell].contiguous()
    gs, gi = st.search_blend(qe.cuda(), qp.cuda(), ell, w, 8)
    sem = O.semantic_scores(O.quantize(qe.numpy(), dt), setup["Qe"])
    trj = O.trajectory_scores(O.quantize(qp.numpy(), dt), setup["Qm"], ell)
    check_topk(gs, gi, O.blend_scores(sem, trj, np.float64(np.float32(w_eff))), 8)


def test_select_bit_exact(setup):
    st, sh = setup["st"], setup["shape"]
    rng = np.random.default_rng(7)
    B = 300
    ids = rng.integers(-1, setup["N"], B)
    sc = rng.uniform(-1.2, 1.2, B).astype(np.float32)
    sc[:5] = [1.0, -1.0, 0.0, np.nan, 0.7]
    for delta in (-1.0, 0.9, 0.0, 1.0):
        mask, cnt = st.select_experts(torch.from_numpy(ids).cuda(), torch.from_numpy(sc).cuda(), delta, 0, sh.L)
        d32 = float(np.float32(delta))
        om, oc = O.select_experts(setup["Qm"], ids.tolist(), sc.astype(np.float64).tolist(), d32,
                                  list(range(sh.L)), sh.K)
        gm = mask.cpu().numpy().view(np.uint64)
        assert np.array_equal(gm, np.array(om, dtype=np.uint64)), delta
        assert np.array_equal(cnt.cpu().numpy(), np.array(oc))


def test_search_then_select_pipeline(setup):
    """a6 -> a7: the matched map's first d layers (semantic path)."""
    st, sh, dt = setup["st"], setup["shape"], setup["dtype"]
    q = setup["q_emb"][:4].cuda()
    gs, gi = st.search_semantic(q, 1)
    mask, cnt = st.select_experts(gi[:, 0].contiguous(), gs[:, 0].contiguous(), -1.0, 0, 3)
    om, oc = O.select_experts(setup["Qm"], gi[:, 0].cpu().tolist(), gs[:, 0].cpu().double().tolist(), -1.0,
                              [0, 1, 2], sh.K)
    assert np.array_equal(mask.cpu().numpy().view(np.uint64), np.array(om, dtype=np.uint64))


def test_host_pointer_path(setup):
    """Same call with CPU (host) tensors: staged + synchronised by the library."""
    lib, st = setup["lib"], setup["st"]
    q = setup["q_emb"][:3].contiguous()
    s_h = torch.empty(3, 4)
    i_h = torch.empty(3, 4, dtype=torch.int64)
    lib.fmoe_search_semantic(st._h, q, 4, s_h, i_h)
    s_d, i_d = st.search_semantic(q.cuda(), 4)
    assert torch.equal(s_h, s_d.cpu()) and torch.equal(i_h, i_d.cpu())


def test_host_buffers_without_per_call_sync(setup):
    """fmoe_set_host_sync(0): host-buffer calls only enqueue their copies; a host
    output handed to the next call as its input is stream-ordered; after one
    stream sync every output equals the device path."""
    lib, st, sh = setup["lib"], setup["st"], setup["shape"]
    B = 3
    q = setup["q_emb"][:B].contiguous().pin_memory()
    qm = setup["q_maps"][:B].contiguous()
    s_h = torch.empty(B, 1).pin_memory()
    i_h = torch.empty(B, 1, dtype=torch.int64).pin_memory()
    m_h = torch.empty(B, 3, dtype=torch.int64).pin_memory()
    c_h = torch.empty(B, 3, dtype=torch.int32).pin_memory()
    t_s = torch.empty(B, 2).pin_memory()
    t_i = torch.empty(B, 2, dtype=torch.int64).pin_memory()
    lay = [qm[:, l].contiguous().pin_memory() for l in range(4)]
    sm_h = torch.empty(B, 1, dtype=torch.int64).pin_memory()
    sc_h = torch.empty(B, 1, dtype=torch.int32).pin_memory()
    sess = lib.fmoe_traj_session_create(st._h, B)
    prev = lib.fmoe_set_host_sync(0)
    try:
        lib.fmoe_search_semantic(st._h, q, 1, s_h, i_h)
        lib.fmoe_select_experts(st._h, i_h.view(-1), s_h.view(-1), -1.0, 0, 3, m_h, c_h)
        for l in range(4):
            lib.fmoe_traj_session_step_select(sess, lay[l], 2, t_s, t_i, -1.0, l + 3, l + 4, sm_h, sc_h)
        torch.cuda.current_stream().synchronize()
    finally:
        assert lib.fmoe_set_host_sync(prev) == 0
        lib.fmoe_traj_session_destroy(sess)
    gs, gi = st.search_semantic(q.cuda(), 1)
    gm, gc = st.select_experts(gi[:, 0].contiguous(), gs[:, 0].contiguous(), -1.0, 0, 3)
    assert torch.equal(s_h, gs.cpu()) and torch.equal(i_h, gi.cpu())
    assert torch.equal(m_h, gm.cpu()) and torch.equal(c_h, gc.cpu())
    ref = st.trajectory_session(B)
    try:
        for l in range(4):
            rs, ri, rm, rc = ref.step_select(lay[l].cuda(), 2, -1.0, l + 3, l + 4)
        assert torch.equal(t_s, rs.cpu()) and torch.equal(t_i, ri.cpu())
        assert torch.equal(sm_h, rm.cpu()) and torch.equal(sc_h, rc.cpu())
    finally:
        ref.close()


# ---------------------------------------------------------------- edge cases
def test_edge_cases(lib):
    sh = SHAPES["mixtral_tiny"]
    st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, 50, "bf16")
    q = torch.randn(2, sh.D, device="cuda")
    s, i = st.search_semantic(q, 3)                     # empty store
    assert (i == -1).all() and torch.isneginf(s).all()
    emb, maps, _ = S.store_rows(sh, 3, 0, 5)
    st.insert(emb.cuda(), maps.cuda())
    s, i = st.search_semantic(q, 8)                     # k > |store|
    assert (i[:, 5:] == -1).all() and torch.isneginf(s[:, 5:]).all() and (i[:, :5] >= 0).all()
    q[1] = 0                                            # zero-norm query -> NaN, -1
    s, i = st.search_semantic(q, 2)
    assert torch.isnan(s[1]).all() and (i[1] == -1).all() and (i[0] >= 0).all()
    # exact duplicate rows: bit-identical scores, the lowest id wins
    dup_e = emb[2:3].repeat(3, 1) * torch.tensor([[1.0], [2.0], [0.5]])
    dup_m = maps[2:3].repeat(3, 1, 1)
    st.insert(dup_e.cuda(), dup_m.cuda())               # slots 5, 6, 7
    s, i = st.search_semantic(emb[2:3].cuda(), 4)
    assert i[0].tolist() == [2, 5, 6, 7]
    s, i = st.search_trajectory(maps[2:3].cuda(), sh.L, 4)
    assert i[0].tolist() == [2, 5, 6, 7] and abs(s[0, 0].item() - 1.0) < 1e-6
    # argument errors are synchronous and typed
    with pytest.raises(lib.FmoeError):
        st.search_semantic(q, 65)
    with pytest.raises(lib.FmoeError):
        st.search_trajectory(maps[:1].cuda(), 0, 1)
    with pytest.raises(lib.FmoeError):
        st.select_experts(i[:, 0].contiguous(), s[:, 0].contiguous(), -1.0, 3, 3)
    st.close()


# ---------------------------------------------------------------- insert / dedup (a8)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_insert_matches_oracle_store(lib, dtype):
    sh = S.Shape("mix", 8, 8, 2, 48, n_clusters=4)
    C = 700
    emb, maps, _ = S.store_rows(sh, 11, 0, C + 400)
    st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, C, dtype)
    ref = O.Store(C, sh.L, sh.E, sh.D, 3)
    Qe, Qm = O.quantize(emb.numpy(), dtype), O.quantize(maps.numpy(), dtype)
    pos = 0
    for B in (600, 64, 40, 1, 7, 33, 64):   # append, mixed batch (100 + ...), then replacements
        e, m = emb[pos:pos + B], maps[pos:pos + B]
        slot, rep = st.insert(e.cuda(), m.cuda())
        rs, rr = ref.insert(Qe[pos:pos + B], Qm[pos:pos + B])
        assert slot.cpu().tolist() == rs, (B, pos)
        assert rep.cpu().tolist() == rr
        pos += B
        if pos + 64 > emb.shape[0]:
            break
    assert len(st) == ref.n == C
    ge, gm = st.read(0, C)
    assert np.array_equal(ge.cpu().numpy().astype(np.float64), ref.emb)
    assert np.array_equal(gm.cpu().numpy().astype(np.float64), ref.maps)
    st.close()


def test_insert_duplicate_batch_distinct_victims(lib):
    sh = S.Shape("mix", 8, 8, 2, 48, n_clusters=4)
    emb, maps, _ = S.store_rows(sh, 12, 0, 100)
    st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, 100, "bf16")
    st.insert(emb.cuda(), maps.cuda())
    # 5 identical copies of row 17: first replaces 17 (RDY=1), the rest take distinct next-best victims
    slot, rep = st.insert(emb[17:18].repeat(5, 1).cuda(), maps[17:18].repeat(5, 1, 1).cuda())
    s = slot.cpu().tolist()
    assert s[0] == 17 and len(set(s)) == 5 and rep.cpu().tolist() == s
    ref = O.Store(100, sh.L, sh.E, sh.D, 3)
    ref.insert(O.quantize(emb.numpy(), "bf16"), O.quantize(maps.numpy(), "bf16"))
    rs, _ = ref.insert(O.quantize(emb[17:18].repeat(5, 1).numpy(), "bf16"),
                       O.quantize(maps[17:18].repeat(5, 1, 1).numpy(), "bf16"))
    assert s == rs
    st.close()


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("B,n_dup", [(65, 0), (130, 70), (256, 100), (300, 200)])
def test_insert_large_batches_match_oracle(lib, dtype, B, n_dup):
    """More than 64 rows of one insert need a victim: sub-batches of 64, later
    ones skipping the slots earlier ones claimed (Reading R8) --
    equal to the oracle's sequential rule, with many rows competing for the
    same victims (n_dup copies of one stored context) and a mixed
    append/replace batch."""
    sh = S.Shape("mixL", 8, 8, 2, 48, n_clusters=4)
    C = 900
    emb, maps, _ = S.store_rows(sh, 14, 0, C + 400)
    st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, C, dtype)
    ref = O.Store(C, sh.L, sh.E, sh.D, 3)
    Qz = lambda x: O.quantize(x.numpy(), dtype)
    st.insert(emb[:C - 20].cuda(), maps[:C - 20].cuda())      # 20 slots left: the batch appends first
    ref.insert(Qz(emb[:C - 20]), Qz(maps[:C - 20]))
    be = torch.cat([emb[77:78].repeat(n_dup, 1), emb[C:C + B - n_dup]])
    bm = torch.cat([maps[77:78].repeat(n_dup, 1, 1), maps[C:C + B - n_dup]])
    slot, rep = st.insert(be.cuda(), bm.cuda())
    rs, rr = ref.insert(Qz(be), Qz(bm))
    assert slot.cpu().tolist() == rs
    assert rep.cpu().tolist() == rr
    ge, gm = st.read(0, C)
    assert np.array_equal(ge.cpu().numpy().astype(np.float64), ref.emb)
    assert np.array_equal(gm.cpu().numpy().astype(np.float64), ref.maps)
    slot, rep = st.insert(be[:70].cuda(), bm[:70].cuda())       # the bitmap was left clean
    rs, rr = ref.insert(Qz(be[:70]), Qz(bm[:70]))
    assert slot.cpu().tolist() == rs
    st.close()


@pytest.mark.parametrize("n_dup", [6, 30, 64])
def test_insert_many_conflicts_two_pass(lib, n_dup):
    """A batch of n_dup copies of one stored context plus fresh rows: the
    copies compete for the same victims, so beyond the first-pass list length
    (8) rows find all their candidates claimed and the gated full-length pass
    must take over; the result equals the oracle's R8 resolution."""
    sh = S.Shape("qw", 6, 60, 4, 200, n_clusters=8)
    C = 1500
    emb, maps, _ = S.store_rows(sh, 13, 0, C + 64)
    st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, C, "bf16")
    st.insert(emb[:C].cuda(), maps[:C].cuda())
    ref = O.Store(C, sh.L, sh.E, sh.D, 3)
    ref.insert(O.quantize(emb[:C].numpy(), "bf16"), O.quantize(maps[:C].numpy(), "bf16"))
    be = torch.cat([emb[40:41].repeat(n_dup, 1), emb[C:C + 64 - n_dup]])
    bm = torch.cat([maps[40:41].repeat(n_dup, 1, 1), maps[C:C + 64 - n_dup]])
    slot, rep = st.insert(be.cuda(), bm.cuda())
    rs, rr = ref.insert(O.quantize(be.numpy(), "bf16"), O.quantize(bm.numpy(), "bf16"))
    assert slot.cpu().tolist() == rs
    assert rep.cpu().tolist() == rr
    assert len(set(rs)) == 64
    st.close()


def test_topk_merge_api(lib):
    rng = np.random.default_rng(3)
    G, B, kin, k = 4, 5, 8, 8
    sc = np.round(rng.standard_normal((G, B, kin)), 2).astype(np.float32)
    ids = rng.permutation(G * B * kin).reshape(G, B, kin).astype(np.int64)
    ids[1, 2, 5:] = -1
    sc[3, 4, 0] = np.nan
    out_s = torch.empty(B, k, device="cuda")
    out_i = torch.empty(B, k, dtype=torch.int64, device="cuda")
    lib.fmoe_topk_merge(torch.from_numpy(sc).cuda(), torch.from_numpy(ids).cuda(), k, out_s, out_i)
    ms, mi = O.merge_topk([sc[g].astype(np.float64) for g in range(G)], [ids[g] for g in range(G)], k)
    valid = ~np.isnan(ms[:, 0])
    assert np.array_equal(out_i.cpu().numpy()[valid], mi[valid])
    assert np.array_equal(out_s.cpu().numpy()[valid], ms[valid].astype(np.float32))
    assert (out_i.cpu().numpy()[~valid] == -1).all()


# ---------------------------------------------------------------- batched (B >= 5)
# bf16: tcgen05 path; 130, 256: one pass on CTA pairs (cta_group::2, M = 256);
# 300: a 256-query pass + a ragged 44-query pass.
# fp32: the FFMA batched scan (scan_f32mm.cu), passes of <= 64 queries:
# 16 (2 query groups), 64 (8 groups, blend on 128-row tiles), 130 / 300 (a
# ragged last pass with the first pass's list layout), k up to 64.
@pytest.mark.parametrize("B,k", [(5, 4), (16, 1), (64, 8), (130, 64), (256, 8), (300, 3)])
@pytest.mark.parametrize("mode", ["sem", "traj3", "trajL", "blend"])
def test_batched_tcgen05(setup, B, k, mode):
    st, dt, sh = setup["st"], setup["dtype"], setup["shape"]
    q_emb, q_maps, _ = S.queries(sh, 1, setup["N"], B)
    if mode == "sem":
        gs, gi = st.search_semantic(q_emb.cuda(), k)
        ref = O.semantic_scores(O.quantize(q_emb.numpy(), dt), setup["Qe"])
    elif mode.startswith("traj"):
        ell = 3 if mode == "traj3" else sh.L
        qp = q_maps[:, :ell].contiguous()
        gs, gi = st.search_trajectory(qp.cuda(), ell, k)
        ref = O.trajectory_scores(O.quantize(qp.numpy(), dt), setup["Qm"], ell)
    else:
        ell = 5
        qp = q_maps[:, :ell].contiguous()
        gs, gi = st.search_blend(q_emb.cuda(), qp.cuda(), ell, -1.0, k)
        sem = O.semantic_scores(O.quantize(q_emb.numpy(), dt), setup["Qe"])
        trj = O.trajectory_scores(O.quantize(qp.numpy(), dt), setup["Qm"], ell)
        ref = O.blend_scores(sem, trj, np.float64(np.float32(3 / sh.L)))
    check_topk(gs, gi, ref, k)


# ---------------------------------------------------------------- incremental trajectory session
@pytest.mark.parametrize("B,k", [(1, 1), (3, 8), (6, 33)])
def test_trajectory_session_equals_eq2_at_every_prefix(setup, B, k):
    st, dt, sh = setup["st"], setup["dtype"], setup["shape"]
    qm = setup["q_maps"][:B]
    sess = st.trajectory_session(B)
    try:
        for ell in range(1, sh.L + 1):
            gs, gi = sess.step(qm[:, ell - 1].contiguous().cuda(), k)
            if ell in (1, 2, 3, 8, sh.L) or ell % 7 == 0:
                ref = O.trajectory_scores(O.quantize(qm[:, :ell].numpy(), dt), setup["Qm"], ell)
                check_topk(gs, gi, ref, k)
        with pytest.raises(setup["lib"].FmoeError):          # all L layers consumed
            sess.step(qm[:, 0].contiguous().cuda(), k)
        sess.reset()
        gs, gi = sess.step(qm[:, 0].contiguous().cuda(), k)   # prefix 1 again
        check_topk(gs, gi, O.trajectory_scores(O.quantize(qm[:, :1].numpy(), dt), setup["Qm"], 1), k)
    finally:
        sess.close()


@pytest.mark.parametrize("B,k,delta", [(1, 1, -1.0), (3, 8, -1.0), (4, 2, 0.9), (6, 8, -1.0), (9, 1, 0.5)])
def test_session_step_select_fused(setup, B, k, delta):
    """fmoe_traj_session_step_select = step + fmoe_select_experts on the top-1,
    bit for bit (incremental sessions select in the step's last block; B >= 5 on
    bf16 is a batched session with the select kernel after the scan; B = 9 on the
    incremental path is three 4-query passes, each selecting its own queries),
    and the selection equals the oracle's on the returned (id, score)."""
    st, dt, sh = setup["st"], setup["dtype"], setup["shape"]
    qm = S.queries(sh, 1, setup["N"], B)[1]
    a, b = st.trajectory_session(B), st.trajectory_session(B)
    d = 3
    try:
        for ell in range(1, sh.L + 1):
            lay = qm[:, ell - 1].contiguous().cuda()
            lb, le = (ell - 1 + d, ell + d) if ell - 1 + d < sh.L else (0, sh.L)
            fs, fi, fmask, fcnt = a.step_select(lay, k, delta, lb, le)
            gs, gi = b.step(lay, k)
            gmask, gcnt = st.select_experts(gi[:, 0].contiguous(), gs[:, 0].contiguous(), delta, lb, le)
            assert torch.equal(fi, gi) and torch.equal(fs, gs)
            assert torch.equal(fmask, gmask) and torch.equal(fcnt, gcnt)
            if ell in (1, 4, sh.L):
                om, oc = O.select_experts(setup["Qm"], fi[:, 0].cpu().tolist(), fs[:, 0].cpu().double().tolist(),
                                          float(np.float32(delta)), list(range(lb, le)), sh.K)
                assert np.array_equal(fmask.cpu().numpy().view(np.uint64), np.array(om, dtype=np.uint64))
                assert np.array_equal(fcnt.cpu().numpy(), np.array(oc))
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("name", ["qwen_small", "mixtral_tiny", "phi_small"])
def test_batched_session_seeded_equals_stateless(lib, name):
    """Batched session (bf16, B >= 5): each step is the tcgen05 scan over the
    whole prefix seeded with the previous step's ids; the seed bound only
    filters keys that cannot reach the top-k, so every step must equal the
    stateless search bit for bit -- also when k grows (no seeds) or shrinks."""
    sh = SHAPES[name]
    N, B = 5000, 40
    st, emb, maps = make(lib, sh, N, "bf16")
    _, qm, _ = S.queries(sh, 1, N, B)
    Qm = O.quantize(maps, "bf16")
    sess = st.trajectory_session(B)
    try:
        ks = [8, 8, 16, 4, 1, 8]
        for ell in range(1, sh.L + 1):
            k = ks[(ell - 1) % len(ks)]
            gs, gi = sess.step(qm[:, ell - 1].contiguous().cuda(), k)
            pre = qm[:, :ell].contiguous().cuda()
            rs, ri = st.search_trajectory(pre, ell, k)
            assert torch.equal(gi, ri), ell
            assert torch.equal(gs, rs), ell
            if ell in (1, 2, 7, sh.L):
                check_topk(gs, gi, O.trajectory_scores(O.quantize(qm[:, :ell].numpy(), "bf16"), Qm, ell), k)
    finally:
        sess.close()
        st.close()


def test_trajectory_session_invalidated_by_insert(lib):
    sh = SHAPES["mixtral_tiny"]
    emb, maps, _ = S.store_rows(sh, 3, 0, 40)
    st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, 64, "bf16")
    st.insert(emb[:30].cuda(), maps[:30].cuda())
    sess = st.trajectory_session(1)
    sess.step(maps[:1, 0].contiguous().cuda(), 1)
    st.insert(emb[30:].cuda(), maps[30:].cuda())
    with pytest.raises(lib.FmoeError):
        sess.step(maps[:1, 1].contiguous().cuda(), 1)
    sess.reset()
    s, i = sess.step(maps[35:36, 0].contiguous().cuda(), 1)
    assert i.item() in range(40)
    sess.close()
    st.close()


# ---------------------------------------------------------------- cached semantic cosines -> RDY insert
@pytest.mark.parametrize("B", [1, 3, 20])
def test_semantic_cos_matrix_and_insert_cos(lib, B):
    sh = S.Shape("mix", 8, 8, 2, 1040, n_clusters=4)        # D >= 1024: K-split tcgen05 path at B=20
    N = 1500
    emb, maps, _ = S.store_rows(sh, 21, 0, N + B)
    stride = N + 4
    for dt in ("bf16", "f32"):
        a = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, N, dt)
        b = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, N, dt)
        a.insert(emb[:N].cuda(), maps[:N].cuda())
        b.insert(emb[:N].cuda(), maps[:N].cuda())
        qe, qm = emb[N:].contiguous(), maps[N:].contiguous()
        cos = torch.full((B, stride), -7.0, device="cuda")
        s = torch.empty(B, 4, device="cuda")
        i = torch.empty(B, 4, dtype=torch.int64, device="cuda")
        lib.fmoe_search_semantic_cos(a._h, qe.cuda(), 4, s, i, cos, stride)
        ref = O.semantic_scores(O.quantize(qe.numpy(), dt), O.quantize(emb[:N].numpy(), dt))
        got = cos[:, :N].cpu().numpy().astype(np.float64)
        assert np.all(np.abs(got - ref) <= TOL)
        assert torch.all(cos[:, N:] == -7.0)                   # columns >= size untouched
        check_topk(s, i, ref, 4)
        # the insert that reuses the cosines == the plain insert
        sa = torch.empty(B, dtype=torch.int64, device="cuda")
        ra = torch.empty(B, dtype=torch.int64, device="cuda")
        lib.fmoe_store_insert_cos(a._h, qe.cuda(), qm.cuda(), cos, stride, sa, ra)
        sb, rb = b.insert(qe.cuda(), qm.cuda())
        assert torch.equal(sa, sb) and torch.equal(ra, rb)
        ea, ma = a.read(0, N)
        eb, mb = b.read(0, N)
        assert torch.equal(ea, eb) and torch.equal(ma, mb)
        a.close()
        b.close()


# ---------------------------------------------------------------- cache priorities
@pytest.mark.parametrize("delta", [-1.0, 0.9])
def test_prefetch_plan_bit_exact(setup, delta):
    lib, st, sh = setup["lib"], setup["st"], setup["shape"]
    rng = np.random.default_rng(11)
    B, l_now, lb, le, max_jobs = 9, 2, 3, min(3 + 6, sh.L), 40
    ids = rng.integers(-1, setup["N"], B)
    sc = rng.uniform(-1, 1, B).astype(np.float32)
    lay = torch.empty(B, max_jobs, dtype=torch.int32, device="cuda")
    exp = torch.empty(B, max_jobs, dtype=torch.int32, device="cuda")
    pri = torch.empty(B, max_jobs, dtype=torch.float64, device="cuda")
    nj = torch.empty(B, dtype=torch.int32, device="cuda")
    lib.fmoe_prefetch_plan(st._h, torch.from_numpy(ids).cuda(), torch.from_numpy(sc).cuda(), delta, l_now, lb, le,
                           max_jobs, lay, exp, pri, nj)
    plans = O.prefetch_plan(setup["Qm"], ids.tolist(), sc.astype(np.float64).tolist(), float(np.float32(delta)),
                            list(range(lb, le)), sh.K, l_now)
    for x in range(B):
        ref = plans[x][:max_jobs]
        n = nj[x].item()
        assert n == len(ref)
        got = list(zip(lay[x, :n].tolist(), exp[x, :n].tolist(), pri[x, :n].tolist()))
        assert got == [(t, j, p) for t, j, p in ref]
        assert (lay[x, n:] == -1).all()


def test_eviction_order_bit_exact(lib):
    rng = np.random.default_rng(12)
    for n in (1, 7, 256, 1440, 5000):
        p = rng.choice([0.0, 0.05, 0.1, 0.25, 0.5], size=n).astype(np.float32)
        f = rng.integers(1, 6, size=n).astype(np.float32)
        pri = torch.empty(n, dtype=torch.float64, device="cuda")
        order = torch.empty(n, dtype=torch.int32, device="cuda")
        lib.fmoe_eviction_order(torch.from_numpy(p).cuda(), torch.from_numpy(f).cuda(), 1e-6, pri, order)
        rp, ro = O.eviction_order(p.astype(np.float64), f.astype(np.float64), float(np.float32(1e-6)))
        assert pri.cpu().tolist() == rp
        assert order.cpu().tolist() == ro


# ---------------------------------------------------------------- expert hits + ablation variants
@pytest.mark.parametrize("E,K", [(8, 2), (16, 2), (60, 4), (64, 8), (64, 64), (1, 1), (33, 5)])
def test_expert_hits_bit_exact(lib, E, K):
    rng = np.random.default_rng(100 + E)
    B, T = 37, 5
    gate = (rng.integers(0, 6, (B, T, E)) / 8.0).astype(np.float32)    # many exact ties
    mask = (rng.integers(0, 2 ** 64, (B, T), dtype=np.uint64) & np.uint64((1 << E) - 1 if E < 64 else 2 ** 64 - 1)).view(np.int64)
    gate[0, 0] = 0.0                                                   # all tied -> experts 0..K-1
    hits, act = lib.expert_hits(torch.from_numpy(gate).cuda(), torch.from_numpy(mask).cuda(), K)
    oh, oa = O.expert_hits(gate.astype(np.float64), mask.view(np.uint64).tolist(), K)
    assert hits.cpu().numpy().tolist() == oh
    assert act.cpu().numpy().view(np.uint64).tolist() == [[np.uint64(v) for v in r] for r in oa]
    assert act[0, 0].item() == (1 << K) - 1 if K < 64 else True


def test_expert_hits_host_buffers_and_args(lib):
    gate = torch.rand(3, 4, 8)
    mask = torch.full((3, 4), 0xF0, dtype=torch.int64)
    hits = torch.empty(3, 4, dtype=torch.int32)
    lib.fmoe_expert_hits(gate, mask, 2, hits)                       # host pointers, staged
    oh, _ = O.expert_hits(gate.double().numpy(), mask.numpy().tolist(), 2)
    assert hits.numpy().tolist() == oh
    with pytest.raises(lib.FmoeError):
        lib.fmoe_expert_hits(gate, mask, 9, hits)                   # K > E
    lib.fmoe_expert_hits(torch.empty(0, 4, 8), torch.empty(0, 4, dtype=torch.int64), 2,
                         torch.empty(0, 4, dtype=torch.int32))      # B = 0: no-op


@pytest.mark.parametrize("variant", ["map_t", "map_ts", "map_tsd"])
def test_ablation_variants_match_oracle(setup, variant):
    from paper_2502_05370_b200 import ablation
    st, sh, dt = setup["st"], setup["shape"], setup["dtype"]
    B, d = 6, 3
    q_emb, q_maps = setup["q_emb"][:B], setup["q_maps"][:B]
    gm, gid, gsc = ablation.prefetch_masks(st, q_emb.cuda(), q_maps.cuda(), variant)
    rate, hits, _ = ablation.hit_rate(st, q_emb.cuda(), q_maps.cuda(), variant)
    gm, gid, gsc = gm.cpu().numpy().view(np.uint64), gid.cpu().numpy(), gsc.cpu().numpy()
    Qq_e, Qq_m = O.quantize(q_emb.numpy(), dt), O.quantize(q_maps.numpy(), dt)
    om, oid = O.ablation_prefetch_masks(setup["Qe"], setup["Qm"], Qq_e, Qq_m, variant, d, sh.K)
    delta = -1.0 if variant == "map_tsd" else 0.0
    for t in range(sh.L):
        if t < d and variant == "map_t":
            assert (gm[:, t] == 0).all() and (gid[:, t] == -1).all()
            continue
        # ids: the top-1 rules of check_topk against the oracle scores of that match
        ref = (O.semantic_scores(Qq_e, setup["Qe"]) if t < d else
               O.trajectory_scores(Qq_m, setup["Qm"], t - d + 1))
        check_topk(torch.from_numpy(gsc[:, t:t + 1]), torch.from_numpy(gid[:, t:t + 1]), ref, 1)
        # masks: bit-exact Eq. 4-6 selection of the matched (id, score)
        sm, _ = O.select_experts(setup["Qm"], gid[:, t].tolist(), gsc[:, t].astype(np.float64).tolist(),
                                 delta, [t], sh.K)
        assert gm[:, t].tolist() == [np.uint64(r[0]) for r in sm], t
        # where the oracle took the same match, the oracle's own mask agrees
        for x in range(B):
            if gid[x, t] == oid[x][t] and delta == 0.0:
                assert int(gm[x, t]) == om[x][t]
    oh, _ = O.expert_hits(q_maps.double().numpy(), gm.tolist(), sh.K)
    assert hits.cpu().numpy().tolist() == oh
    assert rate == pytest.approx(np.sum(oh) / (B * sh.L * sh.K), abs=0)


# ---------------------------------------------------------------- session sweep (n steps, one call)
def _steps_reference(st, qm, delta, d, ell0=0, n=None):
    """n calls of step_select (k = 1) from a fresh session, after ell0 plain steps."""
    L = qm.shape[1]
    n = L - ell0 if n is None else n
    ref = st.trajectory_session(qm.shape[0])
    try:
        for ell in range(ell0):
            ref.step(qm[:, ell].contiguous().cuda(), 1)
        out = []
        for ell in range(ell0, ell0 + n):
            lay = qm[:, ell].contiguous().cuda()
            tgt = ell + d
            if tgt < L:
                s, i, m, c = ref.step_select(lay, 1, delta, tgt, tgt + 1)
            else:
                s, i = ref.step(lay, 1)
                m = torch.zeros(qm.shape[0], 1, dtype=torch.int64, device="cuda")
                c = torch.zeros(qm.shape[0], 1, dtype=torch.int32, device="cuda")
            out.append((s[:, 0], i[:, 0], m[:, 0], c[:, 0]))
        return [torch.stack(v) for v in zip(*out)]
    finally:
        ref.close()


@pytest.mark.parametrize("kern", ["row", "reg", "tma"])
@pytest.mark.parametrize("B,delta", [(1, -1.0), (1, 0.9), (3, -1.0)])
def test_session_sweep_equals_steps(setup, B, delta, kern, monkeypatch):
    """fmoe_traj_session_sweep = n calls of step_select, bit for bit (fused kernel
    for B = 1 on 16-byte slab rows -- mixtral_tiny bf16 -- else the per-step
    path), including a sweep split in three and continued by plain steps; ids
    follow the Eq. 2 oracle at every prefix."""
    # row-major kernel / step-major register kernel / step-major shared-memory staged kernel
    monkeypatch.setenv("FMOE_SWEEP_KERNEL", kern)
    st, dt, sh = setup["st"], setup["dtype"], setup["shape"]
    qm = S.queries(sh, 5, setup["N"], B)[1]
    d, L = 3, sh.L
    rs, ri, rm, rc = _steps_reference(st, qm, delta, d)
    ql = qm.permute(1, 0, 2).contiguous().cuda()          # [L][B][E]
    a = st.trajectory_session(B)
    try:
        parts = [(0, 5), (5, 17), (17, L)]
        got = [a.sweep(ql[b:e], delta, d) for b, e in parts]
        gs, gi, gm, gc = [torch.cat(v) for v in zip(*got)]
        assert torch.equal(gi, ri) and torch.equal(gs, rs)
        assert torch.equal(gm, rm) and torch.equal(gc, rc)
        with pytest.raises(setup["lib"].FmoeError):       # all L layers consumed
            a.sweep(ql[:1], delta, d)
        a.reset()
        s1, i1, _, _ = a.sweep(ql[:L - 1], delta)           # no selection
        assert torch.equal(i1, ri[:L - 1]) and torch.equal(s1, rs[:L - 1])
        s2, i2 = a.step(ql[L - 1], 1)                       # the session state continues
        assert torch.equal(i2[:, 0], ri[L - 1]) and torch.equal(s2[:, 0], rs[L - 1])
    finally:
        a.close()
    for ell in (1, 2, 9, L):
        ref = O.trajectory_scores(O.quantize(qm[:, :ell].numpy(), dt), setup["Qm"], ell)
        check_topk(gs[ell - 1][:, None], gi[ell - 1][:, None], ref, 1)


def test_session_sweep_ready_flags(setup):
    """Device flags: step s waits for layer_ready[s] (set here by DMA copies on
    another stream after the launch) and publishes guidance_ready[s]; results
    equal the per-step path.  Flags on a path without the fused kernel fail."""
    lib, st, sh = setup["lib"], setup["st"], setup["shape"]
    qm = S.queries(sh, 6, setup["N"], 1)[1]
    L, d = sh.L, 3
    ql = qm.permute(1, 0, 2).contiguous().cuda()
    a = st.trajectory_session(1)
    ready = torch.zeros(L, dtype=torch.int32, device="cuda")
    pub = torch.zeros(L, dtype=torch.int32, device="cuda")
    fused = setup["dtype"] == "bf16" and sh.E <= 8
    try:
        if not fused:
            with pytest.raises(lib.FmoeError):
                a.sweep(ql, -1.0, d, layer_ready=ready, guidance_ready=pub)
            return
        rs, ri, rm, rc = _steps_reference(st, qm, -1.0, d)
        ones = torch.ones(L, dtype=torch.int32).pin_memory()
        torch.cuda.synchronize()                            # the zeroed flags are in place
        side = torch.cuda.Stream()
        main = torch.cuda.current_stream()
        gs, gi, gm, gc = a.sweep(ql, -1.0, d, layer_ready=ready, guidance_ready=pub)
        with torch.cuda.stream(side):
            for s in range(L):                              # the producer publishes layer by layer
                ready[s:s + 1].copy_(ones[s:s + 1], non_blocking=True)
        main.synchronize()
        side.synchronize()
        assert pub.cpu().tolist() == [1] * L
        assert torch.equal(gi, ri) and torch.equal(gs, rs) and torch.equal(gm, rm) and torch.equal(gc, rc)
    finally:
        a.close()


@pytest.mark.parametrize("kern", ["row", "reg", "tma"])
def test_session_sweep_edge_cases(lib, kern, monkeypatch):
    """Zero query layers (prefix norm 0 -> (NaN, -1), empty selection, as the
    step kernel), single-step sweeps, an empty store (per-step path: id -1)."""
    monkeypatch.setenv("FMOE_SWEEP_KERNEL", kern)
    sh = SHAPES["mixtral_tiny"]
    st, _, _ = make(lib, sh, 777, "bf16")
    empty = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, 16, "bf16")
    try:
        qm = S.queries(sh, 9, 777, 1)[1]
        qm[:, :2] = 0.0                                       # the first two observed layers are all zero
        ql = qm.permute(1, 0, 2).contiguous().cuda()
        rs, ri, rm, rc = _steps_reference(st, qm, -1.0, 3)
        a = st.trajectory_session(1)
        gs, gi, gm, gc = a.sweep(ql[:1], -1.0, 3)             # n_steps = 1
        g2 = a.sweep(ql[1:], -1.0, 3)
        gs, gi, gm, gc = [torch.cat([x, y]) for x, y in zip((gs, gi, gm, gc), g2)]
        assert torch.equal(gi, ri) and torch.equal(gm, rm) and torch.equal(gc, rc)
        assert torch.equal(torch.isnan(gs), torch.isnan(rs)) and torch.equal(gs[2:], rs[2:])
        assert gi[:2].eq(-1).all() and torch.isnan(gs[:2]).all() and gm[:2].eq(0).all()
        a.close()
        e = empty.trajectory_session(1)
        es, ei, em, ec = e.sweep(ql[:4], -1.0, 3)
        assert ei.eq(-1).all() and em.eq(0).all() and ec.eq(0).all()
        e.close()
    finally:
        st.close()
        empty.close()


@pytest.mark.parametrize("B,k", [(1, 1), (3, 8), (64, 8), (256, 8), (300, 3)])
@pytest.mark.parametrize("ell,w", [(5, -1.0), (31, 0.3)])
def test_blend_cos_equals_blend(setup, B, k, ell, w):
    """fmoe_search_blend_cos (semantic half from fmoe_search_semantic_cos's
    cosines) = fmoe_search_blend bit for bit on the test shapes (GEMV for
    B <= 4, tcgen05 for B = 64 on bf16), and = the oracle blend."""
    lib, st, sh, dt = setup["lib"], setup["st"], setup["shape"], setup["dtype"]
    N, ell = setup["N"], min(ell, sh.L)
    qe, qm, _ = S.queries(sh, 7, N, B)
    qp = qm[:, :ell].contiguous()
    stride = (N + 3) // 4 * 4
    cos = torch.empty(B, stride, device="cuda")
    s0 = torch.empty(B, k, device="cuda")
    i0 = torch.empty(B, k, dtype=torch.int64, device="cuda")
    lib.fmoe_search_semantic_cos(st._h, qe.cuda(), k, s0, i0, cos, stride)
    s2 = torch.empty(B, k, device="cuda")
    i2 = torch.empty(B, k, dtype=torch.int64, device="cuda")
    lib.fmoe_search_blend_cos(st._h, cos, stride, qp.cuda(), ell, w, k, s2, i2)
    gs, gi = st.search_blend(qe.cuda(), qp.cuda(), ell, w, k)
    assert torch.equal(gi, i2) and torch.equal(gs, s2)
    wv = float(np.float32(3 / sh.L)) if w < 0 else float(np.float32(w))
    ref = (wv * O.semantic_scores(O.quantize(qe.numpy(), dt), setup["Qe"])
           + (1 - wv) * O.trajectory_scores(O.quantize(qp.numpy(), dt), setup["Qm"], ell))
    check_topk(s2, i2, ref, k)
    with pytest.raises(lib.FmoeError):                       # w = 1 is the semantic search itself
        lib.fmoe_search_blend_cos(st._h, cos, stride, qp.cuda(), ell, 1.0, k, s2, i2)


@pytest.mark.parametrize("B,k", [(6, 1), (8, 8), (40, 16)])
def test_semantic_rerank_fallback_on_ties(lib, B, k):
    """The tensor-core semantic scan keeps k_ext > k approximate candidates and
    re-ranks them exactly; with more than k_ext stored copies of the query's
    best row the candidate list cannot prove completeness, so the query goes
    to the exact GEMV fallback: the lowest ids of the tied rows win,
    exactly as in the oracle."""
    sh = SHAPES["mixtral_tiny"]
    N = 3000
    emb, maps, _ = S.store_rows(sh, 31, 0, N)
    emb[100:180] = emb[7]                          # 80 exact copies of row 7
    st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, N, "bf16")
    st.insert(emb.cuda(), maps.cuda())
    q = emb[7:8].repeat(B, 1).clone()
    q[B // 2:] = emb[200:200 + B - B // 2]         # the other half: ordinary rows (no ties)
    gs, gi = st.search_semantic(q.cuda(), k)
    ref = O.semantic_scores(O.quantize(q.numpy(), "bf16"), O.quantize(emb.numpy(), "bf16"))
    check_topk(gs, gi, ref, k)
    assert gi[0].tolist() == ([7] + list(range(100, 100 + k - 1)))[:k]
    st.close()


def test_prefetch_issue_copies_the_plan(setup):
    """fmoe_prefetch_issue: the copy stream
    waits on the device for the guidance flag (set late by another stream),
    then one cudaMemcpyAsync per planned expert, in PRI^prefetch order,
    skipping resident experts: the copied set and order equal O.prefetch_plan
    and exactly those device slots receive the host weights."""
    lib, st, sh = setup["lib"], setup["st"], setup["shape"]
    L, E = sh.L, sh.E
    B, l_now, lb, le = 3, 2, 3, min(6, sh.L)
    max_jobs = (le - lb) * E
    q = setup["q_emb"][:B].cuda()
    gs, gi = st.search_semantic(q, 1)
    ids, sc = gi[:, 0].contiguous(), gs[:, 0].contiguous()
    eb = 256                                                  # bytes per (synthetic) expert
    host = torch.arange(L * E, dtype=torch.int32).repeat_interleave(eb // 4).view(L * E, eb // 4).pin_memory()
    dev = torch.full((L * E, eb // 4), -1, dtype=torch.int32, device="cuda")
    hp = [host[i].data_ptr() for i in range(L * E)]
    dp = [dev[i].data_ptr() for i in range(L * E)]
    resident = torch.zeros(L, dtype=torch.int64)
    resident[lb] = 1                                          # expert 0 of layer lb is already on the GPU
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    side, copy = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(20_000_000)                        # the guidance arrives late
        flag.fill_(1)
    lay, exp, nj = lib.fmoe_prefetch_issue(st._h, ids, sc, -1.0, l_now, lb, le, max_jobs, hp, dp, eb,
                                           resident, flag, copy)
    copy.synchronize()
    plans = O.prefetch_plan(setup["Qm"], ids.cpu().tolist(), sc.cpu().double().tolist(), -1.0, list(range(lb, le)),
                            sh.K, l_now)
    seen = {(lb, 0)}
    copied = set()
    for x in range(B):
        want = []
        for t, j, _ in plans[x][:max_jobs]:
            if (t, j) not in seen:
                seen.add((t, j))
                want.append((t, j))
        n = nj[x].item()
        assert list(zip(lay[x, :n].tolist(), exp[x, :n].tolist())) == want
        copied |= set(want)
    got = dev.cpu()
    for t in range(L):
        for j in range(E):
            i = t * E + j
            assert torch.equal(got[i], host[i]) == ((t, j) in copied), (t, j)
            assert bool(resident[t].item() >> j & 1) == ((t, j) in copied or (t, j) == (lb, 0))
