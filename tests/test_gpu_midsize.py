"""Element-wise oracle parity at sizes where every kernel runs its steady-state
code (VERDICT r1 "What's weak" #1): N ~ 0.5M rows with small D, so that

  * the GEMV scan (B <= 4 per pass) runs its round-robin ``full_rounds`` loop
    (grid rows per round < N) before the balanced remainder;
  * every tcgen05 CTA / CTA pair processes >= 3 tiles of 256 rows: both TMEM
    accumulator stages, the tfull/tempty phase flips across tiles, heaps that
    persist across tiles and the shared per-query admission threshold;
  * the session sweep keeps several rows per thread.

Every check is against a FULL oracle scan (O-store view: the rows the store
holds, read back through fmoe_store_read) with the rules of
DESIGN.md "Parity contract": scores within 1e-5, ids exact at every rank whose
oracle score is separated from its neighbours by more than 1e-5, elsewhere the
returned id's oracle score within 1e-5 of the rank's.
"""
import numpy as np
import pytest
import torch

import fmoe_synth as S
from oracle import fmoe_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-5
N_MID = 524_309            # ragged: not a multiple of 32, 256 or a grid round

SHAPES = {
    "mixtral": S.Shape("mixtral-mid", 32, 8, 2, 64, n_clusters=64),
    "qwen": S.Shape("qwen-mid", 24, 60, 4, 256, n_clusters=64),
    "phi": S.Shape("phi-mid", 32, 16, 2, 200, n_clusters=64),      # D not a multiple of 64
}


def check_topk_fast(gs, gi, ref, k, tol=TOL):
    """check_topk of test_gpu_parity with argpartition instead of full sorts."""
    gs = gs.cpu().numpy().astype(np.float64)
    gi = gi.cpu().numpy()
    B, N = ref.shape
    for x in range(B):
        row = ref[x]
        if np.isnan(row).any():
            assert np.isnan(gs[x]).all() and (gi[x] == -1).all()
            continue
        m = min(N, k + 1)
        part = np.argpartition(-row, m - 1)[:m] if m < N else np.arange(N)
        top = part[np.lexsort((part, -row[part]))]          # score desc, id asc
        nv = min(k, N)
        assert (gi[x, nv:] == -1).all() and np.isneginf(gs[x, nv:]).all()
        ids = gi[x, :nv]
        assert len(set(ids.tolist())) == nv and (ids >= 0).all()
        rs = row[top[:nv]]
        assert np.all(np.abs(gs[x, :nv] - rs) <= tol), (x, gs[x, :nv], rs)
        full = row[top]
        for r in range(nv):
            lo = full[r - 1] - full[r] if r > 0 else np.inf
            hi = full[r] - full[r + 1] if r + 1 < full.shape[0] else np.inf
            if min(lo, hi) > tol:
                assert gi[x, r] == top[r], (x, r, gi[x], top[:nv])
            else:
                assert abs(row[gi[x, r]] - rs[r]) <= tol


def read_store(st, n, D, L, E):
    """The O-store view: the values the device holds (fp32 read-back of the tiles)."""
    # fp32 holds the stored values exactly (bf16 or fp32 tiles); the oracle
    # converts to float64 itself
    e = np.empty((n, D), np.float32)
    m = np.empty((n, L, E), np.float32)
    for a in range(0, n, 65536):
        c = min(65536, n - a)
        ge, gm = st.read(a, c)
        e[a:a + c] = ge.cpu().numpy()
        m[a:a + c] = gm.cpu().numpy()
    return e, m


@pytest.fixture(scope="module", params=[("mixtral", "bf16"), ("qwen", "bf16"), ("phi", "bf16"), ("mixtral", "f32"),
                                        ("qwen", "f32")])
def mid(request, lib):
    name, dtype = request.param
    sh = SHAPES[name]
    st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, N_MID, dtype)
    for a in range(0, N_MID, 65536):
        e, m, _ = S.store_rows(sh, 77, a, min(65536, N_MID - a), device="cuda")
        st.insert(e, m)
    torch.cuda.synchronize()
    Qe, Qm = read_store(st, N_MID, sh.D, sh.L, sh.E)
    yield dict(lib=lib, st=st, sh=sh, dt=dtype, Qe=Qe, Qm=Qm)
    st.close()


def _q(mid, B, seed=5):
    qe, qm, planted = S.queries(mid["sh"], seed, N_MID, B)
    return qe, qm, planted


def _batches(dt):
    # (B, k): GEMV passes (B <= 4, also every f32 batch) and the tcgen05 path
    # (bf16, B >= 5: single CTAs up to 128 queries, CTA pairs above)
    return [(1, 1), (4, 8), (5, 8), (64, 8), (130, 64), (256, 8)] if dt == "bf16" else [(1, 1), (4, 8), (9, 64)]


def test_semantic_midsize(mid):
    st, dt, sh = mid["st"], mid["dt"], mid["sh"]
    for B, k in _batches(dt):
        qe, _, _ = _q(mid, B)
        gs, gi = st.search_semantic(qe.cuda(), k)
        ref = O.semantic_scores(O.quantize(qe.numpy(), dt), mid["Qe"])
        check_topk_fast(gs, gi, ref, k)


@pytest.mark.parametrize("ell", [1, 3, "L"])
def test_trajectory_midsize(mid, ell):
    st, dt, sh = mid["st"], mid["dt"], mid["sh"]
    ell = sh.L if ell == "L" else ell
    for B, k in _batches(dt):
        _, qm, _ = _q(mid, B, seed=6)
        qp = qm[:, :ell].contiguous()
        gs, gi = st.search_trajectory(qp.cuda(), ell, k)
        ref = O.trajectory_scores(O.quantize(qp.numpy(), dt), mid["Qm"][:, :ell], ell)
        check_topk_fast(gs, gi, ref, k)


@pytest.mark.parametrize("ell", [5, 31])
def test_blend_and_blend_cos_midsize(mid, ell):
    """fmoe_search_blend and fmoe_search_blend_cos (semantic half from
    fmoe_search_semantic_cos) against the oracle blend; the cosine
    side output against Eq. 1 element by element."""
    lib, st, dt, sh = mid["lib"], mid["st"], mid["dt"], mid["sh"]
    ell = min(ell, sh.L)
    stride = (N_MID + 3) // 4 * 4
    w = float(np.float32(3 / sh.L))
    for B, k in _batches(dt):
        qe, qm, _ = _q(mid, B, seed=7)
        qp = qm[:, :ell].contiguous()
        sem = O.semantic_scores(O.quantize(qe.numpy(), dt), mid["Qe"])
        trj = O.trajectory_scores(O.quantize(qp.numpy(), dt), mid["Qm"][:, :ell], ell)
        ref = w * sem + (1 - w) * trj
        gs, gi = st.search_blend(qe.cuda(), qp.cuda(), ell, -1.0, k)
        check_topk_fast(gs, gi, ref, k)
        cos = torch.empty(B, stride, device="cuda")
        s0 = torch.empty(B, k, device="cuda")
        i0 = torch.empty(B, k, dtype=torch.int64, device="cuda")
        lib.fmoe_search_semantic_cos(st._h, qe.cuda(), k, s0, i0, cos, stride)
        check_topk_fast(s0, i0, sem, k)
        got = cos[:, :N_MID].cpu().numpy().astype(np.float64)
        assert np.max(np.abs(got - sem)) <= 2e-5
        s2 = torch.empty(B, k, device="cuda")
        i2 = torch.empty(B, k, dtype=torch.int64, device="cuda")
        lib.fmoe_search_blend_cos(st._h, cos, stride, qp.cuda(), ell, -1.0, k, s2, i2)
        check_topk_fast(s2, i2, ref, k)
        del cos


@pytest.mark.parametrize("B", [1, 3, 64])
def test_trajectory_session_midsize(mid, B):
    """Incremental (B <= 4 or f32) and batched (bf16, B >= 5: seeded tcgen05
    scans over the prefix) sessions: Eq. 2 at prefixes 1, 2, 9 and L."""
    st, dt, sh = mid["st"], mid["dt"], mid["sh"]
    if B > 4 and dt != "bf16":
        pytest.skip("incremental session is <= 64 queries; covered by B = 3")
    _, qm, _ = _q(mid, B, seed=8)
    k = 1 if B == 1 else 8
    sess = st.trajectory_session(B)
    try:
        for ell in range(1, sh.L + 1):
            gs, gi = sess.step(qm[:, ell - 1].contiguous().cuda(), k)
            if ell in (1, 2, 9, sh.L):
                ref = O.trajectory_scores(O.quantize(qm[:, :ell].numpy(), dt), mid["Qm"][:, :ell], ell)
                check_topk_fast(gs, gi, ref, k)
    finally:
        sess.close()


def test_session_sweep_midsize(mid):
    """The one-launch sweep (B = 1, 16-byte slab rows: Mixtral bf16, several
    rows per thread at this N): top-1 of every prefix against Eq. 2 and the
    Eq. 4-6 selection of target layer ell + d against the oracle."""
    st, dt, sh = mid["st"], mid["dt"], mid["sh"]
    if not (dt == "bf16" and sh.E <= 8):
        pytest.skip("the fused sweep needs 16-byte slab rows")
    _, qm, _ = _q(mid, 1, seed=9)
    ql = qm.permute(1, 0, 2).contiguous().cuda()
    sess = st.trajectory_session(1)
    try:
        gs, gi, gm, gc = sess.sweep(ql[:sh.L - 1], -1.0, 3)
    finally:
        sess.close()
    for ell in range(1, sh.L):
        ref = O.trajectory_scores(O.quantize(qm[:, :ell].numpy(), dt), mid["Qm"][:, :ell], ell)
        check_topk_fast(gs[ell - 1][:, None], gi[ell - 1][:, None], ref, 1)
        tgt = ell - 1 + 3
        if tgt < sh.L:
            om, oc = O.select_experts(mid["Qm"], [int(gi[ell - 1, 0])], [float(gs[ell - 1, 0])], -1.0, [tgt], sh.K)
            assert int(gm[ell - 1, 0].cpu().numpy().view(np.uint64)) == int(om[0][0])
            assert int(gc[ell - 1, 0]) == oc[0][0]


@pytest.mark.parametrize("B", [64, 256])
@pytest.mark.parametrize("name,dt", [("qwen", "bf16"), ("mixtral", "bf16"), ("mixtral", "f32")])
def test_rdy_insert_midsize(lib, name, dt, B):
    """Insert at full capacity (Reading R8) with many conflicting rows
    (copies of one stored context) next to fresh ones, plain and with the
    cached semantic cosines: slots equal O.Store.insert."""
    sh = SHAPES[name]
    C = 160_013
    st = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, C, dt)
    st2 = lib.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, C, dt)
    for a in range(0, C, 65536):
        e, m, _ = S.store_rows(sh, 78, a, min(65536, C - a), device="cuda")
        st.insert(e, m)
        st2.insert(e, m)
    Qe, Qm = read_store(st, C, sh.D, sh.L, sh.E)
    ref = O.Store(C, sh.L, sh.E, sh.D, 3)
    ref.insert(Qe, Qm)
    fe, fm_, _ = S.store_rows(sh, 79, 0, B)
    n_dup = 24 if B <= 64 else 90
    be = torch.cat([torch.from_numpy(Qe[4321:4322]).float().repeat(n_dup, 1), fe[:B - n_dup]])
    bm = torch.cat([torch.from_numpy(Qm[4321:4322]).float().repeat(n_dup, 1, 1), fm_[:B - n_dup]])
    slot, rep = st.insert(be.cuda(), bm.cuda())
    stride = (C + 3) // 4 * 4
    cos = torch.empty(B, stride, device="cuda")
    s0 = torch.empty(B, 8, device="cuda")
    i0 = torch.empty(B, 8, dtype=torch.int64, device="cuda")
    lib.fmoe_search_semantic_cos(st2._h, be.cuda(), 8, s0, i0, cos, stride)
    slot2 = torch.empty(B, dtype=torch.int64, device="cuda")
    rep2 = torch.empty(B, dtype=torch.int64, device="cuda")
    lib.fmoe_store_insert_cos(st2._h, be.cuda(), bm.cuda(), cos, stride, slot2, rep2)
    rs, rr = ref.insert(O.quantize(be.numpy(), dt), O.quantize(bm.numpy(), dt))
    assert slot.cpu().tolist() == rs and rep.cpu().tolist() == rr
    assert slot2.cpu().tolist() == rs and rep2.cpu().tolist() == rr
    assert slot[0].item() == 4321                            # the exact duplicate is the first victim
    st.close()
    st2.close()
