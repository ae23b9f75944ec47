"""Full-size parity for C4 (Phi-3.5-MoE shape, N = 4M) and C5 (Mixtral shape,
N = 16M, B = 256) -- separate module so the C2/C3 stores are freed first."""
from test_gpu_fullsize import SEED, TOL, build, check_block_not_better, check_returned_scores, rows_for  # noqa: F401
import numpy as np
import pytest
import torch

import fmoe_synth as S

pytestmark = pytest.mark.gpu


@pytest.mark.slow
def test_c4_phi_blend_and_insert(lib):
    sh, N = S.PHI, 4_000_000
    st = build(lib, sh, N)
    try:
        qe, qm, planted = S.queries(sh, SEED, N, 64, device="cuda")
        for ell, B in ((16, 64), (31, 64), (31, 1)):
            pre = qm[:B, :ell].contiguous()
            s, i = st.search_blend(qe[:B], pre, ell, -1.0, 8)
            w = float(np.float32(3 / sh.L))
            check_returned_scores(sh, s, i, qe[:B], pre, ell, w)
            check_block_not_better(sh, N, s[:, 0], qe[:B], pre, ell, w, block=100)
            pl = planted[:B].cpu().numpy()
            assert np.all(i[:, 0].cpu().numpy()[pl >= 0] == pl[pl >= 0])
        victims = list(range(7, 7 + 64 * 61_001, 61_001))
        e, m = rows_for(sh, victims)
        slot, rep = st.insert(torch.from_numpy(e).cuda(), torch.from_numpy(m).cuda())
        assert slot.cpu().tolist() == victims
    finally:
        st.close()


@pytest.mark.slow
def test_c5_sixteen_million_batch_256(lib):
    sh, N = S.MIXTRAL, 16_000_000
    st = build(lib, sh, N)
    try:
        qe, qm, planted = S.queries(sh, SEED, N, 256, device="cuda")
        s, i = st.search_semantic(qe, 8)
        check_returned_scores(sh, s[:32], i[:32], qe[:32], None, 0, 1.0)
        pl = planted.cpu().numpy()
        assert np.all(i[:, 0].cpu().numpy()[pl >= 0] == pl[pl >= 0])
        ell = 31
        pre = qm[:, :ell].contiguous()
        s, i = st.search_blend(qe, pre, ell, -1.0, 8)
        w = float(np.float32(3 / sh.L))
        check_returned_scores(sh, s[:32], i[:32], qe[:32], pre[:32], ell, w)
        check_block_not_better(sh, N, s[:32, 0], qe[:32], pre[:32], ell, w, block=500)
        # queries 128..255 live in the second CTA of each pair (cta_group::2)
        check_returned_scores(sh, s[224:], i[224:], qe[224:], pre[224:], ell, w)
        check_block_not_better(sh, N, s[224:, 0], qe[224:], pre[224:], ell, w, block=500)
        # trajectory only (16-byte map rows: bulk-copy operands)
        s, i = st.search_trajectory(pre, ell, 8)
        check_returned_scores(sh, s[:16], i[:16], qe[:16], pre[:16], ell, 0.0)
        check_returned_scores(sh, s[240:], i[240:], qe[240:], pre[240:], ell, 0.0)
        assert np.all(i[:, 0].cpu().numpy()[pl >= 0] == pl[pl >= 0])
    finally:
        st.close()
