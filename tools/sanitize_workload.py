"""A small workload touching every kernel once, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck  python tools/sanitize_workload.py
    compute-sanitizer --tool racecheck python tools/sanitize_workload.py
    compute-sanitizer --tool synccheck python tools/sanitize_workload.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmoe_synth as S  # noqa: E402
import paper_2502_05370_b200 as fm  # noqa: E402


def main():
    for sh, dt in ((S.Shape("m", 8, 8, 2, 72, 4), "bf16"), (S.Shape("q", 6, 60, 4, 136, 4), "bf16"),
                   (S.Shape("p", 8, 16, 2, 64, 4), "f32")):
        N = 2100
        e, m, _ = S.store_rows(sh, 3, 0, N + 20, device="cuda")
        st = fm.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, N, dt)
        st.insert(e[:N].contiguous(), m[:N].contiguous())
        qe, qm, _ = S.queries(sh, 3, N, 260, device="cuda")
        # (150, 8), (260, 3): CTA-pair passes (cta_group::2), the second one ragged
        for B, k in ((1, 1), (3, 8), (6, 40), (20, 8), (150, 8), (260, 3)):
            st.search_semantic(qe[:B].contiguous(), k)
            st.search_trajectory(qm[:B].contiguous(), 3, k)
            st.search_blend(qe[:B].contiguous(), qm[:B].contiguous(), sh.L, -1.0, k)
        s, i = st.search_semantic(qe[:4].contiguous(), 1)
        st.select_experts(i[:, 0].contiguous(), s[:, 0].contiguous(), -1.0, 0, sh.L)
        for Bs in (2, 6):                   # incremental and (bf16) batched sessions
            sess = st.trajectory_session(Bs)
            for ell in range(sh.L):
                sess.step(qm[:Bs, ell].contiguous(), 4)
            sess.close()
        st.insert(e[N:].contiguous(), m[N:].contiguous())        # replacement path
        st.read(0, 10)
        torch.cuda.synchronize()
        st.close()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
