"""Small fp32 batched-scan check (B = 6, k = 40 and B = 64, k = 8) against the
oracle semantic scores; used under compute-sanitizer."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmoe_synth as S  # noqa: E402
import paper_2502_05370_b200 as fm  # noqa: E402
from oracle import fmoe_oracle as O  # noqa: E402

sh = S.Shape("t", 32, 8, 2, 64, n_clusters=16)
N = 3001
emb, maps, _ = S.store_rows(sh, 1, 0, N)
st = fm.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, N, "f32")
st.insert(emb.cuda(), maps.cuda())
for B, k in ((6, 40), (64, 8), (70, 3)):
    qe, qm, _ = S.queries(sh, 1, N, B)
    gs, gi = st.search_semantic(qe.cuda(), k)
    ref = O.semantic_scores(qe.numpy(), emb.numpy())
    rs, ri = O.topk(ref, k)
    err = np.abs(gs.cpu().numpy() - rs).max()
    same = (gi.cpu().numpy() == ri).mean()
    gs2, gi2 = st.search_blend(qe.cuda(), qm[:, :5].contiguous().cuda(), 5, -1.0, k)
    torch.cuda.synchronize()
    print(f"B={B} k={k}: max |score err| {err:.2e}, id agreement {same:.4f}", flush=True)
st.close()
