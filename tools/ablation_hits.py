"""Expert hit rate of the map-search ablation variants (SURVEY §8(f)
NEXT #3) on seeded synthetic clustered traces, through the C ABI on one B200.

For each model shape (Table 1): a store of N historical iterations, B new
requests (half planted near a stored context, half fresh cluster draws, the
fmoe_synth recipe of DESIGN.md §4), and for each variant the prefetch guidance
of every layer (paper_2502_05370_b200.ablation) and its hits against the top-K
of each request's own gate (fmoe_expert_hits).  Prints one JSON object.

  python tools/ablation_hits.py [--N 100000] [--B 256] [--out profiles/...json]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import fmoe_synth as S  # noqa: E402
import paper_2502_05370_b200 as fm  # noqa: E402
from paper_2502_05370_b200 import ablation  # noqa: E402


def popcount64(m):
    m = m.clone()
    c = torch.zeros_like(m)
    for _ in range(64):
        c += m & 1
        m = m >> 1   # arithmetic shift: bit 63 pattern is masked by "& 1" each round
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=100_000)
    ap.add_argument("--B", type=int, default=256)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    res = {"N": a.N, "B": a.B + a.B // 2, "queries": f"{a.B} (half planted, half fresh) + {a.B // 2} novel", "store_dtype": a.dtype, "d": 3, "data": "synthetic (fmoe_synth, seeded)",
           "hit_rate_def": "sum |top-K(own gate) & prefetch set| / (B*L*K)  (Reading R14)", "shapes": {}}
    for sh in (S.MIXTRAL, S.QWEN, S.PHI):
        seed = S.BASE_SEED + 7
        st = fm.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, a.N, a.dtype, device=0)
        for b in range(0, a.N, 16384):
            e, m, _ = S.store_rows(sh, seed, b, min(16384, a.N - b), device=dev)
            st.insert(e, m)
        # planted (near a stored context) + fresh (in-distribution clusters) + novel
        # (clusters the store never saw: low similarity, where delta widens the set)
        q_emb, q_maps, planted = S.queries(sh, seed, a.N, a.B, device=dev)
        n_emb, n_maps, _ = S.queries(sh, seed + 1000, 0, a.B // 2, device=dev)
        q_emb, q_maps = torch.cat([q_emb, n_emb]), torch.cat([q_maps, n_maps])
        kind = torch.cat([torch.where(planted >= 0, 0, 1), torch.full((a.B // 2,), 2, device=dev)])
        nq = q_emb.shape[0]
        out = {}
        for var in ablation.VARIANTS:
            ablation.prefetch_masks(st, q_emb, q_maps, var)          # warm-up
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            masks, ids, _ = ablation.prefetch_masks(st, q_emb, q_maps, var)
            t1.record()
            torch.cuda.synchronize()
            hits, _ = fm.expert_hits(q_maps, masks, sh.K)
            cnt = popcount64(masks).float()
            LK = sh.L * sh.K
            out[var] = {
                "hit_rate": round(hits.sum().item() / (nq * LK), 4),
                **{f"hit_rate_{nm}": round(hits[kind == c].sum().item() / max(1, int((kind == c).sum()) * LK), 4)
                   for c, nm in enumerate(("planted", "fresh", "novel"))},
                "mean_prefetched_per_layer": round(cnt.mean().item(), 3),
                **{f"mean_prefetched_{nm}": round(cnt[kind == c].mean().item(), 3)
                   for c, nm in enumerate(("planted", "fresh", "novel"))},
                "guidance_ms_per_iteration": round(t0.elapsed_time(t1), 3),
                "searches": (0 if var == "map_t" else 1) + (sh.L - 3),
            }
        res["shapes"][sh.name] = {"L": sh.L, "E": sh.E, "K": sh.K, "D": sh.D, **out}
        st.close()
        del q_emb, q_maps
        torch.cuda.empty_cache()
    js = json.dumps(res, indent=1)
    print(js)
    if a.out:
        with open(a.out, "w") as f:
            f.write(js + "\n")


if __name__ == "__main__":
    main()
