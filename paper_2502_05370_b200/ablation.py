"""The map-search ablation variants of P:777-790 as switches, and their expert
hit rate on a batch of observed gates (Reading R14).

Host orchestration of C-ABI calls only (every score, top-k, selection and hit
count runs in the library's kernels):

* ``map_t``   -- trajectory search only: layers t >= d are guided by the
  trajectory match over the ell = t - d + 1 observed layers (Eq. 2);
  layers 0..d-1 get no guidance;
* ``map_ts``  -- plus the semantic match (Eq. 1) for layers 0..d-1;
* ``map_tsd`` -- plus similarity-aware selection delta = Clip(1 - s, 0, 1)
  (P:510-526); the two variants above take the fixed top-K of the matched map
  (delta = 0).

The oracle counterpart is ``oracle.fmoe_oracle.ablation_prefetch_masks`` (tests only).
"""
from __future__ import annotations

import torch

from . import expert_hits

VARIANTS = ("map_t", "map_ts", "map_tsd")


def prefetch_masks(store, q_emb, q_maps, variant: str, stream=None):
    """Prefetch masks [B][L] (int64 bit patterns), matched ids [B][L] (-1: no
    guidance) and match scores [B][L] (NaN: none) of one iteration of B
    requests whose full gates q_maps [B][L][E] will be observed."""
    if variant not in VARIANTS:
        raise ValueError(f"variant must be one of {VARIANTS}")
    B, L, d = q_maps.shape[0], store.L, store.d
    delta = -1.0 if variant == "map_tsd" else 0.0
    masks = torch.zeros(B, L, dtype=torch.int64, device=q_maps.device)
    ids = torch.full((B, L), -1, dtype=torch.int64, device=q_maps.device)
    scores = torch.full((B, L), float("nan"), dtype=torch.float32, device=q_maps.device)
    dd = min(d, L)
    if variant != "map_t" and dd > 0:
        s, i = store.search_semantic(q_emb, 1, stream)
        m, _ = store.select_experts(i[:, 0].contiguous(), s[:, 0].contiguous(), delta, 0, dd, stream)
        masks[:, :dd] = m
        ids[:, :dd] = i[:, :1]
        scores[:, :dd] = s[:, :1]
    for t in range(d, L):
        ell = t - d + 1
        s, i = store.search_trajectory(q_maps[:, :ell].contiguous(), ell, 1, stream)
        m, _ = store.select_experts(i[:, 0].contiguous(), s[:, 0].contiguous(), delta, t, t + 1, stream)
        masks[:, t:t + 1] = m
        ids[:, t] = i[:, 0]
        scores[:, t] = s[:, 0]
    return masks, ids, scores


def hit_rate(store, q_emb, q_maps, variant: str, stream=None):
    """(hit rate, hits [B][L], masks [B][L]) of one variant: hits against the
    top-K of each observed gate row, rate = sum(hits) / (B * L * K)."""
    masks, _, _ = prefetch_masks(store, q_emb, q_maps, variant, stream)
    hits, _ = expert_hits(q_maps.contiguous(), masks, store.K, stream)
    B, L = hits.shape
    return float(hits.sum().item()) / float(B * L * store.K), hits, masks
