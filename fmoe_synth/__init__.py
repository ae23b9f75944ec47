"""Seeded synthetic inputs for fMoE expert-map search -- shared by tests, bench and smoke.

This module holds NO arithmetic of the method (no cosine, no blending, no top-k,
no selection): it only draws store contents and queries with the structure of
the paper's workloads, so that both the CUDA path and the CPU oracle can be fed
the same fp32 tensors.  Recipe:

* shapes: Table 1 -- Mixtral L=32 E=8 K=2, Qwen1.5-MoE L=24 E=60
  K=4, Phi-3.5-MoE L=32 E=16 K=2; hidden sizes 4096 / 2048 / 4096;
* embeddings: ``n_clusters`` centroids c ~ N(0, I_D); a row of cluster z is
  ``scale * (c_z + 0.5 * g)`` with g ~ N(0, I_D) and ``scale`` ~ U(0.5, 2)
  (intra-cluster cosine ~0.8; cosine is scale-invariant, the random scale
  exercises it);
* maps: gate distributions, the softmax of router-like logits (P:410-415 defines
  P_l as the gate's probability distribution): per (cluster, layer) an archetype
  logit vector A ~ N(0, 1.5^2 I_E); a row's layer-l gate is
  softmax(A_{z,l} + 0.7 * g'), g' ~ N(0, I_E) -- peaked, top-2 mass ~0.6-0.9;
* queries: a fraction ``planted`` are perturbations of stored rows (embedding
  noise 0.05 relative, gate-logit noise 0.05), the rest are fresh draws from the
  same clusters.

Rows are generated in blocks of ``BLOCK`` global indices, each block from its
own seeded ``torch.Generator`` on the requested device, so any row range is
reproducible without generating the whole store (needed at N = 1M..16M).  The
CPU and CUDA generators differ; a test always feeds the SAME tensor to both
sides.
"""
from __future__ import annotations

import dataclasses

import torch

BLOCK = 16384
BASE_SEED = 2502053700


@dataclasses.dataclass(frozen=True)
class Shape:
    name: str
    L: int
    E: int
    K: int
    D: int
    n_clusters: int = 1024


MIXTRAL = Shape("mixtral-8x7b", 32, 8, 2, 4096)
QWEN = Shape("qwen1.5-moe", 24, 60, 4, 2048)
PHI = Shape("phi-3.5-moe", 32, 16, 2, 4096)
TINY = Shape("tiny-mixtral", 32, 8, 2, 64, n_clusters=16)

# BASELINE.json configs (C1..C5), see SURVEY.md §8
CONFIGS = {
    "C1": dict(shape=TINY, N=1000, B=1, k=1, delta=0.9, dtype="f32"),
    "C2": dict(shape=MIXTRAL, N=1 << 20, B=1, k=1, delta=-1.0, dtype="bf16"),
    "C3": dict(shape=QWEN, N=1 << 20, B=64, k=8, delta=-1.0, dtype="bf16"),
    "C4": dict(shape=PHI, N=4 << 20, B=64, k=8, delta=-1.0, dtype="bf16"),
    "C5": dict(shape=MIXTRAL, N=16 << 20, B=256, k=8, delta=-1.0, dtype="bf16"),
}


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed & 0x7FFFFFFFFFFFFFFF)
    return g


def _centroids(shape: Shape, seed: int, device):
    g = _gen(seed * 7 + 1, device)
    c = torch.randn(shape.n_clusters, shape.D, generator=g, device=device)
    a = 1.5 * torch.randn(shape.n_clusters, shape.L, shape.E, generator=g, device=device)
    return c, a


def store_rows(shape: Shape, seed: int, start: int, count: int, device="cpu"):
    """Rows [start, start+count) of the synthetic store: (emb[count,D] f32, maps[count,L,E] f32, cluster[count])."""
    c, a = _centroids(shape, seed, device)
    embs, maps, zs = [], [], []
    b0, b1 = start // BLOCK, (start + count - 1) // BLOCK
    for b in range(b0, b1 + 1):
        g = _gen(seed * 1_000_003 + b, device)
        z = torch.randint(0, shape.n_clusters, (BLOCK,), generator=g, device=device)
        scale = 0.5 + 1.5 * torch.rand(BLOCK, 1, generator=g, device=device)
        lo = max(start, b * BLOCK) - b * BLOCK
        hi = min(start + count, (b + 1) * BLOCK) - b * BLOCK
        zz = z[lo:hi]
        ge = torch.randn(BLOCK, shape.D, generator=g, device=device)[lo:hi]
        gl = torch.randn(BLOCK, shape.L, shape.E, generator=g, device=device)[lo:hi]
        embs.append(scale[lo:hi] * (c[zz] + 0.5 * ge))
        maps.append(torch.softmax(a[zz] + 0.7 * gl, dim=-1))
        zs.append(zz)
    return torch.cat(embs), torch.cat(maps), torch.cat(zs)


def queries(shape: Shape, seed: int, n_store: int, B: int, planted: float = 0.5, device="cpu"):
    """B queries: (q_emb[B,D], q_maps[B,L,E], planted_id[B] (-1 for fresh draws)).

    A planted query perturbs stored row y (noise 0.05 relative on the embedding,
    0.05 on the gate logits) so its best match is y with a known margin.
    """
    g = _gen(seed * 31 + 17, device)
    n_pl = int(round(B * planted)) if n_store > 0 else 0
    ids = torch.randint(0, max(n_store, 1), (n_pl,), generator=g, device=device)
    ids = torch.unique(ids)  # distinct planted targets
    n_pl = ids.numel()
    q_emb = torch.empty(B, shape.D, device=device)
    q_maps = torch.empty(B, shape.L, shape.E, device=device)
    planted_id = torch.full((B,), -1, dtype=torch.int64, device=device)
    for j in range(n_pl):
        y = int(ids[j])
        e, m, _ = store_rows(shape, seed, y, 1, device)
        ne = torch.randn(1, shape.D, generator=g, device=device)
        q_emb[j] = e[0] + 0.05 * e[0].norm() / shape.D ** 0.5 * ne[0]
        logits = torch.log(m[0].clamp_min(1e-30)) + 0.05 * torch.randn(shape.L, shape.E, generator=g, device=device)
        q_maps[j] = torch.softmax(logits, dim=-1)
        planted_id[j] = y
    n_fresh = B - n_pl
    if n_fresh:
        c, a = _centroids(shape, seed, device)
        z = torch.randint(0, shape.n_clusters, (n_fresh,), generator=g, device=device)
        q_emb[n_pl:] = c[z] + 0.5 * torch.randn(n_fresh, shape.D, generator=g, device=device)
        q_maps[n_pl:] = torch.softmax(a[z] + 0.7 * torch.randn(n_fresh, shape.L, shape.E, generator=g, device=device), dim=-1)
    return q_emb, q_maps, planted_id
