"""CPU oracle for fMoE expert-map search (arXiv 2502.05370) -- TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import this module.  The product path
(`paper_2502_05370_b200`) never imports it, and this module never imports the
product package: the two share no code.

Every function is the plain definition from the paper, evaluated in float64 with
numpy.  A library primitive (a dot product via ``@``, a stable sort) serves as a
step; there is no blocking, fusion or reordering beyond what the definition
states.  Citations are ``P:n`` = ``/root/reference/PAPER.md`` line ``n`` (and
``S:n`` for SPEC.md); every ambiguous passage is resolved by a reading listed in
DESIGN.md "Readings" (R1..R14) and named next to the code that takes it.

Inputs are whatever values the caller gives: to compare with a store that holds
bf16 tiles, pass the bf16-rounded values (``quantize``) -- the "O-store" view of
SURVEY.md §8(c) c8; pass the raw fp32 inputs for the "O-def" view.

Pinning (what makes this oracle trustworthy, see tests/test_oracle_pins.py):
every function below is pinned by SPEC worked examples, closed forms,
invariants and brute force; none is "parity unpinned".
"""
from __future__ import annotations

import itertools
import math

import numpy as np

NEG_INF = float("-inf")


# --------------------------------------------------------------------------
# storage format: the values a store of a given dtype holds (O-store view)
# --------------------------------------------------------------------------
def quantize(x, dtype: str) -> np.ndarray:
    """Round fp32 input to the store dtype with round-to-nearest-even.

    'f32' is the identity on fp32 inputs; 'bf16' keeps the top 16 bits of the
    fp32 pattern after RNE (IEEE/bfloat16 definition).  Reading R9: the store
    holds the raw (not re-normalised) rounded rows; cosine is scale-invariant
    (P:461-466), so no normalisation is needed before rounding.
    """
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    if dtype == "f32":
        return a.astype(np.float64)
    if dtype != "bf16":
        raise ValueError(dtype)
    u = a.view(np.uint32).astype(np.uint64)
    # RNE on the 16 dropped bits: add 0x7FFF + lsb of the kept part, truncate.
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) << 16
    nan = np.isnan(a)
    out = (r & 0xFFFFFFFF).astype(np.uint32).view(np.float32).astype(np.float64)
    out[nan] = np.nan
    return out


# --------------------------------------------------------------------------
# Eq. 1 / Eq. 2 : cosine similarity
# --------------------------------------------------------------------------
def cosine(a, b) -> float:
    """cos(a, b) = a.b / (||a|| ||b||)  -- the kernel of Eq. 1 and Eq. 2.

    Reading R3 (zero norm, the paper is silent): a zero-norm *query* has no
    cosine -> NaN; a zero-norm *stored* row scores 0 (it can never be a match).
    """
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    na = math.sqrt(float(np.dot(a, a)))
    nb = math.sqrt(float(np.dot(b, b)))
    if na == 0.0:
        return float("nan")
    if nb == 0.0:
        return 0.0
    return float(np.dot(a, b)) / (na * nb)


def pairwise_cosine(Q, S) -> np.ndarray:
    """B x C matrix of cosine(Q[x], S[y]) (the score matrices of Eq. 1 / Eq. 2)."""
    Q = np.asarray(Q, dtype=np.float64)
    S = np.asarray(S, dtype=np.float64)
    dots = Q @ S.T
    nq = np.sqrt(np.einsum("ij,ij->i", Q, Q))
    ns = np.sqrt(np.einsum("ij,ij->i", S, S))
    with np.errstate(divide="ignore", invalid="ignore"):
        out = dots / (nq[:, None] * ns[None, :])
    out[:, ns == 0.0] = 0.0          # R3: zero-norm stored row scores 0
    out[nq == 0.0, :] = np.nan       # R3: zero-norm query has no score
    return out


def semantic_scores(q_emb, store_emb) -> np.ndarray:
    """Eq. 1: score^sem_{x,y} = cos(sem^new_x, sem^old_y), a B x C matrix."""
    return pairwise_cosine(q_emb, store_emb)


def trajectory_scores(q_prefix, store_maps, ell: int) -> np.ndarray:
    """Eq. 2: cosine between the observed trajectory and stored map prefixes.

    q_prefix  : B x ell x E (or B x >=ell x E; only the first ell layers are used)
    store_maps: C x L x E
    Reading R1: ``ell`` = number of observed layers (the whole prefix observed so
    far); stored maps are truncated to the same ``ell`` layers and flattened to
    ell*E vectors (P:472 gives the dimension (l-1)J for prefix length l-1).
    """
    q = np.asarray(q_prefix, dtype=np.float64)
    m = np.asarray(store_maps, dtype=np.float64)
    if ell < 1 or ell > m.shape[1]:
        raise ValueError("ell must be in [1, L]")
    B, C, E = q.shape[0], m.shape[0], m.shape[2]
    qf = q[:, :ell, :].reshape(B, ell * E)
    mf = m[:, :ell, :].reshape(C, ell * E)
    return pairwise_cosine(qf, mf)


def blend_scores(sem, traj, w_sem: float) -> np.ndarray:
    """RDY: w*score^sem + (1-w)*score^map; the paper's w is d/L.

    Reading R4: the same weighted sum with a caller-chosen w is the blended
    search (w=1 -> semantic only, w=0 -> trajectory only).
    """
    return w_sem * np.asarray(sem, dtype=np.float64) + (1.0 - w_sem) * np.asarray(traj, dtype=np.float64)


def rdy_scores(q_emb, q_maps, store_emb, store_maps, d: int) -> np.ndarray:
    """RDY_{x,y} = d/L * score^sem + (L-d)/L * score^map over FULL maps."""
    L = np.asarray(store_maps).shape[1]
    sem = semantic_scores(q_emb, store_emb)
    traj = trajectory_scores(q_maps, store_maps, L)
    return (d / L) * sem + ((L - d) / L) * traj


# --------------------------------------------------------------------------
# top-k ("the historical iteration with the highest score is selected")
# --------------------------------------------------------------------------
def topk(scores, k: int, ids=None):
    """Per row, the k best (score desc, id asc); pad with (-inf, -1).

    P:466 / P:477 select the argmax; Reading R5: k>1 generalises it, ties go to
    the lowest id.  A row containing NaN (zero-norm query) returns
    (NaN, -1) everywhere.
    """
    s = np.asarray(scores, dtype=np.float64)
    B, C = s.shape
    if ids is None:
        ids = np.arange(C, dtype=np.int64)
    out_s = np.full((B, k), NEG_INF)
    out_i = np.full((B, k), -1, dtype=np.int64)
    for x in range(B):
        row = s[x]
        if np.isnan(row).any():
            out_s[x, :] = np.nan
            continue
        order = np.lexsort((ids, -row))[:k]      # primary: score desc, secondary: id asc
        for r, j in enumerate(order):
            out_s[x, r] = row[j]
            out_i[x, r] = ids[j]
    return out_s, out_i


# --------------------------------------------------------------------------
# similarity-aware expert selection
# --------------------------------------------------------------------------
def selection_threshold(score: float) -> float:
    """delta_l = Clip(1 - score, 0, 1) = max(0, min(1 - score, 1)).

    Reading R6: the score is clamped to [-1, 1] first; a NaN score
    (no match) gives delta = 1 (prefetch everything).
    """
    s = float(score)
    if math.isnan(s):
        return 1.0
    s = max(-1.0, min(1.0, s))
    return max(0.0, min(1.0 - s, 1.0))


def select_prefetch_set(p, delta: float, K: int):
    """Greedy Eq. 4-6: pick experts by descending probability until
    the picked mass is >= delta AND at least K experts are picked.

    Reading R7: ">= delta" (Constraint 5 at P:519; the prose "exceeds" at P:515
    is the same bound), ties -> lower expert index, K in [1, E]
    (Constraint 6 garbled at P:520), no renormalisation: if the mass never
    reaches delta, all E experts are taken.  The cumulative sum runs in the
    selection order, in float64.
    Returns (ordered expert list, bitmask).
    """
    p = np.asarray(p, dtype=np.float64)
    E = p.shape[0]
    order = sorted(range(E), key=lambda j: (-p[j], j))
    picked = []
    cum = 0.0
    for j in order:
        picked.append(j)
        cum = cum + p[j]
        if cum >= delta and len(picked) >= K:
            break
    mask = 0
    for j in picked:
        mask |= 1 << j
    return picked, mask


def select_experts(store_maps, map_id, score, delta, layers, K: int):
    """For each query x: the prefetch sets of the layers ``layers`` of its matched map.

    delta < 0 selects the similarity-aware threshold of ``score[x]``;
    delta in [0,1] is a fixed threshold (C1 config).  map_id -1 (no match) gives
    empty sets (Reading R10: the caller owns the cold-start fallback).
    Returns masks[B][T] (python ints) and counts[B][T].
    """
    m = np.asarray(store_maps, dtype=np.float64)
    B = len(map_id)
    masks, counts = [], []
    for x in range(B):
        mr, cr = [], []
        dl = selection_threshold(score[x]) if delta < 0 else float(delta)
        for t in layers:
            if map_id[x] < 0:
                mr.append(0)
                cr.append(0)
                continue
            picked, mask = select_prefetch_set(m[map_id[x], t], dl, K)
            mr.append(mask)
            cr.append(len(picked))
        masks.append(mr)
        counts.append(cr)
    return masks, counts


# --------------------------------------------------------------------------
# Expert Map Store with RDY de-duplication
# --------------------------------------------------------------------------
class Store:
    """Capacity-C store of (embedding, map) contexts; slot index = context id.

    Insert follows P:552-553 with Reading R8:
      * while |S| < C, a new context is appended to the next slot;
      * once full, every remaining new context x (batch order) replaces the old
        context y* = argmax_y RDY_{x,y} over OLD contexts not yet claimed in this
        batch (ties -> lowest id).  RDY is computed against the store as it stands
        after this batch's appends; slots written by this batch (appended or
        replaced) are claimed and never chosen again, so a batch never evicts its
        own rows.  With no unclaimed slot left the row is dropped (slot -1).
    """

    def __init__(self, capacity: int, L: int, E: int, D: int, d: int = 3):
        self.C, self.L, self.E, self.D, self.d = capacity, L, E, D, d
        self.emb = np.zeros((capacity, D))
        self.maps = np.zeros((capacity, L, E))
        self.n = 0

    def insert(self, emb, maps):
        emb = np.asarray(emb, dtype=np.float64)
        maps = np.asarray(maps, dtype=np.float64)
        B = emb.shape[0]
        slots = [-1] * B
        replaced = [-1] * B
        claimed = set()
        x = 0
        while x < B and self.n < self.C:
            y = self.n
            self.emb[y], self.maps[y] = emb[x], maps[x]
            self.n += 1
            claimed.add(y)
            slots[x] = y
            x += 1
        if x < B:
            rest = list(range(x, B))
            rdy = rdy_scores(emb[rest], maps[rest], self.emb[: self.n], self.maps[: self.n], self.d)
            writes = []
            for r, xi in enumerate(rest):
                best = -1
                for y in range(self.n):
                    if y in claimed:
                        continue
                    if best < 0 or rdy[r, y] > rdy[r, best]:
                        best = y
                if best >= 0:
                    claimed.add(best)
                    slots[xi] = best
                    replaced[xi] = best
                    writes.append((xi, best))
            for xi, y in writes:
                self.emb[y], self.maps[y] = emb[xi], maps[xi]
        return slots, replaced

    def search(self, q_emb, q_prefix, ell: int, w_sem: float, k: int):
        """Blended search (w_sem=1 semantic, 0 trajectory) + top-k over the stored contexts."""
        n = self.n
        B = (q_emb if q_emb is not None else q_prefix).shape[0]
        sem = semantic_scores(q_emb, self.emb[:n]) if w_sem != 0.0 else np.zeros((B, n))
        traj = trajectory_scores(q_prefix, self.maps[:n], ell) if w_sem != 1.0 else np.zeros((B, n))
        if w_sem == 1.0:
            s = sem
        elif w_sem == 0.0:
            s = traj
        else:
            s = blend_scores(sem, traj, w_sem)
        return topk(s, k)


# --------------------------------------------------------------------------
# sharding: the merge of per-shard top-k is the global top-k
# --------------------------------------------------------------------------
def merge_topk(cand_scores, cand_ids, k: int):
    """Merge candidate lists (score, global id) from several shards: (score desc, id asc)."""
    s = np.concatenate([np.asarray(c, dtype=np.float64) for c in cand_scores], axis=1)
    i = np.concatenate([np.asarray(c, dtype=np.int64) for c in cand_ids], axis=1)
    B = s.shape[0]
    out_s = np.full((B, k), NEG_INF)
    out_i = np.full((B, k), -1, dtype=np.int64)
    for x in range(B):
        if np.isnan(s[x]).any():
            out_s[x, :] = np.nan
            continue
        cand = [(s[x, j], i[x, j]) for j in range(s.shape[1]) if i[x, j] >= 0]
        cand.sort(key=lambda t: (-t[0], t[1]))
        for r, (sc, idx) in enumerate(cand[:k]):
            out_s[x, r], out_i[x, r] = sc, idx
    return out_s, out_i


def brute_force_min_prefetch_set(p, delta: float, K: int):
    """Exhaustive Eq. 4-6 over all 2^E subsets (E <= 16): returns (min size, all feasible
    subsets of that size as sorted tuples), or (E, [all experts]) if no subset reaches
    delta (Reading R7: take all E).  Test pin for ``select_prefetch_set``."""
    p = np.asarray(p, dtype=np.float64)
    E = p.shape[0]
    for size in range(K, E + 1):
        feasible = []
        for sub in itertools.combinations(range(E), size):
            srt = sorted(sub, key=lambda j: (-p[j], j))   # same float64 summation order
            cum = 0.0
            for j in srt:
                cum = cum + p[j]
            if cum >= delta:
                feasible.append(tuple(sorted(sub)))
        if feasible:
            return size, feasible
    return E, [tuple(range(E))]


# --------------------------------------------------------------------------
# Expert-cache priorities
# --------------------------------------------------------------------------
def prefetch_priority(p: float, layer: int, l_now: int) -> float:
    """PRI^prefetch_{l,j} = p_{l,j} / (l - l_now); requires l > l_now."""
    if layer <= l_now:
        raise ValueError("target layer must be after the current layer")
    return float(p) / float(layer - l_now)


def eviction_priority(p: float, freq: float, eps: float = 1e-6) -> float:
    """PRI^evict_{l,j} = 1 / (p_{l,j} * freq_{l,j}), p floored at eps (S:377,
    Reading R13: the paper's formula is undefined at p = 0)."""
    return 1.0 / (max(float(p), eps) * float(freq))


def prefetch_plan(store_maps, map_id, score, delta, layers, K, l_now):
    """Prefetch jobs of each query: every expert of the Eq. 4-6 prefetch set of each
    target layer t (selection as `select_experts`), with PRI^prefetch = p/(t - l_now),
    ordered by priority descending, ties -> lower layer, then lower expert.
    Layers are 0-based on both sides, so t - l_now is the paper's l - l_now.
    Returns, per query, a list of (t, j, priority)."""
    m = np.asarray(store_maps, dtype=np.float64)
    out = []
    for x in range(len(map_id)):
        jobs = []
        if map_id[x] >= 0:
            dl = selection_threshold(score[x]) if delta < 0 else float(delta)
            for t in layers:
                picked, _ = select_prefetch_set(m[map_id[x], t], dl, K)
                for j in picked:
                    jobs.append((t, j, prefetch_priority(m[map_id[x], t, j], t, l_now)))
        jobs.sort(key=lambda r: (-r[2], r[0], r[1]))
        out.append(jobs)
    return out


def eviction_order(p, freq, eps: float = 1e-6):
    """Cache entries (index = insertion order) sorted for eviction: PRI^evict descending,
    ties -> the least recently inserted (lower index) first."""
    pri = [eviction_priority(pp, ff, eps) for pp, ff in zip(p, freq)]
    order = sorted(range(len(pri)), key=lambda i: (-pri[i], i))
    return pri, order


# --------------------------------------------------------------------------
# Expert hit rate and the map-search ablation variants
# --------------------------------------------------------------------------
def activated_experts(gate, K: int):
    """The experts the router activates at one layer: the K highest gate
    probabilities (top-K routing, K from Table 1), ties -> lower
    expert index (Reading R14).  Returns (sorted expert list, bitmask)."""
    g = np.asarray(gate, dtype=np.float64)
    order = sorted(range(g.shape[0]), key=lambda j: (-g[j], j))
    act = sorted(order[:K])
    mask = 0
    for j in act:
        mask |= 1 << j
    return act, mask


def expert_hits(gate, masks, K: int):
    """Expert hits of prefetch guidance (an activated expert that was
    prefetched is a hit): for query x and layer t, hits = |A_{x,t} ∩ P_{x,t}|
    with A = activated_experts(gate[x][t], K) and P the prefetch set (bitmask
    masks[x][t]).  The hit rate is sum(hits) / (B*T*K): every layer activates
    exactly K experts (Constraint 2, "total number of activated experts").
    Returns (hits[B][T], active_masks[B][T])."""
    g = np.asarray(gate, dtype=np.float64)
    B, T = g.shape[0], g.shape[1]
    hits, act = [], []
    for x in range(B):
        hr, ar = [], []
        for t in range(T):
            _, a = activated_experts(g[x, t], K)
            hr.append(bin(a & int(masks[x][t])).count("1"))
            ar.append(a)
        hits.append(hr)
        act.append(ar)
    return hits, act


ABLATION_VARIANTS = ("map_t", "map_ts", "map_tsd")


def ablation_prefetch_masks(store_emb, store_maps, q_emb, q_maps, variant: str, d: int, K: int):
    """Prefetch guidance of one inference iteration under the ablation variants
    of P:777-790, for every layer t of every query:
      * layers t < d (no trajectory observed yet): the semantic match (Eq. 1)
        selects layers 0..d-1 -- "map_ts", "map_tsd"; "map_t"
        (trajectory only) has no guidance there (empty set, Reading R14);
      * layers t >= d: the trajectory match over the observed prefix of
        ell = t - d + 1 layers (Eq. 2, target ell + d, Reading R1) selects layer t;
      * selection: "map_tsd" uses the similarity-aware delta = Clip(1 - s, 0, 1)
        of the match; "map_t"/"map_ts" take the fixed top-K of the
        matched map (delta = 0, i.e. without the delta feature).
    Returns masks[B][L] (python ints) and the matched ids[B][L]."""
    q_emb = np.asarray(q_emb)
    q_maps = np.asarray(q_maps)
    B, L = q_maps.shape[0], q_maps.shape[1]
    if variant not in ABLATION_VARIANTS:
        raise ValueError(variant)
    delta = -1.0 if variant == "map_tsd" else 0.0
    masks = [[0] * L for _ in range(B)]
    ids = [[-1] * L for _ in range(B)]
    if variant != "map_t":
        ss, si = topk(semantic_scores(q_emb, store_emb), 1)
        m, _ = select_experts(store_maps, list(si[:, 0]), list(ss[:, 0]), delta, range(min(d, L)), K)
        for x in range(B):
            for t in range(min(d, L)):
                masks[x][t] = m[x][t]
                ids[x][t] = int(si[x, 0])
    for t in range(d, L):
        ell = t - d + 1
        ts, ti = topk(trajectory_scores(q_maps, store_maps, ell), 1)
        m, _ = select_experts(store_maps, list(ti[:, 0]), list(ts[:, 0]), delta, [t], K)
        for x in range(B):
            masks[x][t] = m[x][0]
            ids[x][t] = int(ti[x, 0])
    return masks, ids
