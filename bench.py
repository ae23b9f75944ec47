"""bench.py -- fMoE expert-map search on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl fmoe|reference]

One STEP = one inference iteration's worth of the paper's matcher for a batch of
B live requests (the whole §8(a) hot path):
  1. semantic search (Eq. 1) + top-k, then expert selection for layers 1..d
     from the matched map;
  2. for every observed prefix ell = 1..L-1: trajectory search (Eq. 2) + top-k,
     then selection for target layer ell+d when it exists;
  3. insert of the finished iteration's context into the full store: RDY scan
     (P:544-551), victim resolution, overwrite.
Per step and query that is 1 + (L-1) + 1 = 33 searches (Mixtral L = 32).

`value` = searches/s over all ranks with inputs resident in HBM; `e2e` = the
same step through the C ABI with HOST (pinned) input/output tensors, the
library staging H2D/D2H inside the timed region.  Timing: CUDA events on the
launching stream after W warm-up steps, barrier + synchronize on both sides,
max over ranks.  The store (>= 8 GB) is far larger than L2 (126 MB), so every
step streams it from HBM.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fmoe_synth as S  # noqa: E402

WORKLOADS = {
    # configs[1] of BASELINE.json: Mixtral-8x7B shape, N = 1M maps, batch 1, trajectory ell = 1..31
    "C2": dict(shape=S.MIXTRAL, N=1_000_000, B=1, k=1, dtype="bf16", delta=-1.0),
    # configs[2]: Qwen1.5-MoE shape, N = 1M, batch 64, top-8
    "C3": dict(shape=S.QWEN, N=1_000_000, B=64, k=8, dtype="bf16", delta=-1.0),
    # configs[3]: Phi-3.5-MoE shape, N = 4M, blended searches (ell = 16, 31; SURVEY §8 C4
    # proposal) + insert of the batch at full capacity (B = 64)
    "C4": dict(shape=S.PHI, N=4_000_000, B=64, k=8, dtype="bf16", delta=-1.0, kind="blend", ells=(16, 31),
               insert=64),
    # configs[4] at 1 GPU: Mixtral shape, N = 16M, B = 256, blend at ell = 31, insert of 64 contexts
    "C5": dict(shape=S.MIXTRAL, N=16_000_000, B=256, k=8, dtype="bf16", delta=-1.0, kind="blend", ells=(31,),
               insert=64),
    # configs[0]: tiny Mixtral-shaped store (correctness config)
    "C1": dict(shape=S.TINY, N=1000, B=1, k=1, dtype="f32", delta=0.9),
}


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=3)
    # default: C5, the configuration BASELINE.json's north-star target names
    # (16M maps, batch 256, bf16 fits one B200); C1..C4 are parity/bench cases
    p.add_argument("--config", default="C5", choices=sorted(WORKLOADS))
    p.add_argument("--impl", default="fmoe", choices=["fmoe", "reference"])
    p.add_argument("--traj", default="sweep", choices=["sweep", "session", "stateless"],
                   help="trajectory steps: one session-sweep call (B = 1, k = 1: every step in one launch, running "
                        "dots in registers; other batches fall back to 'session'), one incremental session step "
                        "per layer (SURVEY §8(f) #1), or one stateless search per prefix")
    p.add_argument("--no-graph", dest="graph", action="store_false",
                   help="time eager launches instead of a CUDA-graph replay of the step")
    p.add_argument("--no-cos", dest="cos", action="store_false",
                   help="insert with a full RDY scan instead of reusing the semantic search's cosines")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--seed", type=int, default=S.BASE_SEED + 1)
    return p.parse_args()


# ------------------------------------------------------------------ accounting
def step_counts(cfg):
    sh = cfg["shape"]
    B = cfg["B"]
    if cfg.get("kind") == "blend":
        n_traj = len(cfg["ells"])
        return B * (1 + n_traj) + cfg["insert"], n_traj
    n_traj = sh.L - 1
    searches = B * (1 + n_traj + 1)
    return searches, n_traj


def batched_session(cfg):
    """A session over a batch on a bf16 store runs the tcgen05 scan over the whole
    prefix each step (seeded with the previous step's rows), not the
    incremental running-dot kernel; its algorithmic bytes are the stateless ones."""
    return cfg["dtype"] == "bf16" and cfg["B"] >= 5


def use_sweep(cfg):
    """fmoe_traj_session_sweep's fused kernel: one request (B = 1), top-1, 16-byte slab rows."""
    s = 2 if cfg["dtype"] == "bf16" else 4
    E16 = (cfg["shape"].E * s + 15) // 16 * 16
    return cfg["B"] == 1 and cfg["k"] == 1 and E16 == 16 and cfg.get("kind") != "blend"


def algorithmic_bytes(cfg, N, traj_mode="stateless", use_cos=False):
    """bytes a scan must stream per launch (store tiles only).
    Session step ell: slab ell-1, the prefix-norm row, and the per-query running
    dot product (read from step 2 on, written every step)."""
    sh = cfg["shape"]
    s = 2 if cfg["dtype"] == "bf16" else 4
    sem = N * sh.D * s
    B = cfg["B"]
    if cfg.get("kind") == "blend":
        traj = {ell: N * (sh.D + ell * sh.E) * s for ell in cfg["ells"]}
        if use_cos:   # fmoe_search_blend_cos: map prefix + the B cached cosines per row
            traj = {ell: N * (ell * sh.E * s + 4 * B) for ell in cfg["ells"]}
    elif traj_mode == "sweep" and use_sweep(cfg):
        # slab + prefix-norm row per step; the running dots live in registers and
        # are written back once (charged to the last step)
        traj = {ell: N * (sh.E * s + 4 + (4 * B if ell == sh.L - 1 else 0)) for ell in range(1, sh.L)}
    elif traj_mode in ("session", "sweep") and not batched_session(cfg):
        traj = {ell: N * (sh.E * s + 4 + 4 * B * (2 if ell > 1 else 1)) for ell in range(1, sh.L)}
    else:
        traj = {ell: N * ell * sh.E * s for ell in range(1, sh.L)}
    rdy = N * (sh.D * s + sh.L * sh.E * s)
    if use_cos:
        # the semantic search also writes its B cosines per row; the RDY scan reads
        # the maps and the inserted rows' cosines instead of the embeddings
        nb = cfg.get("insert", B)
        sem += N * 4 * B
        rdy = N * (sh.L * sh.E * s + 4 * nb)
    return sem, traj, rdy


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, gpu_index: int):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        rows = [r.split(", ") for r in open(self.path).read().strip().splitlines() if r.strip()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for n, v in zip(names, r[3:7]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ the fMoE arm
def build_store(fm, cfg, N_local, offset, dev, seed):
    sh = cfg["shape"]
    st = fm.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, N_local, cfg["dtype"], device=dev.index, id_offset=offset)
    chunk = 65536 if sh.D <= 4096 else 16384
    for a in range(0, N_local, chunk):
        c = min(chunk, N_local - a)
        e, m, _ = S.store_rows(sh, seed, offset + a, c, device=dev)
        st.insert(e, m)
    torch.cuda.synchronize(dev)
    return st


class Step:
    """One matcher iteration (see module docstring) on a (possibly sharded) store."""

    def __init__(self, fm, st, cfg, traj_mode="stateless", use_cos=True):
        self.fm, self.st, self.cfg = fm, st, cfg
        self.sh = cfg["shape"]
        # (blend workloads search at fixed prefixes: no trajectory sweep, no session)
        self.sess = (fm.fmoe_traj_session_create(st._h, cfg["B"])
                     if traj_mode in ("session", "sweep") and cfg.get("kind") != "blend" else None)
        self.sweep = traj_mode == "sweep" and use_sweep(cfg)
        if self.sweep:
            n, B = self.sh.L - 1, cfg["B"]
            self.sw = (torch.empty(n, B, device=st.device), torch.empty(n, B, dtype=torch.int64, device=st.device),
                       torch.empty(n, B, dtype=torch.int64, device=st.device),
                       torch.empty(n, B, dtype=torch.int32, device=st.device))
        # semantic cosines kept on the device for the RDY insert (fmoe_store_insert_cos):
        # the iteration's new context carries the embedding its semantic search used
        # (a sharded store's cosine side output holds this rank's local columns)
        n = getattr(st, "cap_local", None) or len(st)
        self.stride = (n + 3) // 4 * 4
        # (B x N fp32; C5: 256 x 16M = 16.4 GB next to the 148 GB store -- allocated
        # when it leaves >= 6 GB of the device free)
        cos_b = cfg["B"] * self.stride * 4
        free = torch.cuda.mem_get_info(st.device)[0] if use_cos else 0
        self.cos = (torch.empty(cfg["B"], self.stride, device=st.device)
                    if use_cos and cos_b + (6 << 30) <= free else None)

    def semantic(self, h, q_emb, k, out_s, out_i):
        if self.cos is not None:
            self.fm.fmoe_search_semantic_cos(h, q_emb, k, out_s, out_i, self.cos, self.stride)
        else:
            self.fm.fmoe_search_semantic(h, q_emb, k, out_s, out_i)

    def blend(self, h, q_emb, pre, ell, k, out_s, out_i):
        # the semantic half from this iteration's semantic search (same queries, same store)
        if self.cos is not None:
            self.fm.fmoe_search_blend_cos(h, self.cos, self.stride, pre, ell, -1.0, k, out_s, out_i)
        else:
            self.fm.fmoe_search_blend(h, q_emb, pre, ell, -1.0, k, out_s, out_i)

    def insert(self, h, ne, nm):
        if self.cos is not None:
            self.fm.fmoe_store_insert_cos(h, ne, nm, self.cos, self.stride, None, None)
        else:
            self.fm.fmoe_store_insert(h, ne, nm, None, None)

    def run(self, q_emb, q_maps, new_emb, new_maps, ev=None):
        """ev: optional dict kind -> list of (start, end) CUDA events around the searches."""
        fm, st, sh, cfg = self.fm, self.st, self.sh, self.cfg
        k, d, L = cfg["k"], 3, sh.L
        h = st._h
        B = q_emb.shape[0]
        dev = q_emb.device
        out_s = torch.empty(B, k, device=dev)
        out_i = torch.empty(B, k, dtype=torch.int64, device=dev)
        mask = torch.empty(B, d, dtype=torch.int64, device=dev)
        cnt = torch.empty(B, d, dtype=torch.int32, device=dev)

        def rec(kind, fn):
            if ev is None:
                fn()
                return
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            ev.setdefault(kind, []).append((a, b))

        rec("semantic", lambda: self.semantic(h, q_emb, k, out_s, out_i))
        top_i = out_i[:, 0].contiguous()
        top_s = out_s[:, 0].contiguous()
        fm.fmoe_select_experts(h, top_i, top_s, cfg["delta"], 0, d, mask, cnt)
        m1 = torch.empty(B, 1, dtype=torch.int64, device=dev)
        c1 = torch.empty(B, 1, dtype=torch.int32, device=dev)
        if cfg.get("kind") == "blend":
            # blended searches (RDY weighting, w = d/L) at the configured prefixes
            for ell in cfg["ells"]:
                pre, _ = q_maps[ell - 1]
                rec(f"traj{ell}", lambda: self.blend(h, q_emb, pre, ell, k, out_s, out_i))
                tgt = ell - 1 + d
                if tgt < L:
                    top_i = out_i[:, 0].contiguous()
                    top_s = out_s[:, 0].contiguous()
                    fm.fmoe_select_experts(h, top_i, top_s, cfg["delta"], tgt, tgt + 1, m1, c1)
            nb = cfg["insert"]
            rec("rdy_insert", lambda: self.insert(h, new_emb[:nb].contiguous(), new_maps[:nb].contiguous()))
            return
        if self.sess is not None:
            fm.fmoe_traj_session_reset(self.sess)        # the store changed at the last insert
        if self.sweep:
            # layers 0..L-2 observed; step ell selects target layer ell-1+d (none past L)
            ql = new_maps[:, :L - 1].permute(1, 0, 2)     # [L-1][1][E]: a contiguous view for B = 1
            sw_s, sw_i, sw_m, sw_c = self.sw
            rec("traj_sweep", lambda: fm.fmoe_traj_session_sweep(self.sess, ql, sw_s, sw_i, cfg["delta"], d,
                                                                 sw_m, sw_c))
            rec("rdy_insert", lambda: self.insert(h, new_emb, new_maps))
            return
        for ell in range(1, L):
            pre, lay = q_maps[ell - 1]
            tgt = ell - 1 + d
            if self.sess is not None and tgt < L:
                # session step + selection of target layer ell+d in one call
                rec(f"traj{ell}", lambda: fm.fmoe_traj_session_step_select(self.sess, lay, k, out_s, out_i,
                                                                          cfg["delta"], tgt, tgt + 1, m1, c1))
                continue
            if self.sess is not None:
                rec(f"traj{ell}", lambda: fm.fmoe_traj_session_step(self.sess, lay, k, out_s, out_i))
            else:
                rec(f"traj{ell}", lambda: fm.fmoe_search_trajectory(h, pre, ell, k, out_s, out_i))
            if tgt < L:
                top_i = out_i[:, 0].contiguous()
                top_s = out_s[:, 0].contiguous()
                fm.fmoe_select_experts(h, top_i, top_s, cfg["delta"], tgt, tgt + 1, m1, c1)
        rec("rdy_insert", lambda: self.insert(h, new_emb, new_maps))


class HostStep(Step):
    """The same step through the C ABI with host (pinned) buffers: the library
    stages inputs H2D and outputs D2H inside the timed region.  Calls run with
    fmoe_set_host_sync(0): copies are stream-ordered and the step synchronises
    once, before it reads its result on the host (and, for k > 1, before the
    host picks each search's top-1 for the selection).  A top-1 with k = 1 is
    the search's own host output, handed to the next call as its input."""

    def __init__(self, fm, st, cfg, traj_mode="stateless", use_cos=True):
        super().__init__(fm, st, cfg, traj_mode, use_cos)
        B, k, d = cfg["B"], cfg["k"], 3
        pin = lambda *shape, dtype=torch.float32: torch.empty(*shape, dtype=dtype).pin_memory()
        self.out_s, self.out_i = pin(B, k), pin(B, k, dtype=torch.int64)
        self.top_s, self.top_i = pin(B), pin(B, dtype=torch.int64)
        self.mask, self.cnt = pin(B, d, dtype=torch.int64), pin(B, d, dtype=torch.int32)
        self.m1, self.c1 = pin(B, 1, dtype=torch.int64), pin(B, 1, dtype=torch.int32)
        if self.sweep:
            n = self.sh.L - 1
            self.sw = (pin(n, B), pin(n, B, dtype=torch.int64), pin(n, B, dtype=torch.int64),
                       pin(n, B, dtype=torch.int32))

    def top1(self, out_s, out_i):
        """Host buffers holding each query's top-1 (score, id) of the last search."""
        if out_s.shape[1] == 1:
            return out_s.view(-1), out_i.view(-1)      # the search's own output, stream-ordered
        torch.cuda.current_stream().synchronize()
        self.top_s.copy_(out_s[:, 0]); self.top_i.copy_(out_i[:, 0])
        return self.top_s, self.top_i

    def run(self, q_emb, q_maps, new_emb, new_maps, ev=None):
        prev = self.fm.fmoe_set_host_sync(0)
        try:
            return self._run(q_emb, q_maps, new_emb, new_maps)
        finally:
            self.fm.fmoe_set_host_sync(prev)

    def _run(self, q_emb, q_maps, new_emb, new_maps):
        fm, cfg = self.fm, self.cfg
        k, d, L = cfg["k"], 3, self.sh.L
        h = self.st._h
        out_s, out_i = self.out_s, self.out_i
        self.semantic(h, q_emb, k, out_s, out_i)      # cosines stay in device memory
        top_s, top_i = self.top1(out_s, out_i)
        fm.fmoe_select_experts(h, top_i, top_s, cfg["delta"], 0, d, self.mask, self.cnt)
        if cfg.get("kind") == "blend":
            for ell in cfg["ells"]:
                pre, _ = q_maps[ell - 1]
                self.blend(h, q_emb, pre, ell, k, out_s, out_i)
                tgt = ell - 1 + d
                if tgt < L:
                    top_s, top_i = self.top1(out_s, out_i)
                    fm.fmoe_select_experts(h, top_i, top_s, cfg["delta"], tgt, tgt + 1, self.m1, self.c1)
            nb = cfg["insert"]
            self.insert(h, new_emb[:nb].contiguous(), new_maps[:nb].contiguous())
            torch.cuda.current_stream().synchronize()   # the step's result, read on the host
            return float(out_s[0, 0])
        if self.sess is not None:
            fm.fmoe_traj_session_reset(self.sess)
        if self.sweep:
            sw_s, sw_i, sw_m, sw_c = self.sw
            fm.fmoe_traj_session_sweep(self.sess, new_maps[:, :L - 1].permute(1, 0, 2), sw_s, sw_i, cfg["delta"], d,
                                       sw_m, sw_c)
            self.insert(h, new_emb, new_maps)
            torch.cuda.current_stream().synchronize()   # the step's result, read on the host
            return float(sw_s[-1, 0])
        for ell in range(1, L):
            pre, lay = q_maps[ell - 1]
            tgt = ell - 1 + d
            if self.sess is not None and tgt < L:
                fm.fmoe_traj_session_step_select(self.sess, lay, k, out_s, out_i, cfg["delta"], tgt, tgt + 1,
                                                 self.m1, self.c1)
                continue
            if self.sess is not None:
                fm.fmoe_traj_session_step(self.sess, lay, k, out_s, out_i)
            else:
                fm.fmoe_search_trajectory(h, pre, ell, k, out_s, out_i)
            if tgt < L:
                top_s, top_i = self.top1(out_s, out_i)
                fm.fmoe_select_experts(h, top_i, top_s, cfg["delta"], tgt, tgt + 1, self.m1, self.c1)
        self.insert(h, new_emb, new_maps)
        torch.cuda.current_stream().synchronize()       # the step's result, read on the host
        return float(out_s[0, 0])

    @staticmethod
    def bytes_per_step(cfg, B, traj_mode="stateless"):
        sh, k, d, L = cfg["shape"], cfg["k"], 3, cfg["shape"].L
        if cfg.get("kind") == "blend":
            nb, ells = cfg["insert"], cfg["ells"]
            h2d = B * sh.D * 4 + sum(B * (sh.D + ell * sh.E) * 4 for ell in ells) + nb * (sh.D + L * sh.E) * 4
            n_sel = 1 + sum(1 for ell in ells if ell - 1 + d < L)
            h2d += n_sel * B * 12
            d2h = (1 + len(ells)) * B * k * 12 + B * d * 12 + (n_sel - 1) * B * 12
            return h2d, d2h
        inc = traj_mode in ("session", "sweep")
        traj_in = sum(B * (1 if inc else ell) * sh.E * 4 for ell in range(1, L))
        h2d = B * sh.D * 4 + traj_in + B * (sh.D + L * sh.E) * 4
        n_sel = 1 + sum(1 for ell in range(1, L) if ell - 1 + d < L)
        # map ids + scores into select (a session step selects on the device: no copy)
        h2d += (1 if inc else n_sel) * B * (8 + 4)
        if traj_mode == "sweep" and use_sweep(cfg):
            n_sel = L           # the sweep writes a (zero) mask + count for the steps past the last layer too
        d2h = (L) * B * k * (4 + 8)                                 # search outputs
        d2h += B * d * (8 + 4) + (n_sel - 1) * B * (8 + 4)          # masks + counts
        return h2d, d2h


def make_queries(cfg, N, pool, seed, dev):
    sh = cfg["shape"]
    B = cfg["B"]
    qs = []
    for p in range(pool):
        qe, qm, _ = S.queries(sh, seed + 101 * p, N, B, device=dev)
        pre = [(qm[:, :ell].contiguous(), qm[:, ell - 1].contiguous()) for ell in range(1, sh.L)]
        # the iteration's new context = its own semantic embedding + its full gate map
        qs.append((qe.contiguous(), pre, qe.contiguous(), qm.contiguous()))
    return qs


def build_sharded(cfg, rank, world, dev, seed):
    """The store sharded over the ranks by the library (fmoe_store_create_sharded):
    every rank makes the same collective insert calls; each writes only its slots."""
    from paper_2502_05370_b200 import dist as fdist
    sh = cfg["shape"]
    transport = os.environ.get("FMOE_DIST_TRANSPORT", "nccl")
    sst = fdist.ShardedExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, cfg["N"], cfg["dtype"], device=dev.index,
                                      transport=transport)
    chunk = 65536
    for a in range(0, cfg["N"], chunk):
        c = min(chunk, cfg["N"] - a)
        e, m, _ = S.store_rows(sh, seed, a, c, device=dev)
        sst.insert(e, m)
    torch.cuda.synchronize(dev)
    return sst


def run_fmoe(args, cfg, rank, world, local_rank):
    import paper_2502_05370_b200 as fm
    dev = torch.device("cuda", bench_device(local_rank))
    torch.cuda.set_device(dev)
    N_total = cfg["N"]
    if world > 1:
        # the same Step: every ABI call on a sharded store is collective (local
        # kernels + one in-library all-gather + merge), so N > 1 runs exactly
        # the N = 1 calls (session sweep, cached cosines, blend, RDY insert)
        st = build_sharded(cfg, rank, world, dev, args.seed)
        N_local = st.cap_local
        step = Step(fm, st, cfg, args.traj, args.cos)
    else:
        N_local = N_total
        st = build_store(fm, cfg, N_local, 0, dev, args.seed)
        step = Step(fm, st, cfg, args.traj, args.cos)
    pool = 4
    qs = make_queries(cfg, N_total, pool, args.seed, dev)
    searches, n_traj = step_counts(cfg)
    sem_b, traj_b, rdy_b = algorithmic_bytes(cfg, N_local, args.traj, getattr(step, "cos", None) is not None)

    # graphs at N > 1 need the NCCL transport (the HOST transport synchronises)
    use_graph = args.graph and (world == 1 or os.environ.get("FMOE_DIST_TRANSPORT", "nccl") == "nccl")
    run_stream = torch.cuda.Stream(device=dev) if use_graph else torch.cuda.current_stream(dev)
    with torch.cuda.stream(run_stream):
        for w in range(args.warmup):               # also creates this stream's scratch
            step.run(*qs[w % pool])
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ev = {}
    # 1. eager timed pass: CUDA events around every search call (roofline source)
    l0 = fm.kernel_launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    eager_steps = args.steps
    with torch.cuda.stream(run_stream):
        t0.record()
        for i in range(eager_steps):
            step.run(*qs[i % pool], ev=ev)
        t1.record()
    torch.cuda.synchronize()
    ms_eager = t0.elapsed_time(t1)
    launches_per_step = (fm.kernel_launch_count() - l0) / eager_steps
    graphs = []
    if use_graph:
        # 2. the step captured once per query set as a CUDA graph (no host launch
        #    overhead between the ~100 kernels of a step); the timed region replays it
        for p_ in range(pool):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=run_stream):
                step.run(*qs[p_])
            graphs.append(g)
        with torch.cuda.stream(run_stream):
            for p_ in range(pool):
                graphs[p_].replay()
        torch.cuda.synchronize()
    clk = ClockSampler(local_rank) if rank == 0 else None
    # FMOE_PROFILE_RANGE=1: the timed region is the profiler range (for
    # `ncu --profile-from-start off`: the launch list of the timed steps only,
    # not the store build)
    prof = os.environ.get("FMOE_PROFILE_RANGE") == "1"
    if prof:
        torch.cuda.profiler.start()
    if graphs:
        with torch.cuda.stream(run_stream):
            t0.record()
            for i in range(args.steps):
                graphs[i % pool].replay()
            t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
    else:
        with torch.cuda.stream(run_stream):
            t0.record()
            for i in range(args.steps):
                step.run(*qs[i % pool])
            t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
    if prof:
        torch.cuda.profiler.stop()
    launches = int(round(launches_per_step * args.steps))
    clocks = clk.stop() if clk else None
    if world > 1:
        t = torch.tensor([ms], device=dev if os.environ.get("FMOE_DIST_TRANSPORT", "nccl") == "nccl" else "cpu")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
        torch.distributed.barrier()
    ms_step = ms / args.steps

    # per-kind search durations (events on the launching stream, inside the timed region)
    kind_ms = {kk: sum(a.elapsed_time(b) for a, b in v) / eager_steps for kk, v in ev.items()}
    traj_ms = sum(v for kk, v in kind_ms.items() if kk.startswith("traj"))
    scan_ms = kind_ms.get("semantic", 0) + traj_ms + kind_ms.get("rdy_insert", 0)
    scan_bytes = sem_b + sum(traj_b.values()) + rdy_b
    peaks = load_peaks()
    # the dominant kernel of the step: the semantic scan (one launch per step at B <= 4;
    # prep + scan + merge (+ exact re-rank) at B >= 5), algorithmic bytes (or FLOPs) per
    # launch / its mean event time.  Bound by arithmetic intensity: the scan does
    # 2*B FLOPs per stored element of s bytes (AI = B FLOP/B for bf16); above the
    # ridge (sustained bf16 peak / HBM copy bandwidth) it is a tensor-core roofline.
    sem_ms = kind_ms.get("semantic", 0.0)
    sh_ = cfg["shape"]
    s_el = 2 if cfg["dtype"] == "bf16" else 4
    sem_store_b = N_local * sh_.D * s_el                      # the embeddings streamed once
    sem_flops = 2.0 * cfg["B"] * N_local * sh_.D
    ai = sem_flops / sem_store_b
    ridge = peaks["bf16_tflops_sustained"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    achieved = sem_b / (sem_ms * 1e-3) / 1e9 if sem_ms > 0 else 0.0
    tflops = sem_flops / (sem_ms * 1e-3) / 1e12 if sem_ms > 0 else 0.0
    agg = scan_bytes / (scan_ms * 1e-3) / 1e9 if scan_ms > 0 else 0.0
    tensor = cfg["dtype"] == "bf16" and cfg["B"] >= 5 and ai > ridge
    traffic = measured_traffic(args.config) if world == 1 else None   # the ncu capture is of the 1-GPU launch
    if tensor:
        head = {"bound": "tensor", "achieved": round(tflops, 1), "peak": peaks["bf16_tflops_sustained"],
                "unit": "TFLOP/s", "frac": round(tflops / peaks["bf16_tflops_sustained"], 4),
                "traffic": traffic.get("bytes") if isinstance(traffic, dict) else traffic,
                "peak_kind": "bf16 dense, sustained (kernel timed inside a long step), MEASURED_PEAKS.json",
                "algorithmic_flops_per_launch": sem_flops,
                "hbm": {"achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": round(achieved / peaks["hbm_gbs"], 4)}}
    else:
        head = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(achieved / peaks["hbm_gbs"], 4),
                "traffic": traffic.get("bytes") if isinstance(traffic, dict) else traffic,
                "peak_kind": "HBM copy bandwidth, MEASURED_PEAKS.json"}
    roofline = dict(head, **{
                "arithmetic_intensity": round(ai, 2), "ridge": round(ridge, 1),
                "ncu": traffic if isinstance(traffic, dict) else None,
                "kernel": "semantic scan (Eq. 1 + fused top-k), the largest share of the step; CUDA events "
                          "around each call on the launching stream, eager timed pass",
                "algorithmic_bytes_per_launch": sem_b,
                "share_of_step": round(sem_ms / (ms_eager / eager_steps), 3) if ms_eager > 0 else None,
                "step_aggregate": {"achieved": round(agg, 1), "frac": round(agg / peaks["hbm_gbs"], 4),
                                   "bytes": scan_bytes, "what": "all scans of a step (semantic, trajectory, RDY)"},
                "eager_ms_per_step": round(ms_eager / eager_steps, 4),
                "peak_source": peaks["source"],
                "breakdown": {
                    "semantic": {"ms": round(kind_ms.get("semantic", 0), 4), "GBps": round(sem_b / kind_ms.get("semantic", 1) / 1e6, 1)},
                    "trajectory_sweep": {"ms": round(traj_ms, 4), "GBps": round(sum(traj_b.values()) / max(traj_ms, 1e-9) / 1e6, 1)},
                    "rdy_insert": {"ms": round(kind_ms.get("rdy_insert", 0), 4), "GBps": round(rdy_b / kind_ms.get("rdy_insert", 1) / 1e6, 1)},
                    **({"traj_ell31_GBps": round(traj_b[sh_L(cfg) - 1] / kind_ms[f"traj{sh_L(cfg) - 1}"] / 1e6, 1)}
                       if f"traj{sh_L(cfg) - 1}" in kind_ms else {}),
                }})
    # strong scaling: a search covers the whole (sharded) store, so the job
    # completes `searches` per step whatever the number of ranks
    value = searches / (ms_step * 1e-3)

    e2e = None
    used_cos = getattr(step, "cos", None) is not None
    if not args.no_e2e and world == 1:
        hq = []
        for qe, pre, ne, nm in qs:
            hq.append((qe.cpu().pin_memory(), [(p.cpu().pin_memory(), l.cpu().pin_memory()) for p, l in pre],
                       ne.cpu().pin_memory(), nm.cpu().pin_memory()))
        used_cos = getattr(step, "cos", None) is not None   # what the timed step ran (read before clearing)
        if used_cos:
            # the host-buffer step allocates its own cosine side output (C5: 16 GB)
            graphs.clear()
            step.cos = None
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
        hstep = HostStep(fm, st, cfg, args.traj, args.cos)
        for w in range(2):
            hstep.run(*hq[w % pool])
        torch.cuda.synchronize()
        e_steps = max(3, args.steps // 2)
        t0h = time.perf_counter()
        for i in range(e_steps):
            hstep.run(*hq[i % pool])
        torch.cuda.synchronize()
        e_ms = (time.perf_counter() - t0h) * 1e3 / e_steps
        h2d, d2h = HostStep.bytes_per_step(cfg, cfg["B"], args.traj)
        e2e = {"value": round(searches / (e_ms * 1e-3), 2), "unit": "searches/s", "ms_per_step": round(e_ms, 4),
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "note": "host pinned buffers through the C ABI (library stages H2D/D2H on the stream); "
                       "fmoe_set_host_sync(0): one stream sync per step before the host reads the result "
                       "(plus one per top-1 hand-off when k > 1)"}
    for obj in (step, locals().get("hstep")):
        if obj is not None and getattr(obj, "sess", None) is not None:
            fm.fmoe_traj_session_destroy(obj.sess)
    st.close()
    return dict(value=value, ms_step=ms_step, roofline=roofline, e2e=e2e, clocks=clocks, launches=launches,
                N_local=N_local, cos=used_cos, graph=bool(graphs) or (use_graph and world == 1))


def cos_keys(cfg, cos):
    """What the step reused from the semantic search's B x N cosine side output."""
    out = {"insert": "RDY semantic half reused from the step's semantic search (fmoe_store_insert_cos)"
                     if cos else "full RDY scan"}
    if cfg.get("kind") == "blend":
        out["blend"] = ("semantic half reused from the step's semantic search (fmoe_search_blend_cos)"
                        if cos else "full blended scan (embeddings re-read)")
    return out


def bench_device(local_rank):
    """CUDA device of this rank: LOCAL_RANK, or FMOE_BENCH_DEVICE (ranks sharing one GPU, tests only)."""
    return int(os.environ.get("FMOE_BENCH_DEVICE", local_rank))


def sh_L(cfg):
    return cfg["shape"].L


def measured_traffic(config):
    """dram read+write bytes per launch of the dominant kernel from the committed
    `ncu --set full` capture summary (profiles/traffic.json), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        return json.load(open(p)).get(config)
    return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d.get("bf16_tflops"),
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d.get("bf16_tflops")),
                "source": "MEASURED_PEAKS.json (measured)"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "source": "B200_PROFILING.md fallback"}


# ------------------------------------------------------------------ the oracle arm (CPU)
def oracle_step_sample(cfg, seed, n_sample, steps=None, warmup=0, budget_s=15.0, max_steps=50):
    """Times the oracle (as it stands, never tuned) on steps of the workload,
    each against a bounded sample of n_sample stored rows (the same B queries,
    the same calls: search, select, blend, insert); returns (searches/s scaled
    to the full N -- every scan is linear in N --, timed steps, seconds, mean
    seconds per sample step).  steps=None: as many steps as fit in budget_s."""
    from oracle import fmoe_oracle as O
    sh = cfg["shape"]
    B, k, dt, d, L = cfg["B"], cfg["k"], cfg["dtype"], 3, sh.L
    emb, maps, _ = S.store_rows(sh, seed, 0, n_sample)
    store = O.Store(n_sample, L, sh.E, sh.D, d)
    store.insert(O.quantize(emb.numpy(), dt), O.quantize(maps.numpy(), dt))
    qe, qm, _ = S.queries(sh, seed, n_sample, B)
    qe, qm = O.quantize(qe.numpy(), dt), O.quantize(qm.numpy(), dt)
    ne, nm = qe, qm                      # the iteration's own context is inserted (as in the fMoE arm)
    searches, _ = step_counts(cfg)

    def one_step():
        s, i = store.search(qe, None, 0, 1.0, k)
        O.select_experts(store.maps, i[:, 0].tolist(), s[:, 0].tolist(), cfg["delta"], list(range(d)), sh.K)
        if cfg.get("kind") == "blend":
            for ell in cfg["ells"]:
                s, i = store.search(qe, qm, ell, d / L, k)
                if ell - 1 + d < L:
                    O.select_experts(store.maps, i[:, 0].tolist(), s[:, 0].tolist(), cfg["delta"], [ell - 1 + d],
                                     sh.K)
            store.insert(ne[:cfg["insert"]], nm[:cfg["insert"]])
            return
        for ell in range(1, L):
            s, i = store.search(None, qm, ell, 0.0, k)
            if ell - 1 + d < L:
                O.select_experts(store.maps, i[:, 0].tolist(), s[:, 0].tolist(), cfg["delta"], [ell - 1 + d], sh.K)
        store.insert(ne, nm)

    for _ in range(warmup):
        one_step()
    n, t0 = 0, time.perf_counter()
    while True:
        one_step()
        n += 1
        el = time.perf_counter() - t0
        if steps is not None:
            if n >= steps:
                break
        elif el >= budget_s or n >= max_steps:
            break
    per_step = el / n
    scale = cfg["N"] / n_sample
    return searches / (per_step * scale), n, el, per_step


def oracle_sample_rows(cfg):
    """Rows of the bounded sample one oracle step scans (about 1-4 s of fp64 work per step)."""
    sh = cfg["shape"]
    per_row = cfg["B"] * (sh.D + sh.L * sh.E) * (1 + len(cfg.get("ells", ())) + 1) if cfg["B"] > 1 else sh.D * 40
    return int(min(cfg["N"], max(4096, 4e9 // per_row)))


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=1)
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, seed):
    """The oracle as it stands on the host: once with every BLAS thread the host
    offers (`value`, `cores`), once pinned to one thread (`single_thread`)."""
    n_sample = oracle_sample_rows(cfg)
    v, steps, el, _ = oracle_step_sample(cfg, seed, n_sample, budget_s=12.0)
    single = None
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            v1, steps1, el1, _ = oracle_step_sample(cfg, seed, n_sample, budget_s=8.0, max_steps=3)
        single = {"value": round(v1, 4), "cores": 1, "sample": f"{steps1} step(s), {el1:.1f}s"}
    except ImportError:
        pass
    return {"value": round(v, 4), "unit": "searches/s", "cores": blas_threads(), "kind": "oracle",
            "cpu": cpu_model(), "nproc": os.cpu_count(), "single_thread": single,
            "sample": f"{steps} full step(s) ({step_counts(cfg)[0]} searches each) against {n_sample} of the "
                      f"{cfg['N']} stored maps, {el:.1f}s; time scaled x{cfg['N'] / n_sample:.2f} to N (scans are linear in N)"}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return f"{line.split(':', 1)[1].strip()} ({os.cpu_count()} logical CPUs)"
    except OSError:
        pass
    return f"{os.cpu_count()} logical CPUs"


# ------------------------------------------------------------------ main
def main():
    args = parse()
    cfg = WORKLOADS[args.config]
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    searches, n_traj = step_counts(cfg)
    sh = cfg["shape"]
    what = (f"semantic + blend (w=d/L) at ell={','.join(map(str, cfg['ells']))} + select + RDY insert of "
            f"{cfg['insert']} contexts" if cfg.get("kind") == "blend" else
            f"semantic + trajectory ell=1..{sh.L - 1} + select + RDY insert of the batch")
    # `config` names the WORKLOAD only (identical in both arms); how an arm runs
    # it goes to `impl_notes`
    base_config = {"workload": f"{args.config}: {sh.name} store N={cfg['N']} maps, L={sh.L}, E={sh.E}, D={sh.D}, "
                               f"batch {cfg['B']}, {what} at full capacity", "N": cfg["N"], "L": sh.L, "E": sh.E,
                   "D": sh.D, "B": cfg["B"], "k": cfg["k"], "store_dtype": cfg["dtype"],
                   "searches_per_step": searches,
                   "l2": "inputs larger than L2 (store >> 126 MB), no flush",
                   "parallelism": f"store sharded over {args.gpus} GPU(s)" if args.gpus > 1 else "1 GPU"}
    traj_note = ("blends at fixed prefixes (no per-layer trajectory steps)" if cfg.get("kind") == "blend" else
                 "stateless: one search over the whole prefix per ell" if args.traj == "stateless" else
                 "session sweep: the L-1 incremental steps of the request in one call "
                 "(fmoe_traj_session_sweep: running dots in registers, slab + norm row per step, "
                 "per-step top-1 + Eq. 4-6 selection by each step's last block)"
                 if args.traj == "sweep" and use_sweep(cfg) else
                 "batched session: per ell one tcgen05 scan over the whole prefix, seeded with "
                 "the previous step's rows (fmoe_traj_session_step)" if batched_session(cfg) else
                 "incremental session: step ell reads slab ell + running dots (SURVEY §8(f) #1)")
    fmoe_notes = {"trajectory": traj_note,
                  "launch": "CUDA graph replay of the step" if args.graph else "eager"}

    if args.impl == "reference":
        if rank != 0:
            return
        # W untimed + K timed oracle steps, each a bounded row sample of the
        # workload (the full store would take hours per step in fp64 on the host);
        # ms_per_step is the measured sample step, value the throughput scaled to N
        n_sample = oracle_sample_rows(cfg)
        v, steps, el, per_step = oracle_step_sample(cfg, args.seed, n_sample, steps=args.steps, warmup=args.warmup)
        cores = blas_threads()
        line = {"metric": "expert-map searches/sec (batched)", "impl": "reference", "value": round(v, 4),
                "unit": "searches/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": round(per_step * 1e3, 3), "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": base_config,
                "impl_notes": {"engine": "fp64 numpy oracle (oracle/fmoe_oracle.py) on the host cores: every search "
                                         "scores the whole (sampled) store, RDY insert scans embeddings + maps"},
                "ms_per_full_step_extrapolated": round(searches / v * 1e3, 3),
                "cpu_baseline": {"value": round(v, 4), "unit": "searches/s", "cores": cores, "kind": "oracle",
                                 "cpu": cpu_model(),
                                 "sample": f"{steps} timed step(s) after {args.warmup} warm-up, each against "
                                           f"{n_sample} of the {cfg['N']} stored maps ({el:.1f}s); time scaled "
                                           f"x{cfg['N'] / n_sample:.2f} to N (scans are linear in N)"},
                "e2e": {"value": round(v, 4), "unit": "searches/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    if world > 1:
        torch.cuda.set_device(bench_device(local_rank))
        if os.environ.get("FMOE_DIST_TRANSPORT", "nccl") == "host":
            # ranks sharing a GPU (tests): gloo for the plumbing and the store's HOST transport
            torch.distributed.init_process_group("gloo")
        else:
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", bench_device(local_rank)))
    res = run_fmoe(args, cfg, rank, world, local_rank)
    if rank != 0:
        torch.distributed.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args.seed)
    line = {"metric": "expert-map searches/sec (batched)", "value": round(res["value"], 2), "unit": "searches/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms_step"], 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": cfg["dtype"],
            "data": "synthetic (seeded clustered embeddings + softmax gate maps, fmoe_synth)",
            "config": base_config,
            "impl_notes": dict(fmoe_notes, launch="CUDA graph replay of the step" if res["graph"] else "eager",
                               **cos_keys(cfg, res["cos"])),
            "roofline": res["roofline"], "cpu_baseline": cpu, "e2e": res["e2e"], "clocks": res["clocks"],
            "gpu_launches": res["launches"]}
    print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
