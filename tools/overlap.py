"""Asynchronous matcher next to a synthetic MoE forward on one B200
(P:528-533 publisher-subscriber, "non-async ops < 30 ms";
SURVEY §8(f) NEXT #4).

Main stream: a Mixtral-8x7B-shaped decode forward of one token (L = 32 layers;
per layer the router GEMM and the K = 2 activated experts' SwiGLU FFNs,
4096 -> 14336 -> 4096, bf16, random weights, cuBLAS via torch -- the forward is
workload, not product), each layer captured as a CUDA graph.
Side stream: the fMoE matcher of the C2 step through the C ABI -- semantic search
+ selection of layers 1..d at the iteration start, then, as soon as layer ell's
gate is observed (an event on the main stream), the trajectory-session step with
the fused selection of target layer ell + d, and the insert of the iteration's
context at the end.

Reports: forward time per iteration alone / with the matcher (the interference
overhead), the matcher alone, and per target layer the slack between "guidance
ready" (side-stream event) and "forward starts that layer" (main-stream event):
negative slack = the guidance arrived too late to prefetch.

  python tools/overlap.py [--N 1000000] [--iters 20] [--out profiles/...json] [--copies --expert-mb 352]

--copies adds the expert loading the guidance drives (P:573-580, P:595-597,
P:618-619): after each session step the side stream records an event; a
copy-manager thread waits for it and calls fmoe_prefetch_issue, which computes
the PRI^prefetch plan of the target layer on a copy stream and issues one
cudaMemcpyAsync per planned expert from pinned host memory into device expert
slots (a ring: weights of every expert share one pinned buffer
of --expert-mb MB; content is irrelevant, the DMA is real).  Reports per target
layer the copy completion vs the forward reaching that layer.
"""
import threading
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import fmoe_synth as S  # noqa: E402
import paper_2502_05370_b200 as fm  # noqa: E402

H, F = 4096, 14336


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1_000_000)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--tokens", type=int, default=1)
    ap.add_argument("--out", default=None)
    ap.add_argument("--copies", action="store_true")
    ap.add_argument("--expert-mb", type=float, default=3 * 4096 * 14336 * 2 / 2 ** 20)   # one Mixtral expert
    ap.add_argument("--slots", type=int, default=8)
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    cfg = dict(bench.WORKLOADS["C2"])
    cfg["N"] = a.N
    sh = cfg["shape"]
    L, d, K = sh.L, 3, sh.K
    print("build", file=sys.stderr, flush=True)
    st = bench.build_store(fm, cfg, a.N, 0, dev, S.BASE_SEED + 1)
    step = bench.Step(fm, st, cfg, "session", True)
    q_emb, q_pre, new_emb, new_maps = bench.make_queries(cfg, a.N, 1, S.BASE_SEED + 1, dev)[0]

    # ---- synthetic forward: weights of the activated experts of every layer (22.5 GB bf16)
    g = torch.Generator(device=dev).manual_seed(1)
    w_r = torch.randn(L, H, sh.E, device=dev, dtype=torch.bfloat16, generator=g) * 0.02
    w_up = torch.empty(L, K, H, 2 * F, device=dev, dtype=torch.bfloat16).normal_(0, 0.02, generator=g)
    w_dn = torch.empty(L, K, F, H, device=dev, dtype=torch.bfloat16).normal_(0, 0.02, generator=g)
    x = torch.randn(a.tokens, H, device=dev, dtype=torch.bfloat16, generator=g)
    main_s = torch.cuda.Stream(device=dev)
    side_s = torch.cuda.Stream(device=dev)

    def layer_fn(l):
        def f():
            gate = torch.softmax((x @ w_r[l]).float(), dim=-1)          # the observed gate of layer l
            y = torch.zeros_like(x)
            for e in range(K):
                h = x @ w_up[l, e]
                y += (torch.nn.functional.silu(h[:, :F]) * h[:, F:]) @ w_dn[l, e]
            x.add_(y * 1e-3)
            return gate
        return f

    graphs = []
    with torch.cuda.stream(main_s):
        for l in range(L):
            f = layer_fn(l)
            f()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=main_s):
                f()
            graphs.append(gr)
    torch.cuda.synchronize()

    k = 1
    h = st._h
    out_s = torch.empty(1, k, device=dev)
    out_i = torch.empty(1, k, dtype=torch.int64, device=dev)
    mask = torch.empty(1, d, dtype=torch.int64, device=dev)
    cnt = torch.empty(1, d, dtype=torch.int32, device=dev)
    m1 = torch.empty(1, 1, dtype=torch.int64, device=dev)
    c1 = torch.empty(1, 1, dtype=torch.int32, device=dev)

    def E():
        return torch.cuda.Event(enable_timing=True)

    # ---- expert copies driven by the guidance (--copies)
    eb = int(a.expert_mb * 2 ** 20) // 16 * 16
    if a.copies:
        host_w = torch.empty(eb, dtype=torch.uint8).pin_memory()
        dev_slots = torch.empty(a.slots, eb, dtype=torch.uint8, device=dev)
        host_ptrs = [host_w.data_ptr()] * (L * sh.E)
        dev_ptrs = [dev_slots[(t * sh.E + j) % a.slots].data_ptr() for t in range(L) for j in range(sh.E)]
        copy_s = torch.cuda.Stream(device=dev)
        step_ids = torch.empty(L, 1, dtype=torch.int64, device=dev)
        step_sc = torch.empty(L, 1, device=dev)

    def copy_manager(t0, copied, n_jobs, guide_ev, guide_set):
        """One fmoe_prefetch_issue per target layer, each after its step's guidance event.
        (The library can also make the copy stream wait on a device flag -- wait_flag -- but a
        device-side wait ahead of the flag's producer in a shared hardware queue deadlocks, and
        here the producer is enqueued later by another thread: the host waits on the event.)"""
        resident = torch.zeros(L, dtype=torch.int64)
        for ell in range(1, L):
            tgt = ell - 1 + d
            if tgt >= L:
                break
            guide_set[ell].wait()              # the main thread has recorded the event
            guide_ev[ell].synchronize()        # the guidance of step ell is written
            lay, exp, nj = fm.fmoe_prefetch_issue(h, step_ids[ell], step_sc[ell], -1.0, ell - 1, tgt, tgt + 1, sh.E,
                                                  host_ptrs, dev_ptrs, eb, resident, None, copy_s)
            ev = E()
            ev.record(copy_s)
            copied[tgt] = ev
            n_jobs[tgt] = int(nj[0])

    def iteration(do_fwd, do_match, rec=None, do_copy=False):
        t0, start, ready, gate_ev = E(), [E() for _ in range(L)], [None] * L, [E() for _ in range(L)]
        f_end, m_end = E(), E()
        main_s.wait_stream(torch.cuda.current_stream())
        side_s.wait_stream(torch.cuda.current_stream())
        copied, n_jobs, th = [None] * L, [0] * L, None
        guide_ev = [E() for _ in range(L)]
        guide_set = [threading.Event() for _ in range(L)]
        if do_copy:
            copy_s.wait_stream(torch.cuda.current_stream())
            torch.cuda.synchronize()
        t0.record(main_s)
        side_s.wait_event(t0)
        if do_copy:
            copy_s.wait_event(t0)
            th = threading.Thread(target=copy_manager, args=(t0, copied, n_jobs, guide_ev, guide_set))
            th.start()
        if do_match:
            with torch.cuda.stream(side_s):
                step.semantic(h, q_emb, k, out_s, out_i)
                fm.fmoe_select_experts(h, out_i[:, 0].contiguous(), out_s[:, 0].contiguous(), -1.0, 0, d, mask, cnt)
                r = E()
                r.record(side_s)
                for t in range(d):
                    ready[t] = r
                fm.fmoe_traj_session_reset(step.sess)
        for l in range(L):
            if do_fwd:
                with torch.cuda.stream(main_s):
                    start[l].record(main_s)
                    graphs[l].replay()
                    gate_ev[l].record(main_s)
            if do_match and l + 1 < L:
                ell, tgt = l + 1, l + d
                with torch.cuda.stream(side_s):
                    if do_fwd:
                        side_s.wait_event(gate_ev[l])
                    lay = q_pre[ell - 1][1]
                    if tgt < L:
                        fm.fmoe_traj_session_step_select(step.sess, lay, k, out_s, out_i, -1.0, tgt, tgt + 1, m1, c1)
                        r = E()
                        r.record(side_s)
                        ready[tgt] = r
                        if do_copy:                                  # publish the guidance of step ell
                            step_ids[ell].copy_(out_i[0])
                            step_sc[ell].copy_(out_s[0])
                            guide_ev[ell].record(side_s)
                            guide_set[ell].set()
                    else:
                        fm.fmoe_traj_session_step(step.sess, lay, k, out_s, out_i)
        if do_match:
            with torch.cuda.stream(side_s):
                step.insert(h, new_emb, new_maps)
        f_end.record(main_s)
        m_end.record(side_s)
        if th is not None:
            th.join()
        torch.cuda.current_stream().wait_stream(main_s)
        torch.cuda.current_stream().wait_stream(side_s)
        if do_copy:
            torch.cuda.current_stream().wait_stream(copy_s)
        torch.cuda.synchronize()
        res = {"fwd_ms": t0.elapsed_time(f_end) if do_fwd else None,
               "match_ms": t0.elapsed_time(m_end) if do_match else None}
        if do_fwd and do_match:
            res["slack_ms"] = [t0.elapsed_time(start[t]) - t0.elapsed_time(ready[t]) for t in range(L)]
        if do_copy:
            res["copy_slack_ms"] = [t0.elapsed_time(start[t]) - t0.elapsed_time(copied[t]) if copied[t] else None
                                    for t in range(L)]
            res["copy_done_ms"] = max(t0.elapsed_time(c) for c in copied if c)
            res["experts_copied"] = sum(n_jobs)
        return res

    log = lambda *m: print(*m, file=sys.stderr, flush=True)  # noqa: E731
    log("warm-up")
    for _ in range(3):
        iteration(True, True)
    runs = {}
    for name, fw, mt in (("forward_alone", True, False), ("matcher_alone", False, True), ("concurrent", True, True)):
        log(name)
        rs = [iteration(fw, mt) for _ in range(a.iters)]
        runs[name] = rs
    if a.copies:
        log("with copies")
        iteration(True, True, do_copy=True)
        runs["with_copies"] = [iteration(True, True, do_copy=True) for _ in range(a.iters)]
    med = lambda v: sorted(v)[len(v) // 2]  # noqa: E731
    fa = med([r["fwd_ms"] for r in runs["forward_alone"]])
    fc = med([r["fwd_ms"] for r in runs["concurrent"]])
    ma = med([r["match_ms"] for r in runs["matcher_alone"]])
    mc = med([r["match_ms"] for r in runs["concurrent"]])
    slack = [med([r["slack_ms"][t] for r in runs["concurrent"]]) for t in range(L)]
    res = {
        "what": "Mixtral-shaped 1-token decode forward (router + 2 SwiGLU experts per layer, bf16, per-layer CUDA "
                "graphs) on the main stream; the C2 matcher (semantic + select, 31 session steps with fused "
                "selection of layer ell+d gated on layer ell's gate event, insert) on a side stream",
        "N": a.N, "iters": a.iters, "tokens": a.tokens,
        "forward_ms_alone": round(fa, 4), "forward_ms_with_matcher": round(fc, 4),
        "forward_overhead_frac": round(fc / fa - 1.0, 4),
        "matcher_ms_alone": round(ma, 4), "matcher_ms_concurrent": round(mc, 4),
        "guidance_slack_ms_per_target_layer": [round(v, 4) for v in slack],
        "late_layers": [t for t in range(L) if slack[t] < 0],
        "expert_weight_bytes_per_forward": int(L * K * (H * 2 * F + F * H) * 2),
    }
    if a.copies:
        wc = runs["with_copies"]
        cs = [med([r["copy_slack_ms"][t] for r in wc]) if wc[0]["copy_slack_ms"][t] is not None else None
              for t in range(L)]
        nexp = med([r["experts_copied"] for r in wc])
        done = med([r["copy_done_ms"] for r in wc])
        res["copies"] = {
            "expert_bytes": eb, "experts_copied_per_iteration": nexp,
            "forward_ms_with_matcher_and_copies": round(med([r["fwd_ms"] for r in wc]), 4),
            "copies_done_ms_after_start": round(done, 4),
            "copy_GBps": round(nexp * eb / (done * 1e-3) / 1e9, 2) if done > 0 else None,
            "copy_slack_ms_per_target_layer": [None if v is None else round(v, 4) for v in cs],
            "what": "fmoe_prefetch_issue per target layer ell+d, called by a copy-manager thread once step ell's "
                    "guidance event completed: PRI^prefetch plan on the copy stream, then one cudaMemcpyAsync per planned expert "
                    "(pinned host -> device slot), PRI^prefetch order; slack = forward reaches the layer - "
                    "that layer's copies done (negative: late)"}
    js = json.dumps(res, indent=1)
    print(js)
    if a.out:
        with open(a.out, "w") as f:
            f.write(js + "\n")
    st.close()


if __name__ == "__main__":
    main()
