"""Batched (tcgen05) search timings at the C5 per-rank shape.

    python tools/batched_micro.py [--n 2000000] [--B 256] [--k 8] [--reps 5] [--once]

N = 2M rows is one rank's shard of C5 (16M maps) at G = 8.  Prints µs per
call, algorithmic GB/s and TFLOP/s for semantic, trajectory (ell = 31) and
blend (ell = 31) searches.  --once runs each call once after one warm-up
(for ncu captures)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmoe_synth as S  # noqa: E402
import paper_2502_05370_b200 as fm  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=2_000_000)
    p.add_argument("--D", type=int, default=4096)
    p.add_argument("--E", type=int, default=8)
    p.add_argument("--L", type=int, default=32)
    p.add_argument("--B", type=int, default=256)
    p.add_argument("--k", type=int, default=8)
    p.add_argument("--ell", type=int, default=31)
    p.add_argument("--ells", default="", help="comma list: trajectory sweep over these prefixes")
    p.add_argument("--reps", type=int, default=5)
    p.add_argument("--once", action="store_true")
    p.add_argument("--only", default="")
    p.add_argument("--dtype", default="bf16", help="store dtype: bf16 (tcgen05 path) or f32 (FFMA batched scan)")
    a = p.parse_args()
    sh = S.Shape("m", a.L, a.E, 2, a.D, 1024)
    st = fm.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, a.n, a.dtype)
    es = 2 if a.dtype == "bf16" else 4
    for s0 in range(0, a.n, 65536):
        c = min(65536, a.n - s0)
        e, m, _ = S.store_rows(sh, 1, s0, c, device="cuda")
        st.insert(e, m)
    torch.cuda.synchronize()
    qe, qm, _ = S.queries(sh, 1, a.n, a.B, device="cuda")
    out_s = torch.empty(a.B, a.k, device="cuda")
    out_i = torch.empty(a.B, a.k, dtype=torch.int64, device="cuda")
    pre = qm[:, :a.ell].contiguous()
    stride = (a.n + 3) // 4 * 4
    cos = torch.empty(a.B, stride, device="cuda") if "cos" in a.only else None
    calls = {
        "semantic_cos": (lambda: fm.fmoe_search_semantic_cos(st._h, qe, a.k, out_s, out_i, cos, stride), a.D),
        "blend_cos": (lambda: fm.fmoe_search_blend_cos(st._h, cos, stride, pre, a.ell, -1.0, a.k, out_s, out_i),
                      a.ell * a.E),
        "semantic": (lambda: fm.fmoe_search_semantic(st._h, qe, a.k, out_s, out_i), a.D),
        "trajectory": (lambda: fm.fmoe_search_trajectory(st._h, pre, a.ell, a.k, out_s, out_i), a.ell * a.E),
        "blend": (lambda: fm.fmoe_search_blend(st._h, qe, pre, a.ell, -1.0, a.k, out_s, out_i), a.D + a.ell * a.E),
    }
    if a.ells:
        for ell in [int(x) for x in a.ells.split(",")]:
            pre_l = qm[:, :ell].contiguous()
            fn = lambda: fm.fmoe_search_trajectory(st._h, pre_l, ell, a.k, out_s, out_i)
            fn()
            torch.cuda.synchronize()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            for _ in range(a.reps):
                fn()
            ev1.record()
            torch.cuda.synchronize()
            us = ev0.elapsed_time(ev1) * 1e3 / a.reps
            print(f"traj ell={ell:2d} B={a.B}: {us:8.1f} us  {a.n * ell * a.E * es / us / 1e3:7.1f} GB/s", flush=True)
        st.close()
        return
    for name, (fn, kdim) in calls.items():
        if (a.only and name not in a.only.split(",")) or (not a.only and name.endswith("_cos")):
            continue
        fn()
        torch.cuda.synchronize()
        if a.once:
            fn()
            torch.cuda.synchronize()
            continue
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(a.reps):
            fn()
        ev1.record()
        torch.cuda.synchronize()
        us = ev0.elapsed_time(ev1) * 1e3 / a.reps
        gb = (a.n * kdim * es + (a.n * a.B * 4 if name.endswith("_cos") else 0)) / us / 1e3
        tf = 2.0 * a.B * a.n * kdim / us / 1e6
        print(f"{name:10s} B={a.B} n={a.n}: {us:9.1f} us  {gb:7.1f} GB/s  {tf:7.1f} TFLOP/s", flush=True)
    st.close()


if __name__ == "__main__":
    main()
