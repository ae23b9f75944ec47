"""Micro-timings of single ABI calls (CUDA events, back-to-back launches).

    python tools/micro.py [--n 1000000]
Prints average µs per call and GB/s of algorithmic bytes for trajectory
searches at several prefix lengths, semantic search, and select."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmoe_synth as S  # noqa: E402
import paper_2502_05370_b200 as fm  # noqa: E402


GRAPH = False


def timeit(fn, reps=200, warm=10):
    """µs per call: back-to-back stream launches, or (GRAPH) replay of a CUDA
    graph of `reps` calls, which removes host launch overhead."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if GRAPH:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            g.capture_begin()
            for _ in range(reps):
                fn()
            g.capture_end()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3 / reps
    import time
    h0 = time.perf_counter()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    timeit.host_us = (h1 - h0) * 1e6 / reps
    return a.elapsed_time(b) * 1e3 / reps


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=1_000_000)
    p.add_argument("--D", type=int, default=4096)
    p.add_argument("--E", type=int, default=8)
    p.add_argument("--L", type=int, default=32)
    p.add_argument("--B", type=int, default=1)
    p.add_argument("--k", type=int, default=1)
    p.add_argument("--dtype", default="bf16")
    p.add_argument("--graph", action="store_true")
    a = p.parse_args()
    global GRAPH
    GRAPH = a.graph
    sh = S.Shape("m", a.L, a.E, 2, a.D, 64)
    st = fm.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, a.n, a.dtype)
    for s0 in range(0, a.n, 65536):
        c = min(65536, a.n - s0)
        e, m, _ = S.store_rows(sh, 1, s0, c, device="cuda")
        st.insert(e, m)
    torch.cuda.synchronize()
    qe, qm, _ = S.queries(sh, 1, a.n, a.B, device="cuda")
    s = 2 if a.dtype == "bf16" else 4
    out_s = torch.empty(a.B, a.k, device="cuda")
    out_i = torch.empty(a.B, a.k, dtype=torch.int64, device="cuda")
    for ell in (1, 2, 4, 8, 16, a.L - 1):
        pre = qm[:, :ell].contiguous()
        us = timeit(lambda: fm.fmoe_search_trajectory(st._h, pre, ell, a.k, out_s, out_i))
        print(f"traj ell={ell:2d}: {us:8.2f} us  {a.n * ell * a.E * s / us / 1e3:8.1f} GB/s  host {getattr(timeit, 'host_us', 0):.1f} us/call")
    sess = fm.fmoe_traj_session_create(st._h, a.B)
    lays = [qm[:, l].contiguous() for l in range(a.L)]

    def sweep():
        fm.fmoe_traj_session_reset(sess)
        for ell in range(1, a.L):
            fm.fmoe_traj_session_step(sess, lays[ell - 1], a.k, out_s, out_i)
    us = timeit(sweep, reps=5, warm=2)
    print(f"session sweep ell=1..{a.L - 1}: {us:8.2f} us ({us / (a.L - 1):.2f} us/step)")
    # per-step times of one eager sweep (events between steps)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.L)]
    for rep in range(2):
        fm.fmoe_traj_session_reset(sess)
        ev[0].record()
        for ell in range(1, a.L):
            fm.fmoe_traj_session_step(sess, lays[ell - 1], a.k, out_s, out_i)
            ev[ell].record()
        torch.cuda.synchronize()
    per = [ev[i - 1].elapsed_time(ev[i]) * 1e3 for i in range(1, a.L)]
    print("session step us: " + " ".join(f"{ell}:{t:.0f}" for ell, t in enumerate(per, 1)))
    fm.fmoe_traj_session_destroy(sess)
    us = timeit(lambda: fm.fmoe_search_semantic(st._h, qe, a.k, out_s, out_i), reps=50)
    print(f"semantic   : {us:8.2f} us  {a.n * a.D * s / us / 1e3:8.1f} GB/s")
    pre = qm.contiguous()
    us = timeit(lambda: fm.fmoe_search_blend(st._h, qe, pre, a.L, -1.0, a.k, out_s, out_i), reps=50)
    print(f"blend ell=L: {us:8.2f} us  {a.n * (a.D + a.L * a.E) * s / us / 1e3:8.1f} GB/s")
    ids = out_i[:, 0].contiguous()
    sc = out_s[:, 0].contiguous()
    mk = torch.empty(a.B, 1, dtype=torch.int64, device="cuda")
    ct = torch.empty(a.B, 1, dtype=torch.int32, device="cuda")
    us = timeit(lambda: fm.fmoe_select_experts(st._h, ids, sc, -1.0, 5, 6, mk, ct))
    print(f"select     : {us:8.2f} us")
    x = torch.empty(1, device="cuda")
    us = timeit(lambda: x.add_(1))
    print(f"torch add_ : {us:8.2f} us (launch floor reference)")
    st.close()


if __name__ == "__main__":
    main()
