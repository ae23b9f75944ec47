"""Per-block phase timeline of one search call (device %globaltimer stamps).

    python tools/trace.py [--ell 1] [--n 1000000] [--D 8] [--mode traj|sem]
Phases: 0 block start, 1 after griddepcontrol.wait, 2 queries staged,
3 main loop done, 4 block merge done, 5 (last block) grid merge start,
6 (last block) end.  Prints µs relative to the earliest block start."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmoe_synth as S  # noqa: E402
import paper_2502_05370_b200 as fm  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", type=int, default=1_000_000)
    p.add_argument("--D", type=int, default=8)
    p.add_argument("--E", type=int, default=8)
    p.add_argument("--L", type=int, default=32)
    p.add_argument("--ell", type=int, default=1)
    p.add_argument("--mode", default="traj")
    p.add_argument("--B", type=int, default=1)
    p.add_argument("--k", type=int, default=1)
    a = p.parse_args()
    lib = fm._lib
    lib.fmoe_debug_trace.restype = ctypes.c_int
    lib.fmoe_debug_trace.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    sh = S.Shape("m", a.L, a.E, 2, a.D, 64)
    st = fm.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, a.n, "bf16")
    for s0 in range(0, a.n, 65536):
        e, m, _ = S.store_rows(sh, 1, s0, min(65536, a.n - s0), device="cuda")
        st.insert(e, m)
    qe, qm, _ = S.queries(sh, 1, a.n, a.B, device="cuda")
    pre = qm[:, :a.ell].contiguous()
    out_s = torch.empty(a.B, a.k, device="cuda")
    out_i = torch.empty(a.B, a.k, dtype=torch.int64, device="cuda")

    sess = fm.fmoe_traj_session_create(st._h, a.B) if a.mode == "session" else None
    stride = (a.n + 3) // 4 * 4
    cos = None
    if a.mode == "blend_cos":
        cos = torch.empty(a.B, stride, device="cuda")
        fm.fmoe_search_semantic_cos(st._h, qe, a.k, out_s, out_i, cos, stride)
    lays = [qm[:, l].contiguous() for l in range(a.L)]

    def call():
        if a.mode == "session":
            fm.fmoe_traj_session_reset(sess)
            for l in range(a.ell - 1):
                fm.fmoe_traj_session_step(sess, lays[l], a.k, out_s, out_i)
            torch.cuda.synchronize()
            if lib.fmoe_debug_trace(-1, None, 0) == 0 and getattr(call, "arm", False):
                lib.fmoe_debug_trace(1, None, 0)
                ev0.record()
            fm.fmoe_traj_session_step(sess, lays[a.ell - 1], a.k, out_s, out_i)
            return
        if a.mode == "traj":
            fm.fmoe_search_trajectory(st._h, pre, a.ell, a.k, out_s, out_i)
        elif a.mode == "blend_cos":
            fm.fmoe_search_blend_cos(st._h, cos, stride, pre, a.ell, -1.0, a.k, out_s, out_i)
        else:
            fm.fmoe_search_semantic(st._h, qe, a.k, out_s, out_i)
    for _ in range(5):
        call()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if a.mode == "session":
        call.arm = True
    else:
        lib.fmoe_debug_trace(1, None, 0)
        ev0.record()
    call()
    ev1.record()
    torch.cuda.synchronize()
    buf = np.zeros((4096, 8), dtype=np.uint64)
    lib.fmoe_debug_trace(-1, buf.ctypes.data, 4096)
    lib.fmoe_debug_trace(0, None, 0)
    used = buf[:, 0] > 0
    t = buf[used].astype(np.int64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    rel[t == 0] = np.nan
    print(f"mode={a.mode} ell={a.ell} blocks={used.sum()} event time {ev0.elapsed_time(ev1) * 1e3:.1f} us")
    names = ["start", "pdl_wait", "staged", "loop_done", "blk_merge", "last_start", "last_end", "ph7"]
    if a.B >= 5:
        names = ["start", "epi_tile0_done", "epi_wait0", "epi_all_done", "epi_tile0_ready", "tma_done", "end", "mma_done"]
    for ph in range(8):
        col = rel[:, ph]
        col = col[~np.isnan(col)]
        if col.size:
            print(f"  {names[ph]:10s} n={col.size:4d} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f} us")
    flat = buf.reshape(-1)
    if a.B >= 5:
        roles = flat[8192:8192 + 4 * 256].reshape(4, 256).astype(np.int64)
        ntile = int((roles[0] > 0).sum())
        print("  CTA 0 per-tile timeline (us from kernel start): tile | tma_issued | mma_committed | epi_got | epi_done")
        for i in range(min(ntile, 12)):
            print("   ", i, " ".join(f"{(roles[r, i] - t0) / 1e3:8.2f}" for r in range(4)))
        iss = flat[16384:16384 + 1024].astype(np.int64)
        got = flat[17408:17408 + 1024].astype(np.int64)
        nk = int((iss > 0).sum())
        if nk:
            lat = (got[:nk] - iss[:nk]) / 1e3
            gap = np.diff(got[:nk]) / 1e3
            print(f"  CTA 0 stages: n={nk} load issue->MMA-got latency med {np.median(lat):.2f} p10 {np.percentile(lat,10):.2f}"
                  f" p90 {np.percentile(lat,90):.2f} us; MMA-got interval med {np.median(gap):.3f} us")
            print("   first 24 (issue, got) us:", [(round((iss[i]-t0)/1e3,2), round((got[i]-t0)/1e3,2)) for i in range(min(24,nk))])
            print("   steady 200..212:", [(round((iss[i]-t0)/1e3,2), round((got[i]-t0)/1e3,2)) for i in range(200, min(212,nk))])
        cy = flat[12288:12288 + 256 * 18].reshape(256, 3, 6).astype(np.int64)
        if cy.any():      # library built with -DFMOE_EPI_PROFILE
            print("  epilogue kcycles of lane 0 per warp [tfull bar tmem_ld fast rare other] (rest: other = candidates of the warp, tiles >= 2):")
            for w in range(8):
                c = cy[w * 32] // 1000; c[2, 5] = cy[w * 32:(w + 1) * 32, 2, 5].sum()
                print(f"    warp {w}: tile0 {c[0].tolist()}  tile1 {c[1].tolist()}  rest {c[2].tolist()}")
            def ksc(u):
                u = int(u) >> 32
                if u == 0:
                    return float("-inf")
                b = (u & 0x7fffffff) if (u & 0x80000000) else (~u & 0xffffffff)
                return float(np.array([b], dtype=np.uint32).view(np.float32)[0])
            g0 = [ksc(v) for v in cy[0:64:8, 0, 5]]
            g1 = [ksc(v) for v in cy[0:64:8, 1, 5]]
            print("  initial g score (lanes 0,8,..,56):", ["%.5f" % v for v in g0])
            print("  final   g score (lanes 0,8,..,56):", ["%.5f" % v for v in g1])
    st.close()


if __name__ == "__main__":
    main()
