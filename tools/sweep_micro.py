"""Session-sweep micro-timing: one fmoe_traj_session_sweep of the L-1 steps of a
B = 1 request, per sweep kernel (FMOE_SWEEP_KERNEL = row | reg | tma), CUDA
events around back-to-back sweeps, algorithmic GB/s = (L-1) * N * (E*s + 4) + 4N
(slab row + prefix norm per row and step, the accumulator write-back).

    python tools/sweep_micro.py [--n 1000000] [--kernels row,reg]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmoe_synth as S  # noqa: E402
import paper_2502_05370_b200 as fm  # noqa: E402


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--n", default="1000000", help="comma list of store sizes")
    p.add_argument("--L", type=int, default=32)
    p.add_argument("--E", type=int, default=8)
    p.add_argument("--dtype", default="bf16")
    p.add_argument("--kernels", default="row,reg")
    p.add_argument("--reps", type=int, default=20)
    a = p.parse_args()
    out = []
    for n in [int(x) for x in a.n.split(",")]:
        sh = S.Shape("m", a.L, a.E, 2, 64, 64)           # D = 64: the sweep reads only the maps
        st = fm.ExpertMapStore(sh.L, sh.E, sh.K, sh.D, 3, n, a.dtype)
        for s0 in range(0, n, 1 << 20):
            c = min(1 << 20, n - s0)
            e, m, _ = S.store_rows(sh, 1, s0, c, device="cuda")
            st.insert(e, m)
        qm = S.queries(sh, 2, n, 1, device="cuda")[1]
        ql = qm.permute(1, 0, 2).contiguous()[:a.L - 1]
        es = 2 if a.dtype == "bf16" else 4
        nbytes = (a.L - 1) * n * (a.E * es + 4) + 4 * n
        ref = None
        for kern in a.kernels.split(","):
            os.environ["FMOE_SWEEP_KERNEL"] = kern
            sess = st.trajectory_session(1)
            try:
                res = None
                for _ in range(3):
                    sess.reset()
                    res = sess.sweep(ql, -1.0, 3)
                torch.cuda.synchronize()
                if ref is None:
                    ref = res
                same = all(torch.equal(x, y) for x, y in zip(res, ref))
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * a.reps)]
                for r in range(a.reps):
                    sess.reset()
                    ev[2 * r].record()
                    sess.sweep(ql, -1.0, 3)
                    ev[2 * r + 1].record()
                torch.cuda.synchronize()
                ts = sorted(ev[2 * r].elapsed_time(ev[2 * r + 1]) * 1e3 for r in range(a.reps))
                med = ts[len(ts) // 2]
                row = {"n": n, "kernel": kern, "us_median": round(med, 2), "us_min": round(ts[0], 2),
                       "GBps": round(nbytes / med / 1e3, 1), "bytes": nbytes, "bit_identical_to_first": same}
                print(json.dumps(row))
                out.append(row)
            finally:
                sess.close()
        st.close()
    os.makedirs("gpurun_out", exist_ok=True)
    json.dump(out, open("gpurun_out/sweep_micro.json", "w"), indent=1)


if __name__ == "__main__":
    main()
