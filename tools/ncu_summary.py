"""Summarise ncu reports (.ncu-rep) and launch lists (.csv) into profiles/.

    python tools/ncu_summary.py gpurun_out/prof_sem.ncu-rep [...] > profiles/xx.md
    python tools/ncu_summary.py --launches gpurun_out/launches_c2.csv [--last N]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("lts__t_bytes.sum", "L2 bytes"),
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(f"(no data in {path})")
        return
    h, units = rows[0], rows[1]
    print(f"### {path}\n")
    for r in rows[2:]:
        d = dict(zip(h, r))
        u = dict(zip(h, units))
        print(f"- kernel: `{d.get('Kernel Name', '?')[:140]}`")
        for k, name in KEYS:
            if k in d and d[k] != "":
                print(f"  - {name} (`{k}`): {d[k]} {u.get(k, '')}")
        print()


def launches(path, last):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    data = data[-last:] if last else data
    tot = 0.0
    print("| # | kernel | grid | block | time (us) |\n|---|---|---|---|---|")
    for i, d in enumerate(data):
        us = float(d["Metric Value"]) / 1e3 if d["Metric Unit"] in ("ns", "nsecond") else float(d["Metric Value"])
        tot += us
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        print(f"| {i} | `{name[:80]}` | {d['Grid Size']} | {d['Block Size']} | {us:.1f} |")
    print(f"\nsum of {len(data)} launches: {tot:.1f} us (ncu-serialised, cold caches: compare shares, not absolutes)")


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--launches":
        last = int(args[3]) if len(args) > 3 and args[2] == "--last" else 0
        launches(args[1], last)
    else:
        for p in args:
            report(p)
