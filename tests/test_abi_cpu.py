"""Host-side checks that need no GPU: the C-ABI library builds for sm_100a,
loads, and exports every symbol include/fmoe.h declares; the binding fails
loudly rather than falling back."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "fmoe.h")


def declared_functions():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fmoe_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def libpath():
    import __graft_entry__
    return __graft_entry__._builder().build()


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for required in ("fmoe_store_create", "fmoe_store_insert", "fmoe_search_semantic",
                     "fmoe_search_trajectory", "fmoe_select_experts"):
        assert required in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (fmoe_\w+)", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_library_is_sm100a_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_binding_loads_and_reports_errors_without_gpu(libpath):
    import ctypes
    import paper_2502_05370_b200 as fm
    for n in declared_functions():
        assert hasattr(fm._lib, n)
        assert n in fm.ABI_SYMBOLS
    assert fm._lib.fmoe_status_string(1) == b"invalid argument"
    # a bad config is rejected on the host before touching a device
    cfg = fm.fmoe_store_config(32, 65, 2, 64, 3, fm.FMOE_BF16, 10, 0)   # E > 64
    h = ctypes.c_void_p()
    assert fm._lib.fmoe_store_create(ctypes.byref(cfg), 0, ctypes.byref(h)) == 2
    cfg = fm.fmoe_store_config(32, 8, 2, 64, 32, fm.FMOE_BF16, 10, 0)   # d >= L
    assert fm._lib.fmoe_store_create(ctypes.byref(cfg), 0, ctypes.byref(h)) == 2
    assert b"d < L" in fm._lib.fmoe_last_error()
    # null store -> INVALID_ARG
    assert fm._lib.fmoe_search_semantic(None, 1, None, 1, None, None, None) == 1
    # expert hits: K > E, E > 64, T < 1 are rejected on the host; B = 0 is a no-op
    assert fm._lib.fmoe_expert_hits(2, 3, 8, 9, None, None, None, None, 0, None) == 1
    assert fm._lib.fmoe_expert_hits(2, 3, 65, 2, None, None, None, None, 0, None) == 1
    assert fm._lib.fmoe_expert_hits(2, 0, 8, 2, None, None, None, None, 0, None) == 1
    assert fm._lib.fmoe_expert_hits(0, 3, 8, 2, None, None, None, None, 0, None) == 0
    # session sweep: null session / outputs -> INVALID_ARG before any device work
    assert fm._lib.fmoe_traj_session_sweep(None, None, 1, None, None, -1.0, 3, None, None, None, None, None) == 1
    assert fm._lib.fmoe_kernel_launch_count() == 0


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2502_05370_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle|#include\s+\S*oracle", src, re.M), f


def test_bench_reference_arm_runs_on_cpu():
    """bench.py --impl reference (the oracle arm of the driver's comparison)
    prints one JSON line with the contract's keys, on the host only."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "searches/s"
    assert line["cpu_baseline"]["kind"] == "oracle" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["config"]["workload"].startswith("C1")
