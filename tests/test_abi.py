"""The C-ABI library loads and exports every symbol include/*.h declares; host-side
argument validation (no GPU, no compute calls)."""
import ctypes
import glob
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = []
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        names += re.findall(r"^\s*(?:sm_status|int64_t|int32_t|void|const\s+char\s*\*)\s*\*?\s*(\w+)\s*\(", text, flags=re.M)
    return names


@pytest.fixture(scope="module")
def sm():
    import build_native
    build_native.build()
    import paper_1202_6575_b200 as sm
    return sm


def test_header_declares_entry_points():
    names = declared_functions()
    for kt in ("u32", "i32", "i64", "u64", "f32", "f64", "u128"):
        for f in ("merge_stable", "mergesort_stable", "merge_stable_ex", "merge_plan_ex", "mergesort_stable_ex",
                  "merge_stable_batched", "ranks_stable"):
            assert f"{f}_{kt}" in names
            assert f"{f}_desc_{kt}" in names          # descending order
        for f in ("merge_stable_wide", "merge_stable_batched_wide", "mergesort_stable_wide"):
            assert f"{f}_{kt}" in names and f"{f}_desc_{kt}" in names   # wide payloads (row 2)
    assert len(names) == 156          # + sm_sort_run_n, sm_set_k1_variant, sm_plan_from_ranks, sm_debug_cover,
    #                                     sm_is_debug_build, sm_set_small_fuse, sm_plan_tasks, sm_set_sort_ways,
    #                                     sm_sort_merge_passes


def test_library_exports_every_declared_symbol(sm):
    lib = ctypes.CDLL(sm.LIB_PATH)
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", sm.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(\w+)$", out, flags=re.M))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a(sm):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sm.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_host_validation_without_gpu(sm):
    lib = sm._lib
    P = ctypes.c_void_p
    # negative sizes -> SM_EINVAL before any CUDA call
    assert lib.merge_stable_u32(None, None, -1, None, None, 0, None, None, None) == sm.SM_EINVAL
    assert lib.mergesort_stable_i64(None, None, -5, None) == sm.SM_EINVAL
    # NULL keys with a nonzero size
    assert lib.merge_stable_i32(None, None, 10, None, None, 0, None, None, None) == sm.SM_EINVAL
    # payload pointers half set
    assert lib.merge_stable_u32(P(0x1000), P(0x2000), 4, P(0x3000), None, 4, P(0x9000), None, None) == sm.SM_EINVAL
    # sizes beyond 32-bit in-kernel indices: accepted by merge_stable (coarse
    # partition; here the aliasing check answers first), rejected with options
    assert lib.merge_stable_u64(P(0x1000), None, 1 << 31, P(0x1000), None, 1, P(0x1000), None, None) == sm.SM_EALIAS
    opt = sm.SmOptions(0, 0, 1024, 0, 0)
    assert lib.merge_stable_ex_u64(P(1 << 40), None, 1 << 31, P(1 << 41), None, 1, P(1 << 42), None, None,
                                   ctypes.byref(opt)) == sm.SM_EINVAL
    # output overlapping an input -> SM_EALIAS
    assert lib.merge_stable_u32(P(0x10000), None, 100, P(0x20000), None, 100, P(0x10100), None, None) == sm.SM_EALIAS
    assert sm._lib.sm_status_string(sm.SM_EALIAS).startswith(b"SM_EALIAS")
    assert b"invalid" in sm._lib.sm_status_string(sm.SM_EINVAL)
    # invalid tuning options
    opt = sm.SmOptions(0, 0, 10 ** 6, 0, 0)
    assert lib.merge_stable_ex_u32(P(0x10000), None, 100, P(0x20000), None, 100, P(0x30000), None, None,
                                   ctypes.byref(opt)) == sm.SM_EINVAL
    opt = sm.SmOptions(1, 0, 0, 0, 0)
    assert lib.merge_stable_ex_u32(P(0x10000), None, 100, P(0x20000), None, 100, P(0x30000), None, None,
                                   ctypes.byref(opt)) == sm.SM_EINVAL


def test_tile_constants(sm):
    cap = sm.tile_capacity("u32", True)
    assert cap >= 256 and sm.sort_run("u32", True) >= 256
    # block-sort runs: 256 x 33 for key + payload slots of <= 8 bytes, else 256 x 17
    assert [sm.sort_run(kt, v) for kt, v in (("u32", True), ("i32", False), ("i64", False), ("u64", True),
                                             ("f64", True), ("u128", False))] == [8448, 8448, 8448, 4352, 4352, 4352]


def test_product_path_never_imports_the_oracle():
    """The oracle is test infrastructure: importing and using the product
    package (and its distributed module) must not load `oracle` or `synth`,
    and the package sources never mention them in an import."""
    import glob as _glob
    code = (
        "import sys, build_native; build_native.build();"
        "import paper_1202_6575_b200, paper_1202_6575_b200.distributed;"
        "bad = [m for m in sys.modules if m == 'oracle' or m.startswith('oracle.') or m == 'synth'];"
        "print(bad); sys.exit(1 if bad else 0)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    for f in _glob.glob(os.path.join(ROOT, "paper_1202_6575_b200", "**", "*.py"), recursive=True):
        src = open(f).read()
        assert not re.search(r"^\s*(import|from)\s+(oracle|synth)\b", src, flags=re.M), f


def test_oracle_and_cuda_sources_share_nothing():
    """No include or import crosses between oracle/ and the CUDA library."""
    inc = re.compile(r"^\s*(#\s*include|import|from)\s+\S*(paper_1202_6575_b200|sm_device|sm_kernels|stablemerge)",
                     flags=re.M)
    for f in _glob_all("oracle"):
        assert not inc.search(open(f).read()), f
    for f in _glob_all(os.path.join("paper_1202_6575_b200", "csrc")):
        assert not re.search(r"^\s*#\s*include\s+\S*oracle", open(f).read(), flags=re.M), f


def _glob_all(d):
    out = []
    for ext in ("*.c", "*.h", "*.cu", "*.cuh", "*.py"):
        out += glob.glob(os.path.join(ROOT, d, "**", ext), recursive=True)
    return out


def test_host_plan_from_ranks_matches_oracle_plan(sm):
    """The host's coarse Steps 3-4 (sm_plan_from_ranks: the partition of the
    host-buffer pipeline and of merges >= 2^31) equal oracle/plan.py's
    classification of the same cross ranks, task for task (PAPER.md
    L310-340; p = 5 is Fig. 1's), on random inputs incl. empty blocks."""
    import numpy as np
    from oracle import plan as P
    rng = np.random.default_rng(41)
    for trial in range(300):
        n, m = int(rng.integers(0, 60)), int(rng.integers(0, 60))
        p = int(rng.integers(1, 9)) if trial else 5
        K = int(rng.integers(1, 8))
        A = sorted(int(v) for v in rng.integers(0, K, n))
        B = sorted(int(v) for v in rng.integers(0, K, m))
        x, y, xbar, ybar, tasks = P.build_plan(A, B, p, p)
        got = sm.plan_from_ranks(n, m, p, xbar, ybar)
        want = sorted((t.a0, t.a1, t.b0, t.b1) for t in tasks)
        assert sorted(got) == want, (n, m, p, A, B)
        offs = [a0 + b0 for a0, a1, b0, b1 in got]
        assert offs == sorted(offs)


def test_host_plan_tasks_matches_oracle_plan(sm):
    """sm_plan_tasks -- the classification the device's K2 runs, compiled for
    the host with 64-bit indices (the sharded merge's Steps 3-4) -- equals
    oracle/plan.py task for task and in task order (A side, then B side),
    with p_A != p_B (reading R7), on Fig. 1 and random
    inputs with heavy ties and empty blocks."""
    import json
    import os
    import numpy as np
    from oracle import plan as P
    fig = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "fig1.json")))
    cases = [(fig["A"], fig["B"], 5, 5)]
    rng = np.random.default_rng(43)
    for _ in range(400):
        n, m = int(rng.integers(0, 70)), int(rng.integers(0, 70))
        K = int(rng.integers(1, 9))
        cases.append((sorted(int(v) for v in rng.integers(0, K, n)), sorted(int(v) for v in rng.integers(0, K, m)),
                      int(rng.integers(1, 10)), int(rng.integers(1, 10))))
    for A, B, pA, pB in cases:
        _, _, xbar, ybar, tasks = P.build_plan(A, B, pA, pB)
        got = sm.plan_tasks(len(A), len(B), pA, pB, xbar, ybar)
        assert got == [(t.a0, t.a1, t.b0, t.b1) for t in tasks], (A, B, pA, pB)
