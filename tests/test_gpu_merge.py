"""GPU parity of the stable merge (rows a0-a7) against the CPU oracle.

Bit-exact (keys and payloads) on seeded synthetic inputs of every BASELINE.json
merge config: at reduced sizes spanning many tiles with ragged tails, at the
full sizes in the launch configuration bench.py times, and on the edge cases.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import plan as P
from gpu_util import assert_bit_exact, gpu_merge, lib, oracle_merge

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
FIG1 = json.load(open(os.path.join(HERE, "golden", "fig1.json")))


# ------------------------------------------------------- plan (Steps 1-4)

def test_fig1_plan_on_device():
    sm = lib()
    A = torch.tensor(FIG1["A"], dtype=torch.int32, device="cuda")
    B = torch.tensor(FIG1["B"], dtype=torch.int32, device="cuda")
    xbar, ybar, tasks = sm.merge_plan(A, B, 5, 5)
    assert xbar.tolist() == FIG1["xbar"]
    assert ybar.tolist() == FIG1["ybar"]
    *_, otasks = P.build_plan(FIG1["A"], FIG1["B"], 5)
    assert tasks.cpu().numpy().tolist() == P.task_table(otasks).tolist()
    offs = (tasks[:, 2] + tasks[:, 4]).tolist()
    assert offs == [g["C"][0] for g in FIG1["tasks"]]


def test_fig1_merge_on_device():
    sm = lib()
    A = torch.tensor(FIG1["A"], dtype=torch.int32, device="cuda")
    B = torch.tensor(FIG1["B"], dtype=torch.int32, device="cuda")
    va = torch.arange(18, dtype=torch.int32, device="cuda")
    vb = (torch.arange(15, dtype=torch.int64, device="cuda") - (1 << 31)).to(torch.int32)
    for p in (1, 2, 3, 5, 8):
        ck, cv = sm.merge_stable(A, va, B, vb, p_A=p, p_B=p)
        assert ck.tolist() == FIG1["C_keys"]
        wk, wv = oracle.merge(A.cpu(), va.cpu(), B.cpu(), vb.cpu(), "i32")
        assert np.array_equal(oracle.vals_np(cv.cpu()), wv)


@pytest.mark.parametrize("kt,dist", [("i32", "bounded:7"), ("u32", "full"), ("i64", "bounded:1000"),
                                     ("u64", "mostly:0x8000000000000000:9/10")])
@pytest.mark.parametrize("pApB", [(1, 1), (3, 3), (17, 5), (64, 64), (1000, 7), (5, 999)])
def test_plan_parity_random(kt, dist, pApB):
    sm = lib()
    pA, pB = pApB
    inp = synth.merge_input(5003, 2999, kt, dist, seed=77 + pA, payload=False)
    a, b = oracle.as_np(inp.a_keys, kt), oracle.as_np(inp.b_keys, kt)
    x, y, oxbar, oybar, otasks = P.build_plan(a, b, pA, pB, vectorised=True)
    xbar, ybar, tasks = sm.merge_plan(inp.a_keys.cuda(), inp.b_keys.cuda(), pA, pB, key_type=kt)
    assert xbar.tolist() == oxbar and ybar.tolist() == oybar
    assert np.array_equal(tasks.cpu().numpy(), P.task_table(otasks))


@pytest.mark.parametrize("variant", [1, 2, 3])
@pytest.mark.parametrize("kt,dist", [("i32", "bounded:7"), ("u32", "full"), ("i64", "bounded:1000"),
                                     ("u64", "mostly:0x8000000000000000:9/10"), ("f32", "special"),
                                     ("f64", "special")])
def test_cross_ranks_every_k1_variant(kt, dist, variant):
    """x̄ / ȳ (Steps 1-2) of each cross-rank kernel forced
    in turn -- a warp per search, the shared-memory-sample kernel (every large
    plain merge), one thread per search (every sort round) -- equal the
    oracle plan's ranks, and so do the task tables, with p_A + p_B + 2 from
    a few to > 4096 searches."""
    sm = lib()
    try:
        sm.set_k1_variant(variant)
        for n, m, pA, pB in ((5003, 2999, 17, 5), (40000, 30001, 3000, 2501), (1, 9000, 1, 4500)):
            inp = synth.merge_input(n, m, kt, dist, seed=n + variant, payload=False)
            a, b = oracle.as_np(inp.a_keys, kt), oracle.as_np(inp.b_keys, kt)
            if kt.startswith("f"):                  # totalOrder ranks from the oracle's own search
                x, y = P.block_starts(n, pA), P.block_starts(m, pB)
                oxbar = [oracle.rank_low(a[x[i]], b, kt) if x[i] < n else m for i in range(pA)] + [m]
                oybar = [oracle.rank_high(b[y[j]], a, kt) if y[j] < m else n for j in range(pB)] + [n]
            else:
                _, _, oxbar, oybar, _ = P.build_plan(a, b, pA, pB, vectorised=True)
            xbar, ybar, tasks = sm.merge_plan(inp.a_keys.cuda(), inp.b_keys.cuda(), pA, pB, key_type=kt)
            assert xbar.tolist() == oxbar and ybar.tolist() == oybar, (n, m, pA, pB)
    finally:
        sm.set_k1_variant(0)


def test_cross_ranks_full_size_c2_sample_kernel():
    """BASELINE configs[1] at full size with p_A = p_B = 2^15: 65538 searches,
    so the automatic choice is the shared-memory-sample kernel; every x̄, ȳ
    equals numpy's searchsorted (rank_low = side left, rank_high = right)."""
    sm = lib()
    inp = synth.config_input(2, device="cuda")
    p = 1 << 15
    xbar, ybar, _ = sm.merge_plan(inp.a_keys, inp.b_keys, p, p, key_type="i32")
    a, b = inp.a_keys.cpu().numpy(), inp.b_keys.cpu().numpy()
    x = np.asarray(P.block_starts(a.size, p)[:-1])
    y = np.asarray(P.block_starts(b.size, p)[:-1])
    assert np.array_equal(xbar.cpu().numpy()[:-1], np.searchsorted(b, a[x], side="left"))
    assert np.array_equal(ybar.cpu().numpy()[:-1], np.searchsorted(a, b[y], side="right"))
    assert int(xbar[-1]) == b.size and int(ybar[-1]) == a.size


def _one_launch(sm, n, m, kt="u32", payload=True):
    """The library's rule for a one-launch small merge: at most 8 tasks per
    resident K2 CTA (two per SM for <= 8-byte elements)."""
    T = sm.tile_capacity(kt, payload) // 2
    tasks = max(1, -(-n // T)) + max(1, -(-m // T))
    return tasks <= 8 * 2 * torch.cuda.get_device_properties(0).multi_processor_count


@pytest.mark.parametrize("small_fuse", [True, False])
def test_launches_per_device_merge(small_fuse):
    """A device merge has exactly one synchronisation between Steps 1-2 and
    the tasks (SURVEY §2.2 acceptance 6): two launches, K1
    then K2 behind it (PDL griddepcontrol.wait); or, for a small merge, ONE
    launch in which every CTA computes the ranks its own tasks read before
    classifying them.  Either way, the oracle's merge."""
    sm = lib()
    try:
        sm.set_small_fuse(small_fuse)
        for n, m in ((1 << 20, 1 << 20), (5000, 3), (1 << 23, 1 << 16), (3 << 20, 3 << 20)):
            inp = synth.merge_input(n, m, "u32", "full", seed=n, payload=True)
            d = inp.to("cuda")
            ck, cv = sm.merge_stable(d.a_keys, d.a_vals, d.b_keys, d.b_vals, key_type="u32")
            assert sm.last_launch_count() == (1 if small_fuse and _one_launch(sm, n, m) else 2), (n, m)
            torch.cuda.synchronize()
            assert_bit_exact(ck.cpu(), cv.cpu(), *oracle_merge(inp), "u32")
    finally:
        sm.set_small_fuse(False)


@pytest.mark.parametrize("small_fuse", [True, False])
@pytest.mark.parametrize("kt,dist,payload", [("i32", "full", False), ("u32", "bounded:3", True),
                                             ("u32", "bounded:65536", True), ("i64", "bounded:1000", True),
                                             ("u64", "mostly:7:9/10", True), ("f32", "special", True),
                                             ("f64", "bounded:50", False), ("u128", "tuple:5", True)])
@pytest.mark.parametrize("nm", [(1, 0), (0, 7), (5, 3), (1921, 3839), (70001, 12345), (3, 200003),
                                (1_000_003, 999_999), (2_000_000, 4099), (17, 2_000_000), (1 << 20, 1 << 20)])
def test_small_merge_one_launch_parity(small_fuse, kt, dist, payload, nm):
    """One-launch small merges (each CTA ranks its own tasks: balanced,
    unbalanced -- where the other side's entries come from the second round
    of searches -- and degenerate sizes) and the two-launch path give the
    oracle's merge, bit for bit."""
    sm = lib()
    n, m = nm
    inp = synth.merge_input(n, m, kt, dist, seed=n + 3 * m + small_fuse, payload=payload)
    try:
        sm.set_small_fuse(small_fuse)
        got = gpu_merge(sm, inp)
        got_desc = None
        if kt in ("u32", "i64"):
            dinp = synth.merge_input(n, m, kt, dist, seed=n + 5 * m, payload=payload, descending=True)
            got_desc = (gpu_merge(sm, dinp, descending=True), dinp)
    finally:
        sm.set_small_fuse(False)
    assert_bit_exact(*got, *oracle_merge(inp), kt)
    if got_desc is not None:
        (gk, gv), dinp = got_desc
        want = oracle.merge(dinp.a_keys, dinp.a_vals, dinp.b_keys, dinp.b_vals, kt, descending=True)
        assert_bit_exact(gk, gv, *want, kt)


def test_plan_parity_exhaustive_small():
    sm = lib()
    import itertools
    seqs = [list(c) for L in range(5) for c in itertools.combinations_with_replacement(range(3), L)]
    for a in seqs[::3]:
        for b in seqs[::2]:
            for p in (1, 2, 3, 5):
                A = torch.tensor(a, dtype=torch.int32, device="cuda")
                B = torch.tensor(b, dtype=torch.int32, device="cuda")
                xbar, ybar, tasks = sm.merge_plan(A, B, p, p)
                _, _, oxbar, oybar, otasks = P.build_plan(a, b, p)
                assert xbar.tolist() == oxbar and ybar.tolist() == oybar
                assert tasks.cpu().numpy().tolist() == P.task_table(otasks).tolist()


# --------------------------------------------------- merge parity (small)

@pytest.mark.parametrize("cfg,scale", [(1, 16), (1, 1), (2, 256), (3, 256), (4, 128)])
def test_config_merge_reduced(cfg, scale):
    sm = lib()
    inp = synth.config_input(cfg, scale=scale)
    want = oracle_merge(inp)
    got = gpu_merge(sm, inp)
    assert_bit_exact(*got, *want, inp.key_type)


@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
@pytest.mark.parametrize("nm", [(1, 0), (0, 1), (1, 1), (5, 3), (959, 961), (1920, 1), (1921, 3839),
                                (70001, 12345), (12345, 70001), (100000, 17), (3, 200003)])
@pytest.mark.parametrize("payload", [True, False])
def test_merge_ragged(kt, nm, payload):
    sm = lib()
    n, m = nm
    for dist in ("bounded:3", "full"):
        inp = synth.merge_input(n, m, kt, dist, seed=n * 31 + m, payload=payload)
        assert_bit_exact(*gpu_merge(sm, inp), *oracle_merge(inp), kt)


@pytest.mark.parametrize("kt,payload", [("u32", True), ("i32", False)])
def test_merge_tile_boundaries(kt, payload):
    """Sizes around the block size T and the tile capacity NV = 2T of the
    layout actually used (they differ per key width / payload mode)."""
    sm = lib()
    nv = sm.tile_capacity(kt, payload)
    T = nv // 2
    for n, m in ((T, T), (T + 1, T - 1), (2 * T, 1), (nv - 1, nv + 1), (3 * T + 7, 5 * T - 3), (nv * 4, 3)):
        inp = synth.merge_input(n, m, kt, "bounded:40", seed=n + 7 * m, payload=payload)
        assert_bit_exact(*gpu_merge(sm, inp), *oracle_merge(inp), kt)
        inp = synth.merge_input(n, m, kt, "full", seed=n + 11 * m, payload=payload)
        assert_bit_exact(*gpu_merge(sm, inp, p_A=max(1, -(-n // T)), p_B=max(1, -(-m // T))),
                         *oracle_merge(inp), kt)


@pytest.mark.parametrize("block", [1, 2, 7, 32, 257, 960])
def test_merge_metamorphic_block_size(block):
    """Output must not depend on the tuning (T, p_A vs p_B) -- S:L262."""
    sm = lib()
    inp = synth.merge_input(30011, 20011, "u32", "bounded:50", seed=5)
    want = oracle_merge(inp)
    assert_bit_exact(*gpu_merge(sm, inp, block=block), *want, "u32")
    assert_bit_exact(*gpu_merge(sm, inp, block=block, pdl=False), *want, "u32")


def test_merge_paper_single_p():
    sm = lib()
    inp = synth.merge_input(50000, 30000, "i64", "bounded:100", seed=9)
    want = oracle_merge(inp)
    for p in (60, 100, 1000):
        assert_bit_exact(*gpu_merge(sm, inp, p_A=p, p_B=p), *want, "i64")


def test_merge_repeatable():
    sm = lib()
    inp = synth.config_input(1, scale=4).to("cuda")
    r1 = sm.merge_stable(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, key_type="u32")
    r2 = sm.merge_stable(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, key_type="u32")
    assert torch.equal(r1[0], r2[0]) and torch.equal(r1[1], r2[1])


# ------------------------------------------------------------- edge cases

def _mk(a, b, kt):
    dt = {"u32": np.uint32, "i32": np.int32, "i64": np.int64, "u64": np.uint64}[kt]
    a = np.sort(np.array(a, dtype=dt)); b = np.sort(np.array(b, dtype=dt))
    ct = torch.int32 if kt in ("u32", "i32") else torch.int64
    A = torch.from_numpy(a.view(np.int32 if ct == torch.int32 else np.int64).copy())
    B = torch.from_numpy(b.view(np.int32 if ct == torch.int32 else np.int64).copy())
    va, vb = synth.source_payloads(len(a), len(b))
    return synth.MergeInput(kt, A, B, va, vb)


@pytest.mark.parametrize("case", ["all_equal", "a_below_b", "a_above_b", "extremes", "interleaved_ties"])
@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64"])
def test_merge_edge_cases(case, kt):
    sm = lib()
    big = 5000
    info = np.iinfo({"u32": np.uint32, "i32": np.int32, "i64": np.int64, "u64": np.uint64}[kt])
    if case == "all_equal":
        a, b = [7] * big, [7] * (big // 2 + 3)
    elif case == "a_below_b":
        a, b = list(range(big)), list(range(big, 2 * big + 11))
    elif case == "a_above_b":
        a, b = list(range(big, 2 * big + 11)), list(range(big))
    elif case == "extremes":
        a = [info.min] * 1000 + [info.max] * 1001 + [0] * 17
        b = [info.min] * 999 + [info.max] * 3000 + [1] * 5
    else:
        a = [i // 3 for i in range(3 * big)]
        b = [i // 2 for i in range(2 * big)]
    inp = _mk(a, b, kt)
    assert_bit_exact(*gpu_merge(sm, inp), *oracle_merge(inp), kt)
    if case == "all_equal":   # P7: C = A || B
        _, cv = gpu_merge(sm, inp)
        assert cv.tolist() == inp.a_vals.tolist() + inp.b_vals.tolist()


def test_merge_empty_both():
    sm = lib()
    e = torch.empty(0, dtype=torch.int32, device="cuda")
    ck, cv = sm.merge_stable(e, e, e, e)
    assert ck.numel() == 0 and cv.numel() == 0


def test_merge_host_buffers():
    """The C ABI accepts host (pinned or pageable) buffers and stages them."""
    sm = lib()
    inp = synth.config_input(4, scale=512)
    want = oracle_merge(inp)
    got = sm.merge_stable(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, key_type="u64")
    assert_bit_exact(*got, *want, "u64")
    pin = lambda t: t.pin_memory()
    out_k = torch.empty(inp.n + inp.m, dtype=torch.int64).pin_memory()
    out_v = torch.empty(inp.n + inp.m, dtype=torch.int32).pin_memory()
    got = sm.merge_stable(pin(inp.a_keys), pin(inp.a_vals), pin(inp.b_keys), pin(inp.b_vals), out_k, out_v,
                          key_type="u64")
    assert_bit_exact(*got, *want, "u64")


@pytest.mark.parametrize("kt,payload,dist", [("i32", False, "full"), ("u32", True, "bounded:65536"),
                                             ("u64", True, "mostly:0x8000000000000000:9/10"),
                                             ("i64", True, "equal")])
@pytest.mark.parametrize("pinned", [True, False])
def test_merge_host_pipelined(kt, payload, dist, pinned):
    """Host inputs above the pipelining threshold (>= 64 MB): the library
    cuts the call into sub-merges with the paper's Steps 1-4 on the host and
    streams them over three CUDA streams -- same bytes as the oracle."""
    sm = lib()
    eb = synth.elem_bytes(kt, payload)
    n = (100 << 20) // eb // 2 + 12345
    m = (100 << 20) // eb // 2 - 999
    inp = synth.merge_input(n, m, kt, dist, seed=4242, payload=payload)
    want = oracle_merge(inp)
    f = (lambda t: None if t is None else t.pin_memory()) if pinned else (lambda t: t)
    got = sm.merge_stable(f(inp.a_keys), f(inp.a_vals), f(inp.b_keys), f(inp.b_vals), key_type=kt)
    assert_bit_exact(*got, *want, kt)


@pytest.mark.parametrize("cfg,scale", [(1, 4), (2, 64), (3, 64), (4, 32)])
def test_merge_path_comparison_same_bytes(cfg, scale):
    """The merge-path comparison variant produces the
    same unique stable merge."""
    sm = lib()
    inp = synth.config_input(cfg, scale=scale)
    assert_bit_exact(*gpu_merge(sm, inp, merge_path=True), *oracle_merge(inp), inp.key_type)


@pytest.mark.parametrize("nm", [(1, 0), (0, 1), (5, 3), (8095, 8097), (20000, 1), (3, 70001)])
def test_merge_path_comparison_ragged(nm):
    sm = lib()
    for kt in ("i32", "u64"):
        inp = synth.merge_input(*nm, kt, "bounded:3", seed=sum(nm), payload=kt == "u64")
        assert_bit_exact(*gpu_merge(sm, inp, merge_path=True), *oracle_merge(inp), kt)


@pytest.mark.parametrize("kt", ["f32", "f64"])
@pytest.mark.parametrize("dist", ["special", "full", "bounded:9"])
def test_merge_float_total_order(kt, dist):
    """Floating-point keys: IEEE totalOrder, NaNs, signed
    zeros, infinities and subnormals -- bit-exact against the oracle, on the
    device path, the merge-path comparison and the pipelined host path."""
    sm = lib()
    inp = synth.merge_input(70001, 50003, kt, dist, seed=23, payload=True)
    want = oracle_merge(inp)
    assert_bit_exact(*gpu_merge(sm, inp), *want, kt)
    assert_bit_exact(*gpu_merge(sm, inp, merge_path=True), *want, kt)
    big = synth.merge_input((40 << 20) // 12, (30 << 20) // 12, kt, dist, seed=24, payload=True)
    got = sm.merge_stable(big.a_keys.pin_memory(), big.a_vals.pin_memory(), big.b_keys.pin_memory(),
                          big.b_vals.pin_memory(), key_type=kt)
    assert_bit_exact(*got, *oracle_merge(big), kt)


@pytest.mark.parametrize("kt,payload", [("u32", True), ("i32", False), ("u64", True), ("f32", True)])
@pytest.mark.parametrize("merge_path", [False, True])
def test_unsorted_inputs_never_write_outside_output(kt, payload, merge_path):
    """The header's promise for a violated precondition (unsorted A or B):
    unspecified output, but no write outside C (guard zones on both sides;
    compute-sanitizer is closed on this pool, so the guard is the check)."""
    sm = lib()
    n, m = 70001, 50003
    ct = synth.KEY_TYPES[kt][0]
    a = synth._keys("full" if kt != "f32" else "special", kt, 91, 1, n, "cpu").cuda()   # NOT sorted
    b = synth._keys("full" if kt != "f32" else "special", kt, 91, 2, m, "cpu").cuda()
    va = torch.arange(n, dtype=torch.int32, device="cuda") if payload else None
    vb = torch.arange(m, dtype=torch.int32, device="cuda") if payload else None
    G = 4096
    kbuf = torch.full((n + m + 2 * G,), 77, dtype=ct, device="cuda")
    vbuf = torch.full((n + m + 2 * G,), 77, dtype=torch.int32, device="cuda") if payload else None
    sm.merge_stable(a, va, b, vb, kbuf[G:G + n + m], None if vbuf is None else vbuf[G:G + n + m], key_type=kt,
                    merge_path=merge_path)
    torch.cuda.synchronize()
    assert bool((kbuf[:G] == 77).all()) and bool((kbuf[G + n + m:] == 77).all())
    if payload:
        assert bool((vbuf[:G] == 77).all()) and bool((vbuf[G + n + m:] == 77).all())


def test_unsorted_host_inputs_pipelined_path_terminates_in_bounds():
    """Unsorted host inputs above the pipelining threshold: the host plan's
    tasks are clamped, the call terminates, nothing outside C is written."""
    sm = lib()
    n, m = (40 << 20) // 4, (36 << 20) // 4
    a = synth._keys("full", "i32", 5, 1, n, "cpu").pin_memory()
    b = synth._keys("full", "i32", 5, 2, m, "cpu").pin_memory()
    G = 4096
    buf = torch.full((n + m + 2 * G,), 77, dtype=torch.int32).pin_memory()
    sm.merge_stable(a, None, b, None, buf[G:G + n + m], key_type="i32")
    assert bool((buf[:G] == 77).all()) and bool((buf[G + n + m:] == 77).all())


def test_merge_errors():
    sm = lib()
    a = torch.arange(100, dtype=torch.int32, device="cuda")
    with pytest.raises(sm.StableMergeError) as e:
        sm.merge_stable(a, None, a, None, out_keys=a.new_empty(200), block=100000)
    assert e.value.status == 1
    out = torch.empty(300, dtype=torch.int32, device="cuda")
    with pytest.raises(sm.StableMergeError) as e:      # output overlaps input
        sm.merge_stable(out[:100], None, a, None, out_keys=out[50:250])
    assert e.value.status == 2
    with pytest.raises(sm.StableMergeError) as e:      # tile bound violated by explicit p
        sm.merge_stable(torch.arange(20000, dtype=torch.int32, device="cuda"), None, a, None, p_A=1, p_B=1)
    assert e.value.status == 1


# ----------------------------------------------------- full-size parity

@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
def test_config_merge_full_size(cfg):
    """BASELINE.json sizes, default launch configuration (as bench.py times it):
    the whole output against the oracle's merge, bit for bit."""
    sm = lib()
    dev = synth.config_input(cfg, device="cuda")
    ck, cv = sm.merge_stable(dev.a_keys, dev.a_vals, dev.b_keys, dev.b_vals, key_type=dev.key_type)
    torch.cuda.synchronize()
    host = dev.to("cpu")
    del dev
    want_k, want_v = oracle_merge(host)
    assert_bit_exact(ck.cpu(), None if cv is None else cv.cpu(), want_k, want_v, host.key_type)


@pytest.mark.parametrize("kt", ["u32", "i64", "f32", "u64"])
@pytest.mark.parametrize("shift", [(1, 3, 5, 7, 2, 9), (2, 1, 1, 3, 3, 1)])
def test_merge_misaligned_views(kt, shift):
    """Inputs, outputs and payloads as tensor views at element offsets that
    are not 16-byte aligned: the TMA loads read 16-byte supersets inside the
    same allocations and the stores write exactly the output range."""
    sm = lib()
    inp = synth.merge_input(70001, 50003, kt, "bounded:1000", seed=41, payload=True)
    sa, sb, sc, sva, svb, svc = shift
    ct = synth.KEY_TYPES[kt][0]

    def view(t, s):
        base = torch.zeros(t.numel() + s + 8, dtype=t.dtype, device="cuda")
        v = base[s:s + t.numel()]
        v.copy_(t.cuda())
        return base, v

    ba, a = view(inp.a_keys, sa)
    bb, b = view(inp.b_keys, sb)
    bva, va = view(inp.a_vals, sva)
    bvb, vb = view(inp.b_vals, svb)
    bc = torch.full((inp.n + inp.m + sc + 8,), -1, dtype=ct, device="cuda")
    bvc = torch.full((inp.n + inp.m + svc + 8,), -1, dtype=torch.int32, device="cuda")
    c, vc = bc[sc:sc + inp.n + inp.m], bvc[svc:svc + inp.n + inp.m]
    sm.merge_stable(a, va, b, vb, c, vc, key_type=kt)
    torch.cuda.synchronize()
    assert_bit_exact(c.cpu(), vc.cpu(), *oracle_merge(inp), kt)
    # nothing written outside the output views
    assert bool((bc[:sc] == -1).all()) and bool((bc[sc + inp.n + inp.m:] == -1).all())
    assert bool((bvc[:svc] == -1).all()) and bool((bvc[svc + inp.n + inp.m:] == -1).all())


def test_merges_on_side_streams_concurrently():
    """The library is stream-ordered: calls on two side streams (torch's
    current stream, picked up by the binding) run concurrently and each is
    complete after its own stream synchronises."""
    sm = lib()
    inps = [synth.merge_input(2_000_003, 1_500_007, kt, "full", seed=i, payload=True).to("cuda")
            for i, kt in enumerate(("u32", "i64"))]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    torch.cuda.synchronize()
    for inp, st in zip(inps, streams):
        with torch.cuda.stream(st):
            outs.append(sm.merge_stable(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, key_type=inp.key_type))
    for (ck, cv), inp, st in zip(outs, inps, streams):
        st.synchronize()
        cpu = inp.to("cpu")
        assert_bit_exact(ck.cpu(), cv.cpu(), *oracle.merge(cpu.a_keys, cpu.a_vals, cpu.b_keys, cpu.b_vals,
                                                           inp.key_type), inp.key_type)


def test_concurrent_merges_dynamic_task_assignment():
    """Two merges large enough for K2's task counter (more than 8 tasks per
    resident CTA) on two side streams at once: each call's counter is its
    own (per-call scratch), so the concurrent K2 grids never take each
    other's tasks -- both the oracle's merge."""
    sm = lib()
    inps = [synth.merge_input((1 << 23) + 5, (1 << 23) - 3, "i32", "full", seed=20 + i, payload=False).to("cuda")
            for i in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    torch.cuda.synchronize()
    outs = []
    for rep in range(3):
        outs = []
        for inp, st in zip(inps, streams):
            with torch.cuda.stream(st):
                outs.append(sm.merge_stable(inp.a_keys, None, inp.b_keys, None, key_type="i32"))
        for st in streams:
            st.synchronize()
    for (ck, _), inp in zip(outs, inps):
        cpu = inp.to("cpu")
        assert_bit_exact(ck.cpu(), None, *oracle.merge(cpu.a_keys, None, cpu.b_keys, None, "i32"), "i32")


@pytest.mark.parametrize("kt,payload", [("i32", False), ("u32", True), ("i64", True), ("f32", False)])
def test_chained_merges_search_ahead(kt, payload):
    """Back-to-back calls on one stream where the second merge reads what the
    first one writes (pre-filled with zeros, so a kernel that read its inputs
    ahead of the stream order -- K1 and K2 are chained by programmatic
    dependent launches -- would rank against wrong data): both outputs must be
    the oracle's, every time.  Also the regression test of the search-ahead
    experiment (scripts/experiments/k1_search_ahead.patch)."""
    sm = lib()
    n = 1 << 23
    a = synth.merge_input(n, n, kt, "full", seed=5, payload=payload)
    d2 = synth.merge_input(2 * n, 2 * n, kt, "full", seed=6, payload=payload)   # its B is merge 2's B
    da, dd = a.to("cuda"), d2.to("cuda")
    w1k, w1v = oracle_merge(a)
    w1k_t = torch.from_numpy(np.ascontiguousarray(w1k).view({4: np.int32, 8: np.int64}[w1k.dtype.itemsize]))
    w1v_t = None if w1v is None else torch.from_numpy(np.ascontiguousarray(w1v).view(np.int32))
    w2k, w2v = oracle.merge(w1k_t, w1v_t, d2.b_keys, d2.b_vals, kt)
    c1k = torch.empty(2 * n, dtype=da.a_keys.dtype, device="cuda")
    c1v = torch.empty(2 * n, dtype=torch.int32, device="cuda") if payload else None
    c2k = torch.empty(4 * n, dtype=da.a_keys.dtype, device="cuda")
    c2v = torch.empty(4 * n, dtype=torch.int32, device="cuda") if payload else None
    for rep in range(6):
        c1k.zero_()
        if payload:
            c1v.zero_()
        sm.merge_stable(da.a_keys, da.a_vals, da.b_keys, da.b_vals, c1k, c1v, key_type=kt)
        sm.merge_stable(c1k, c1v, dd.b_keys, dd.b_vals, c2k, c2v, key_type=kt)
        if rep % 2:                                  # a third call queued behind, reading the first's output again
            sm.merge_stable(c1k, c1v, dd.b_keys, dd.b_vals, c2k, c2v, key_type=kt)
        torch.cuda.synchronize()
        assert_bit_exact(c1k.cpu(), None if c1v is None else c1v.cpu(), w1k, w1v, kt)
        assert_bit_exact(c2k.cpu(), None if c2v is None else c2v.cpu(), w2k, w2v, kt)


@pytest.mark.parametrize("kt,payload,dist", [("u32", True, "bounded:65536"), ("f32", True, "special"),
                                             ("i32", True, "full"), ("i64", False, "bounded:1000"),
                                             ("u64", False, "mostly:7:9/10"), ("f64", False, "full")])
@pytest.mark.parametrize("nm", [((1 << 22) + 5, (1 << 22) - 5), ((1 << 23) + 12345, 70001), (333, (1 << 23) + 77)])
def test_large_default_merges_take_the_large_shape(kt, payload, dist, nm):
    """Default plain merges of >= 2^23 elements with 8-byte slots run K2 with
    its large tile (512 x 17 / 448 x 17 at one CTA per SM): the
    oracle's merge, bit for bit, and the same as with an explicit block size
    (which keeps the small shape)."""
    sm = lib()
    n, m = nm
    inp = synth.merge_input(n, m, kt, dist, seed=n % 1000 + m % 7, payload=payload)
    want = oracle_merge(inp)
    assert_bit_exact(*gpu_merge(sm, inp), *want, kt)
    assert_bit_exact(*gpu_merge(sm, inp, block=sm.tile_capacity(kt, payload) // 2), *want, kt)
    if kt in ("u32", "i64"):
        dinp = synth.merge_input(n, m, kt, dist, seed=n % 1000 + 3, payload=payload, descending=True)
        gk, gv = gpu_merge(sm, dinp, descending=True)
        assert_bit_exact(gk, gv, *oracle.merge(dinp.a_keys, dinp.a_vals, dinp.b_keys, dinp.b_vals, kt,
                                               descending=True), kt)
