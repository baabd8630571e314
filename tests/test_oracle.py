"""Pins for the CPU oracle (`oracle/`), run with -m "not gpu".

Each test ties an oracle function to something other than itself: the values
PAPER.md prints for its worked example (tests/golden/fig1.json), brute force
(Python's stable `sorted` of the tagged concatenation), the closed form of
PAPER.md L158-166, linear-scan counts, exhaustive small instances, and the
plan invariants of §2.
"""
import itertools
import json
import os
import random

import numpy as np
import pytest

from oracle import plan as P

HERE = os.path.dirname(os.path.abspath(__file__))
FIG1 = json.load(open(os.path.join(HERE, "golden", "fig1.json")))


def nondecreasing(max_len, alphabet):
    for L in range(max_len + 1):
        yield from (list(c) for c in itertools.combinations_with_replacement(range(alphabet), L))


def brute_merge(a, b):
    """Stable sort of the tagged concatenation A||B: A elements come first in
    the concatenation, so a stable sort keeps A before B on equal keys."""
    tagged = [(k, ("A", i)) for i, k in enumerate(a)] + [(k, ("B", j)) for j, k in enumerate(b)]
    return sorted(tagged, key=lambda e: e[0])


# ---------------------------------------------------------------- Fig. 1 (P1)

def test_fig1_block_starts():
    A, B, p = FIG1["A"], FIG1["B"], FIG1["p"]
    assert P.block_starts(len(A), p) == FIG1["x"]
    assert P.block_starts(len(B), p) == FIG1["y"]


def test_fig1_cross_ranks():
    A, B, p = FIG1["A"], FIG1["B"], FIG1["p"]
    for vec in (False, True):
        x, y, xbar, ybar = P.cross_ranks(A, B, p, p, vectorised=vec)
        assert xbar == FIG1["xbar"]
        assert ybar == FIG1["ybar"]


def test_fig1_tasks_match_caption():
    A, B, p = FIG1["A"], FIG1["B"], FIG1["p"]
    *_, tasks = P.build_plan(A, B, p)
    assert len(tasks) == 2 * p
    for t, g in zip(tasks, FIG1["tasks"]):
        assert t.side == g["side"], g["cite"]
        if g["case"] is not None:
            assert t.case == g["case"], g["cite"]
        ga = (g["A"][0], g["A"][1] + 1) if g["A"] else None
        gb = (g["B"][0], g["B"][1] + 1) if g["B"] else None
        assert ((t.a0, t.a1) if t.a1 > t.a0 else None) == ga, g["cite"]
        assert ((t.b0, t.b1) if t.b1 > t.b0 else None) == gb, g["cite"]
        assert (t.off, t.off + t.size - 1) == tuple(g["C"]), g["cite"]


def test_fig1_merge_and_positions(orc):
    A, B = np.array(FIG1["A"], np.int32), np.array(FIG1["B"], np.int32)
    va = np.arange(len(A), dtype=np.uint32)
    vb = (np.arange(len(B)) | (1 << 31)).astype(np.uint32)
    c, vc = orc.merge(A, va, B, vb, "i32")
    assert c.tolist() == FIG1["C_keys"]
    # O4: every input element of a caption task lands inside that task's C range.
    pa, pb = orc.positions(A, B, "i32")
    for g in FIG1["tasks"]:
        lo, hi = g["C"]
        if g["A"]:
            assert all(lo <= pa[i] <= hi for i in range(g["A"][0], g["A"][1] + 1)), g["cite"]
        if g["B"]:
            assert all(lo <= pb[j] <= hi for j in range(g["B"][0], g["B"][1] + 1)), g["cite"]
    # the caption's copies fix positions exactly
    assert pa[:5].tolist() == [0, 1, 2, 3, 4] and pa[8] == 14
    assert pb[3:6].tolist() == [11, 12, 13] and pb[12:15].tolist() == [30, 31, 32]
    # and the payload at those positions is the element itself
    assert vc[pa].tolist() == va.tolist() and vc[pb].tolist() == vb.tolist()


def test_fig1_executed_plan_equals_merge(orc):
    A, B, p = FIG1["A"], FIG1["B"], FIG1["p"]
    *_, tasks = P.build_plan(A, B, p)
    tagA = [(k, "A", i) for i, k in enumerate(A)]
    tagB = [(k, "B", j) for j, k in enumerate(B)]
    C = P.execute_plan(tasks, tagA, tagB)
    assert [e[0] for e in C] == FIG1["C_keys"]
    assert [(e[0], (e[1], e[2])) for e in C] == brute_merge(A, B)


# ------------------------------------------------ O1 / O4 against brute force

def test_merge_exhaustive_vs_brute_force(orc):
    seqs = list(nondecreasing(5, 3))
    assert len(seqs) == 56
    for a in seqs:
        for b in seqs:
            A, B = np.array(a, np.int32), np.array(b, np.int32)
            va = np.arange(len(a), dtype=np.uint32)
            vb = (np.arange(len(b)) | (1 << 31)).astype(np.uint32)
            c, vc = orc.merge(A, va, B, vb, "i32")
            want = brute_merge(a, b)
            assert c.tolist() == [k for k, _ in want]
            assert vc.tolist() == [t[1] if t[0] == "A" else (1 << 31) | t[1] for _, t in want]


@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64"])
def test_merge_random_vs_sorted(orc, kt):
    rng = np.random.default_rng(7)
    dt = orc.NP_DTYPES[kt]
    info = np.iinfo(dt)
    for trial in range(60):
        n, m = int(rng.integers(0, 300)), int(rng.integers(0, 300))
        if trial % 3 == 0:   # few distinct values -> many cross ties
            a = np.sort(rng.integers(0, 4, n).astype(dt)); b = np.sort(rng.integers(0, 4, m).astype(dt))
        else:                # full range incl. sign/top bit
            a = np.sort(rng.integers(info.min, info.max, n, dtype=dt, endpoint=True))
            b = np.sort(rng.integers(info.min, info.max, m, dtype=dt, endpoint=True))
        va = np.arange(n, dtype=np.uint32)
        vb = (np.arange(m) | (1 << 31)).astype(np.uint32)
        c, vc = orc.merge(a, va, b, vb, kt)
        want = brute_merge([int(v) for v in a], [int(v) for v in b])
        assert [int(v) for v in c] == [k for k, _ in want]
        assert vc.tolist() == [t[1] if t[0] == "A" else (1 << 31) | t[1] for _, t in want]
        # keys-only mode gives the same keys
        c2, vc2 = orc.merge(a, None, b, None, kt)
        assert vc2 is None and np.array_equal(c, c2)


@pytest.mark.parametrize("kt", ["u32", "i64", "u64"])
def test_positions_closed_form_is_bijection_onto_merge(orc, kt):
    rng = np.random.default_rng(11)
    dt = orc.NP_DTYPES[kt]
    for _ in range(40):
        n, m = int(rng.integers(0, 200)), int(rng.integers(0, 200))
        a = np.sort(rng.integers(0, 9, n).astype(dt)); b = np.sort(rng.integers(0, 9, m).astype(dt))
        va = np.arange(n, dtype=np.uint32)
        vb = (np.arange(m) | (1 << 31)).astype(np.uint32)
        c, vc = orc.merge(a, va, b, vb, kt)
        pa, pb = orc.positions(a, b, kt)
        allpos = np.concatenate([pa, pb])
        assert np.array_equal(np.sort(allpos), np.arange(n + m))
        assert np.array_equal(vc[pa], va) and np.array_equal(vc[pb], vb)
        ia = rng.integers(0, max(n, 1), 7) if n else np.zeros(0, np.int64)
        jb = rng.integers(0, max(m, 1), 7) if m else np.zeros(0, np.int64)
        sa, sb = orc.positions_sample(a, b, kt, ia, jb)
        assert np.array_equal(sa, pa[ia]) and np.array_equal(sb, pb[jb])


@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64"])
def test_ranks_vs_linear_count(orc, kt):
    rng = np.random.default_rng(3)
    dt = orc.NP_DTYPES[kt]
    info = np.iinfo(dt)
    for _ in range(50):
        X = np.sort(rng.integers(info.min, info.max, int(rng.integers(0, 40)), dtype=dt, endpoint=True))
        if rng.random() < 0.5 and X.size:
            X = np.sort(np.concatenate([X, np.repeat(X[rng.integers(0, X.size)], 5)]))
        probes = list(X[:5]) + [info.min, info.max] + list(rng.integers(info.min, info.max, 5, dtype=dt))
        for v in probes:
            lo = sum(1 for e in X if e < v)
            hi = sum(1 for e in X if e <= v)
            assert orc.rank_low(v, X, kt) == lo == P.rank_low(v, list(X))
            assert orc.rank_high(v, X, kt) == hi == P.rank_high(v, list(X))


def test_rank_examples_from_paper():
    A, B = FIG1["A"], FIG1["B"]
    assert P.rank_low(5, B) == 7 and P.rank_low(0, B) == 0          # x̄_3, x̄_0 (Fig. 1)
    assert P.rank_high(1, A) == 5 and P.rank_high(7, A) == 18       # ȳ_0, ȳ_4 (Fig. 1)
    assert P.rank_low(3, []) == 0 and P.rank_high(3, []) == 0


# --------------------------------------------------------------- O2 the sort

@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64"])
def test_sort_vs_python_stable_sorted(orc, kt):
    rng = np.random.default_rng(5)
    dt = orc.NP_DTYPES[kt]
    info = np.iinfo(dt)
    for trial in range(40):
        N = int(rng.integers(0, 700))
        if trial % 2:
            k = rng.integers(0, 6, N).astype(dt)
        else:
            k = rng.integers(info.min, info.max, N, dtype=dt, endpoint=True)
        v = np.arange(N, dtype=np.uint32)
        sk, sv = orc.sort(k, v, kt)
        want = sorted(range(N), key=lambda i: int(k[i]))       # Python's sort is stable
        assert sv.tolist() == want
        assert [int(e) for e in sk] == [int(k[i]) for i in want]
        sk2, _ = orc.sort(k, None, kt)
        assert np.array_equal(sk, sk2)


def test_sort_exhaustive_small(orc):
    for N in range(8):
        for k in itertools.product(range(3), repeat=N):
            kk = np.array(k, np.uint32)
            sk, sv = orc.sort(kk, np.arange(N, dtype=np.uint32), "u32")
            assert sv.tolist() == sorted(range(N), key=lambda i: k[i])


# ------------------------------------------------------ O3 the paper's plan

def check_plan(A, B, pA, pB, tasks, x, y, xbar, ybar):
    n, m = len(A), len(B)
    # monotone, bounded cross ranks
    assert all(xbar[i] <= xbar[i + 1] for i in range(pA)) and 0 <= xbar[0] and xbar[pA] == m
    assert all(ybar[j] <= ybar[j + 1] for j in range(pB)) and 0 <= ybar[0] and ybar[pB] == n
    # non-crossing (reading R10): y_j < xbar_i  <=>  ybar_j <= x_i
    for i in range(pA):
        for j in range(pB):
            if x[i] < n and y[j] < m:
                assert (y[j] < xbar[i]) == (ybar[j] <= x[i])
    # output tiling, input partition, size bound
    outs = sorted((t.off, t.off + t.size) for t in tasks if t.size)
    pos = 0
    for lo, hi in outs:
        assert lo == pos
        pos = hi
    assert pos == n + m
    for lo_attr, hi_attr, L in (("a0", "a1", n), ("b0", "b1", m)):
        rs = sorted((getattr(t, lo_attr), getattr(t, hi_attr)) for t in tasks if getattr(t, hi_attr) > getattr(t, lo_attr))
        pos = 0
        for lo, hi in rs:
            assert lo == pos
            pos = hi
        assert pos == L
    bound = -(-n // pA) + -(-m // pB)
    for t in tasks:
        assert t.a0 <= t.a1 and t.b0 <= t.b1 and t.size <= bound
        if t.case in "ae":
            assert (t.a1 == t.a0) or (t.b1 == t.b0)
        if t.case == "a" and t.size == 0:
            pass
        elif t.size == 0:
            raise AssertionError("only case (a) tasks may be empty (reading R4)")
    # each range within a single block of its array (L357-361)
    for t in tasks:
        if t.a1 > t.a0:
            assert P.block_of(t.a0, n, pA) == P.block_of(t.a1 - 1, n, pA)
        if t.b1 > t.b0:
            assert P.block_of(t.b0, m, pB) == P.block_of(t.b1 - 1, m, pB)


@pytest.mark.parametrize("pair", [(1, 1), (2, 2), (3, 3), (5, 5), (8, 8), (2, 7), (5, 1), (3, 4)])
def test_plan_exhaustive(pair):
    pA, pB = pair
    seqs = list(nondecreasing(5, 3))
    for a in seqs:
        for b in seqs:
            x, y, xbar, ybar, tasks = P.build_plan(a, b, pA, pB)
            check_plan(a, b, pA, pB, tasks, x, y, xbar, ybar)
            tagA = [(k, "A", i) for i, k in enumerate(a)]
            tagB = [(k, "B", j) for j, k in enumerate(b)]
            C = P.execute_plan(tasks, tagA, tagB)
            assert [(e[0], (e[1], e[2])) for e in C] == brute_merge(a, b)


def test_plan_random_sweep():
    rng = random.Random(1202)
    for _ in range(300):
        n, m = rng.randint(0, 400), rng.randint(0, 400)
        K = rng.choice([2, 5, 50, 10 ** 6])
        a = sorted(rng.randrange(K) for _ in range(n))
        b = sorted(rng.randrange(K) for _ in range(m))
        pA, pB = rng.randint(1, 40), rng.randint(1, 40)
        if rng.random() < 0.5:
            pB = pA
        x, y, xbar, ybar, tasks = P.build_plan(a, b, pA, pB)
        x2, y2, xbar2, ybar2, _ = P.build_plan(np.array(a), np.array(b), pA, pB, vectorised=True)
        assert (xbar, ybar) == (xbar2, ybar2)
        check_plan(a, b, pA, pB, tasks, x, y, xbar, ybar)
        tagA = [(k, "A", i) for i, k in enumerate(a)]
        tagB = [(k, "B", j) for j, k in enumerate(b)]
        C = P.execute_plan(tasks, tagA, tagB)
        assert [(e[0], (e[1], e[2])) for e in C] == brute_merge(a, b)


def test_plan_block_of_roundtrip():
    for L in range(0, 40):
        for p in range(1, 12):
            x = P.block_starts(L, p)
            assert x[0] == 0 and x[p] == L
            sizes = [x[i + 1] - x[i] for i in range(p)]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
            for k in range(L):
                i = P.block_of(k, L, p)
                assert x[i] <= k < x[i + 1]
            assert P.block_of(L, L, p) == p


def test_reading_R1_literal_case_d_fails():
    """Step 3(d) printed as A[x_i, ..., x_{j+1}-1] (L330).  The literal reading
    overlaps another task on A=[1,2], B=[0,0,0,1], p=2; x_{i+1} does not."""
    A, B, p = [1, 2], [0, 0, 0, 1], 2
    x, y, xbar, ybar, tasks = P.build_plan(A, B, p)
    t0 = tasks[0]
    assert t0.case == "d"
    j = P.block_of(xbar[0], len(B), p)
    literal = (x[0], x[j + 1])       # A[x_i, x_{j+1})
    assert literal[1] > x[1]         # spills past block i -> overlaps task 1
    check_plan(A, B, p, p, tasks, x, y, xbar, ybar)


def test_reading_R2_b_side_ties_go_to_a():
    """Ties in B-side merges must still go to A: a B-first merge breaks stability."""
    def merge_bfirst(a, b):
        out, i, j = [], 0, 0
        while i < len(a) and j < len(b):
            if b[j][0] <= a[i][0]:
                out.append(b[j]); j += 1
            else:
                out.append(a[i]); i += 1
        return out + a[i:] + b[j:]

    broken = 0
    seqs = list(nondecreasing(4, 3))
    for a in seqs:
        for b in seqs:
            for p in (1, 2, 3):
                *_, tasks = P.build_plan(a, b, p)
                tagA = [(k, "A", i) for i, k in enumerate(a)]
                tagB = [(k, "B", j) for j, k in enumerate(b)]
                good = P.execute_plan(tasks, tagA, tagB)
                assert [(e[0], (e[1], e[2])) for e in good] == brute_merge(a, b)
                C = [None] * (len(a) + len(b))
                for t in tasks:
                    fn = merge_bfirst if t.side == "B" else P.stable_merge_afirst
                    C[t.off:t.off + t.size] = fn(tagA[t.a0:t.a1], tagB[t.b0:t.b1])
                broken += C != good
    assert broken > 0


def test_special_cases(orc):
    A = np.array([1, 2, 3], np.int64); B = np.array([7, 8], np.int64)
    c, _ = orc.merge(A, None, B, None, "i64"); assert c.tolist() == [1, 2, 3, 7, 8]
    c, _ = orc.merge(B, None, A, None, "i64"); assert c.tolist() == [1, 2, 3, 7, 8]
    E = np.array([], np.int64)
    c, _ = orc.merge(E, None, B, None, "i64"); assert c.tolist() == [7, 8]
    c, _ = orc.merge(A, None, E, None, "i64"); assert c.tolist() == [1, 2, 3]
    # all keys equal: C = A || B
    eq = np.full(4, 5, np.uint64)
    c, vc = orc.merge(eq, np.arange(4, dtype=np.uint32), eq[:3],
                      (np.arange(3) | (1 << 31)).astype(np.uint32), "u64")
    assert vc.tolist() == [0, 1, 2, 3] + [(1 << 31) | j for j in range(3)]
    *_, tasks = P.build_plan([5] * 4, [5] * 3, 2)
    assert all(t.case in "ae" for t in tasks if t.side == "A")
    assert all(t.case == "a" for t in tasks if t.side == "B")


# ------------------------------------------------- floating-point keys (f2)
# IEEE 754 totalOrder written from its definition (sign, then magnitude as
# exponent-and-significand fields, reversed for negatives) -- a formulation
# independent of oracle.c's integer-key trick.

import functools  # noqa: E402


def _fields(bits, width):
    sign = bits >> (width - 1)
    mag = bits & ((1 << (width - 1)) - 1)        # exponent and significand, as one field
    return sign, mag


def _total_order_cmp(width):
    def cmp(x, y):
        sx, mx = _fields(x, width)
        sy, my = _fields(y, width)
        if sx != sy:
            return -1 if sx else 1                 # every negative (incl. -0, -NaN) before every positive
        if sx == 0:
            return (mx > my) - (mx < my)
        return (my > mx) - (my < mx)               # both negative: larger magnitude first
    return cmp


@pytest.mark.parametrize("kt,width,np_u,np_f", [("f32", 32, np.uint32, np.float32), ("f64", 64, np.uint64, np.float64)])
def test_float_merge_and_sort_vs_total_order_definition(orc, kt, width, np_u, np_f):
    import synth
    cmp = _total_order_cmp(width)
    for dist in ("special", "full", "bounded:5"):
        inp = synth.merge_input(300, 211, kt, dist, seed=31)
        a = orc.as_np(inp.a_keys, kt)
        b = orc.as_np(inp.b_keys, kt)
        ab, bb = a.view(np_u).tolist(), b.view(np_u).tolist()
        # inputs sorted under the definition
        assert all(cmp(ab[i], ab[i + 1]) <= 0 for i in range(len(ab) - 1))
        tagged = [(k, 0, i) for i, k in enumerate(ab)] + [(k, 1, j) for j, k in enumerate(bb)]
        want = sorted(tagged, key=functools.cmp_to_key(lambda u, v: cmp(u[0], v[0])))   # stable: A first
        va = np.arange(a.size, dtype=np.uint32)
        vb = np.arange(b.size, dtype=np.uint32) | np.uint32(1 << 31)
        ck, cv = orc.merge(a, va, b, vb, kt)
        assert ck.view(np_u).tolist() == [t[0] for t in want]
        assert cv.tolist() == [t[2] | (t[1] << 31) for t in want]
        # sort: stable sort of the concatenation under the definition
        keys = np.concatenate([b, a])
        sk, sv = orc.sort(keys, np.arange(keys.size, dtype=np.uint32), kt)
        kb = keys.view(np_u).tolist()
        order = sorted(range(len(kb)), key=functools.cmp_to_key(lambda i, j: cmp(kb[i], kb[j])))
        assert sv.tolist() == order
        assert sk.view(np_u).tolist() == [kb[i] for i in order]


@pytest.mark.parametrize("kt,width,np_u,np_f", [("f32", 32, np.uint32, np.float32), ("f64", 64, np.uint64, np.float64)])
def test_float_ranks_vs_total_order_count(orc, kt, width, np_u, np_f):
    """Ascending f32 / f64 ranks (PAPER.md L119-128 under IEEE totalOrder,
    reading R16): rank_low = #{X[t] before x}, rank_high = #{X[t] not after
    x}, counted with the standard's field-by-field comparison."""
    import synth
    cmp = _total_order_cmp(width)
    rng = np.random.default_rng(23)
    for dist in ("special", "full", "bounded:5"):
        for n in (0, 1, 7, 64, 301):
            X = orc.as_np(synth.merge_input(max(n, 1), 1, kt, dist, seed=n + 5).a_keys, kt)[:n]
            xb = X.view(np_u).tolist()
            assert all(cmp(xb[i], xb[i + 1]) <= 0 for i in range(len(xb) - 1))
            specials = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1.0, -1.5], dtype=np_f)
            probes = np.concatenate([X[:6], specials, -specials, X[rng.integers(0, max(n, 1), 4)] if n else X[:0]])
            for v in probes:
                vb = int(np.array([v], dtype=np_f).view(np_u)[0])
                lo = sum(1 for e in xb if cmp(e, vb) < 0)
                hi = sum(1 for e in xb if cmp(e, vb) <= 0)
                assert orc.rank_low(v, X, kt) == lo
                assert orc.rank_high(v, X, kt) == hi


def test_float_total_order_special_values(orc):
    """-NaN < -inf < -1 < -0 < +0 < subnormal < 1 < inf < +NaN, and -0/+0 are
    different keys (totalOrder), so A's +0 follows B's -0."""
    f = np.float32
    neg_nan = np.array([0xFFC00000], dtype=np.uint32).view(f)[0]
    a = np.array([-np.inf, -1.0, 0.0, 1.0, np.inf], dtype=f)
    b = np.array([neg_nan, -0.0, np.float32(1e-45), np.nan], dtype=f)
    ck, _ = orc.merge(a, None, b, None, "f32")
    bits = ck.view(np.uint32).tolist()
    assert bits == [0xFFC00000, 0xFF800000, 0xBF800000, 0x80000000, 0x00000000, 0x00000001, 0x3F800000,
                    0x7F800000, 0x7FC00000]


# ------------------------------------------------ descending order (f row 2)
# The paper's method holds for any total order "<="; the
# desc_* oracle functions instantiate it with the reversed order.  Pinned by
# Python's stable sort under the reversed comparison (reverse=True keeps
# stability), by the reversal identity with the ascending oracle, and by
# linear counts for the ranks.

def _desc_sorted_input(rng, dt, kt, n, few):
    if kt in ("f32", "f64"):
        v = rng.choice(np.array([-np.inf, -2.5, -0.0, 0.0, 1.0, 3.0, np.inf, np.nan], dtype=dt), n) if few \
            else rng.standard_normal(n).astype(dt)
    elif few:
        v = rng.integers(0, 4, n).astype(dt)
    else:
        info = np.iinfo(dt)
        v = rng.integers(info.min, info.max, n, dtype=dt, endpoint=True)
    return v


def _order_int(x, kt):
    """An integer with the key order (floats: totalOrder, test-side)."""
    if kt == "f32":
        u = int(np.array([x], dtype=np.float32).view(np.uint32)[0])
        return (u ^ 0xFFFFFFFF) if u >> 31 else (u | (1 << 31))
    if kt == "f64":
        u = int(np.array([x], dtype=np.float64).view(np.uint64)[0])
        return (u ^ 0xFFFFFFFFFFFFFFFF) if u >> 63 else (u | (1 << 63))
    return int(x)


@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
def test_desc_merge_and_sort_vs_python_reverse_sorted(orc, kt):
    rng = np.random.default_rng(11)
    dt = orc.NP_DTYPES[kt]
    for trial in range(30):
        n, m = int(rng.integers(0, 200)), int(rng.integers(0, 200))
        a = _desc_sorted_input(rng, dt, kt, n, trial % 2 == 0)
        b = _desc_sorted_input(rng, dt, kt, m, trial % 2 == 0)
        a = np.array(sorted(a, key=lambda x: _order_int(x, kt), reverse=True), dtype=dt)
        b = np.array(sorted(b, key=lambda x: _order_int(x, kt), reverse=True), dtype=dt)
        va = np.arange(n, dtype=np.uint32)
        vb = (np.arange(m) | (1 << 31)).astype(np.uint32)
        c, vc = orc.merge(a, va, b, vb, kt, descending=True)
        tagged = [(_order_int(k, kt), int(v)) for k, v in zip(a, va)] + \
                 [(_order_int(k, kt), int(v)) for k, v in zip(b, vb)]
        want = sorted(tagged, key=lambda e: e[0], reverse=True)     # stable: A (first in the list) first
        assert vc.tolist() == [v for _, v in want]
        assert [_order_int(k, kt) for k in c] == [k for k, _ in want]
        # reversal identity: desc(A, B) = reverse(asc(reverse(B), reverse(A)))
        c2, vc2 = orc.merge(b[::-1].copy(), vb[::-1].copy(), a[::-1].copy(), va[::-1].copy(), kt)
        assert vc2[::-1].tolist() == vc.tolist()
        # stable descending sort of the unsorted concatenation
        keys = np.concatenate([b, a])
        rng.shuffle(keys)
        sk, sv = orc.sort(keys, np.arange(keys.size, dtype=np.uint32), kt, descending=True)
        order = sorted(range(keys.size), key=lambda i: _order_int(keys[i], kt), reverse=True)
        assert sv.tolist() == order


@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
def test_desc_ranks_vs_linear_count(orc, kt):
    rng = np.random.default_rng(13)
    dt = orc.NP_DTYPES[kt]
    X = _desc_sorted_input(rng, dt, kt, 150, True)
    X = np.array(sorted(X, key=lambda x: _order_int(x, kt), reverse=True), dtype=dt)
    for x in list(X[::7]) + list(_desc_sorted_input(rng, dt, kt, 10, False)):
        ox = _order_int(x, kt)
        assert orc.rank_low(x, X, kt, descending=True) == sum(_order_int(t, kt) > ox for t in X)
        assert orc.rank_high(x, X, kt, descending=True) == sum(_order_int(t, kt) >= ox for t in X)


# --------------------------------------------- wide / struct payloads (f row 2)
# Pinned by brute force (Python's stable sort of the tagged concatenation,
# rows gathered by the tags) and by agreement with the uint32-payload oracle
# when the wide payload is four copies of the uint32 one.

@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
@pytest.mark.parametrize("desc", [False, True])
def test_wide_merge_and_sort_vs_brute_force(orc, kt, desc):
    rng = np.random.default_rng(17)
    dt = orc.NP_DTYPES[kt]
    rdt = np.dtype([("x", "<f8"), ("tag", "<u2"), ("pad", "u1", (5,))])     # a 15-byte struct
    for trial in range(20):
        n, m = int(rng.integers(0, 120)), int(rng.integers(0, 120))
        a = _desc_sorted_input(rng, dt, kt, n, trial % 2 == 0)
        b = _desc_sorted_input(rng, dt, kt, m, trial % 2 == 0)
        a = np.array(sorted(a, key=lambda x: _order_int(x, kt), reverse=desc), dtype=dt)
        b = np.array(sorted(b, key=lambda x: _order_int(x, kt), reverse=desc), dtype=dt)
        va = np.zeros(n, dtype=rdt); va["x"] = rng.standard_normal(n); va["tag"] = np.arange(n)
        vb = np.zeros(m, dtype=rdt); vb["x"] = rng.standard_normal(m); vb["tag"] = 1000 + np.arange(m)
        va["pad"] = rng.integers(0, 256, (n, 5)); vb["pad"] = rng.integers(0, 256, (m, 5))
        c, vc = orc.merge_wide(a, va, b, vb, kt, descending=desc)
        rows = list(va) + list(vb)
        tagged = [(_order_int(k, kt), r) for k, r in zip(list(a) + list(b), range(n + m))]
        want = sorted(tagged, key=lambda e: e[0], reverse=desc)
        assert [_order_int(k, kt) for k in c] == [k for k, _ in want]
        assert vc.tobytes() == b"".join(rows[r].tobytes() for _, r in want)
        # four copies of a uint32 payload == the uint32 oracle's payload
        ua, ub = np.arange(n, dtype=np.uint32), np.arange(m, dtype=np.uint32) | np.uint32(1 << 31)
        _, vc4 = orc.merge_wide(a, np.repeat(ua[:, None], 4, 1), b, np.repeat(ub[:, None], 4, 1), kt,
                                descending=desc)
        _, vc1 = orc.merge(a, ua, b, ub, kt, descending=desc)
        assert vc4.shape == (n + m, 4) and all(np.array_equal(vc4[:, q], vc1) for q in range(4))
        # sort: stable (tags keep input order among equal keys)
        keys = np.concatenate([b, a]); rng.shuffle(keys)
        vals = np.zeros(keys.size, dtype=rdt); vals["tag"] = np.arange(keys.size)
        sk, sv = orc.sort_wide(keys, vals, kt, descending=desc)
        order = sorted(range(keys.size), key=lambda i: _order_int(keys[i], kt), reverse=desc)
        assert sv["tag"].tolist() == order


# ------------------------------------------------- 128-bit keys (f row 2)
# u128 keys = (high, low) 64-bit tuples in lexicographic order; pinned by
# Python's stable sort of the tagged concatenation on Python ints / tuples.

def _u128_input(rng, n, few):
    hi = rng.integers(0, 3, n, dtype=np.uint64) if few else rng.integers(0, 2**64 - 1, n, dtype=np.uint64,
                                                                           endpoint=True)
    lo = rng.integers(0, 4, n, dtype=np.uint64) if few else rng.integers(0, 2**64 - 1, n, dtype=np.uint64,
                                                                           endpoint=True)
    return [(int(h) << 64) | int(l) for h, l in zip(hi, lo)]


def _u128_arr(ints):
    from oracle import U128
    a = np.empty(len(ints), dtype=U128)
    a["lo"] = [x & (2**64 - 1) for x in ints]
    a["hi"] = [x >> 64 for x in ints]
    return a


@pytest.mark.parametrize("desc", [False, True])
def test_u128_merge_sort_ranks_vs_python(orc, desc):
    rng = np.random.default_rng(19)
    for trial in range(30):
        n, m = int(rng.integers(0, 150)), int(rng.integers(0, 150))
        a = sorted(_u128_input(rng, n, trial % 2 == 0), reverse=desc)
        b = sorted(_u128_input(rng, m, trial % 2 == 0), reverse=desc)
        va = np.arange(n, dtype=np.uint32)
        vb = (np.arange(m) | (1 << 31)).astype(np.uint32)
        c, vc = orc.merge(_u128_arr(a), va, _u128_arr(b), vb, "u128", descending=desc)
        want = sorted([(k, int(v)) for k, v in zip(a, va)] + [(k, int(v)) for k, v in zip(b, vb)],
                      key=lambda e: e[0], reverse=desc)
        assert orc.u128_ints(c) == [k for k, _ in want]
        assert vc.tolist() == [v for _, v in want]
        # tuples: the same order as Python's lexicographic tuple order
        assert sorted([(k >> 64, k & (2**64 - 1)) for k in a], reverse=desc) == [(k >> 64, k & (2**64 - 1)) for k in a]
        keys = a + b
        rng.shuffle(keys)
        sk, sv = orc.sort(_u128_arr(keys), np.arange(len(keys), dtype=np.uint32), "u128", descending=desc)
        assert sv.tolist() == sorted(range(len(keys)), key=lambda i: keys[i], reverse=desc)
        for x in (a[::9] + _u128_input(rng, 3, True)):
            lt = sum((t > x) if desc else (t < x) for t in b)
            le = sum((t >= x) if desc else (t <= x) for t in b)
            assert orc.rank_low(x, _u128_arr(b), "u128", descending=desc) == lt
            assert orc.rank_high(x, _u128_arr(b), "u128", descending=desc) == le


@pytest.mark.parametrize("desc", [False, True])
def test_u128_wide_merge_and_sort_vs_python(orc, desc):
    """merge_wide / sort_wide with 128-bit keys: rows of a 13-byte record
    follow their keys exactly as Python's stable sort of (key, row) moves
    them (brute force)."""
    rng = np.random.default_rng(29)
    rdt = np.dtype([("tag", "<u4"), ("x", "<f8"), ("b", "u1")])
    for trial in range(12):
        n, m = int(rng.integers(0, 90)), int(rng.integers(0, 90))
        a = sorted(_u128_input(rng, n, trial % 2 == 0), reverse=desc)
        b = sorted(_u128_input(rng, m, trial % 2 == 0), reverse=desc)
        va = np.zeros(n, dtype=rdt); va["tag"] = np.arange(n); va["x"] = rng.standard_normal(n)
        vb = np.zeros(m, dtype=rdt); vb["tag"] = 500 + np.arange(m); vb["b"] = rng.integers(0, 256, m)
        c, vc = orc.merge_wide(_u128_arr(a), va, _u128_arr(b), vb, "u128", descending=desc)
        rows = list(va) + list(vb)
        want = sorted(zip(a + b, range(n + m)), key=lambda e: e[0], reverse=desc)
        assert orc.u128_ints(c) == [k for k, _ in want]
        assert vc.tobytes() == b"".join(rows[r].tobytes() for _, r in want)
        keys = a + b
        rng.shuffle(keys)
        vals = np.zeros(len(keys), dtype=rdt); vals["tag"] = np.arange(len(keys))
        sk, sv = orc.sort_wide(_u128_arr(keys), vals, "u128", descending=desc)
        assert sv["tag"].tolist() == sorted(range(len(keys)), key=lambda i: keys[i], reverse=desc)
        assert orc.u128_ints(sk) == sorted(keys, reverse=desc)
