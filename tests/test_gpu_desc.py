"""GPU parity of the descending-order entry points (SURVEY.md §8(f) row 2:
the paper's method for an arbitrary total order "<=", here the
reversed key order) against the oracle's desc_* functions, bit-exact.

Covers every key type on the merge (device and host buffers, with and
without payloads, ragged sizes across tiles), the batched merge, the rank
queries, the merge sort (run boundaries included) and the Steps 1-4 plan.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import plan as P
from gpu_util import assert_bit_exact, lib

pytestmark = pytest.mark.gpu

KTS = ["u32", "i32", "i64", "u64", "f32", "f64"]
DIST = {"u32": "bounded:50", "i32": "full", "i64": "bounded:1000", "u64": "mostly:0x8000000000000000:9/10",
        "f32": "special", "f64": "full"}


def _merge_case(sm, inp, host=False):
    d = inp if host else inp.to("cuda")
    ck, cv = sm.merge_stable(d.a_keys, d.a_vals, d.b_keys, d.b_vals, key_type=inp.key_type, descending=True)
    torch.cuda.synchronize()
    wk, wv = oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, inp.key_type, descending=True)
    assert_bit_exact(ck.cpu(), None if cv is None else cv.cpu(), wk, wv, inp.key_type)


@pytest.mark.parametrize("kt", KTS)
@pytest.mark.parametrize("nm", [(0, 0), (1, 0), (0, 7), (1, 1), (5003, 2999), (70001, 33), (17, 130001),
                                (1 << 20, (1 << 19) + 7)])
@pytest.mark.parametrize("payload", [True, False])
def test_desc_merge_device(kt, nm, payload):
    sm = lib()
    n, m = nm
    inp = synth.merge_input(n, m, kt, DIST[kt], seed=101 + n % 97, payload=payload, descending=True)
    _merge_case(sm, inp)


@pytest.mark.parametrize("kt", ["u32", "i64", "f32"])
def test_desc_merge_ties_only(kt):
    """All keys equal: the output is A then B (stability under any order)."""
    sm = lib()
    inp = synth.merge_input(9001, 7003, kt, "equal", seed=5, descending=True)
    _merge_case(sm, inp)


@pytest.mark.parametrize("kt,nm", [("u32", (300001, 200003)), ("i64", (3 << 20, 3 << 20))])
def test_desc_merge_host_buffers(kt, nm):
    """Host inputs and outputs: small ones staged, large ones (>= 64 MB) cut
    on the host into pipelined sub-merges under the descending order."""
    sm = lib()
    inp = synth.merge_input(nm[0], nm[1], kt, DIST[kt], seed=9, descending=True)
    _merge_case(sm, inp, host=True)


@pytest.mark.parametrize("kt", KTS)
def test_desc_batched(kt):
    sm = lib()
    inp = synth.batch_input(301, 700, kt, DIST[kt], seed=23, descending=True)
    d = inp.to("cuda")
    ck, cv = sm.merge_stable_batched(d.a_keys, d.a_vals, d.a_offsets, d.b_keys, d.b_vals, d.b_offsets,
                                     key_type=kt, descending=True)
    torch.cuda.synchronize()
    ao, bo = inp.a_offsets.tolist(), inp.b_offsets.tolist()
    ck, cv = ck.cpu(), cv.cpu()
    for s in range(inp.S):
        a0, a1, b0, b1 = ao[s], ao[s + 1], bo[s], bo[s + 1]
        wk, wv = oracle.merge(inp.a_keys[a0:a1], inp.a_vals[a0:a1], inp.b_keys[b0:b1], inp.b_vals[b0:b1], kt,
                              descending=True)
        c0 = a0 + b0
        assert_bit_exact(ck[c0:c0 + wk.size], cv[c0:c0 + wk.size], wk, wv, kt)


@pytest.mark.parametrize("kt", KTS)
def test_desc_ranks(kt):
    sm = lib()
    inp = synth.merge_input(20011, 513, kt, DIST[kt], seed=3, payload=False, descending=True)
    X, keys = inp.a_keys, inp.b_keys
    for high in (False, True):
        got = sm.ranks_stable(X.cuda(), keys.cuda(), high, key_type=kt, descending=True).cpu().tolist()
        f = oracle.rank_high if high else oracle.rank_low
        Xn, kn = oracle.as_np(X, kt), oracle.as_np(keys, kt)
        assert got == [f(x, Xn, kt, descending=True) for x in kn]


@pytest.mark.parametrize("kt", KTS)
@pytest.mark.parametrize("N", [0, 1, 2, 4351, 4352, 4353, 5 * 4352 + 3, (1 << 20) + 5])
def test_desc_sort(kt, N):
    sm = lib()
    inp = synth.sort_input(N, kt, DIST[kt], seed=N % 1000 + 1)
    k, v = inp.keys.cuda(), inp.vals.cuda()
    sm.mergesort_stable(k, v, key_type=kt, descending=True)
    torch.cuda.synchronize()
    wk, wv = oracle.sort(inp.keys, inp.vals, kt, descending=True)
    assert_bit_exact(k.cpu(), v.cpu(), wk, wv, kt)


@pytest.mark.parametrize("pApB", [(1, 1), (3, 3), (17, 5), (64, 64), (5, 99)])
def test_desc_plan_is_ascending_plan_of_negated_keys(pApB):
    """Steps 1-4 under the reversed order of i64 keys = the oracle's plan
    (ascending) of the negated keys: the cases (a)-(e) depend on the order
    only."""
    sm = lib()
    pA, pB = pApB
    inp = synth.merge_input(4001, 2999, "i64", "bounded:40", seed=pA, payload=False, descending=True)
    a = [-int(x) for x in inp.a_keys.tolist()]
    b = [-int(x) for x in inp.b_keys.tolist()]
    _, _, oxbar, oybar, otasks = P.build_plan(a, b, pA, pB)
    xbar, ybar, tasks = sm.merge_plan(inp.a_keys.cuda(), inp.b_keys.cuda(), pA, pB, key_type="i64",
                                      descending=True)
    assert xbar.tolist() == oxbar and ybar.tolist() == oybar
    assert np.array_equal(tasks.cpu().numpy(), P.task_table(otasks))
