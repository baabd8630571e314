"""GPU parity of the 128-bit key entry points (SURVEY.md §8(f) row 2:
128-bit keys and (key, tie) tuples = (hi, lo) words in lexicographic order)
against the oracle's u128 functions, bit-exact: merge (device and host
buffers, ragged sizes across tiles, both orders, payload or not), batched,
ranks, sort, wide payloads, the Steps 1-4 plan, and the alignment contract."""
import numpy as np
import pytest
import torch

import oracle
import synth
from oracle import plan as P
from gpu_util import lib

pytestmark = pytest.mark.gpu


def _eq_keys(got, want_np):
    assert np.array_equal(oracle.as_np(got.cpu(), "u128").view(np.uint64), want_np.view(np.uint64))


def _merge_case(sm, inp, desc, host=False):
    d = inp if host else inp.to("cuda")
    ck, cv = sm.merge_stable(d.a_keys, d.a_vals, d.b_keys, d.b_vals, key_type="u128", descending=desc)
    torch.cuda.synchronize()
    wk, wv = oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, "u128", descending=desc)
    _eq_keys(ck, wk)
    if wv is not None:
        assert np.array_equal(oracle.vals_np(cv.cpu()), wv)


@pytest.mark.parametrize("dist", ["tuple:5", "full"])
@pytest.mark.parametrize("nm", [(0, 0), (1, 0), (0, 3), (2816, 2816), (5003, 2999), (70001, 33),
                                ((1 << 20) + 3, (1 << 19) + 7)])
@pytest.mark.parametrize("payload", [True, False])
@pytest.mark.parametrize("desc", [False, True])
def test_u128_merge(dist, nm, payload, desc):
    sm = lib()
    inp = synth.merge_input(nm[0], nm[1], "u128", dist, seed=nm[0] % 101 + 1, payload=payload, descending=desc)
    _merge_case(sm, inp, desc)


@pytest.mark.parametrize("nm", [(300001, 200003), (2 << 20, 2 << 20)])
def test_u128_merge_host_buffers(nm):
    sm = lib()
    inp = synth.merge_input(nm[0], nm[1], "u128", "tuple:1000", seed=8)
    _merge_case(sm, inp, False, host=True)


@pytest.mark.parametrize("desc", [False, True])
def test_u128_batched(desc):
    sm = lib()
    inp = synth.batch_input(257, 500, "u128", "tuple:40", seed=12, descending=desc)
    d = inp.to("cuda")
    ck, cv = sm.merge_stable_batched(d.a_keys, d.a_vals, d.a_offsets, d.b_keys, d.b_vals, d.b_offsets,
                                     key_type="u128", descending=desc)
    torch.cuda.synchronize()
    ao, bo = inp.a_offsets.tolist(), inp.b_offsets.tolist()
    ck, cv = ck.cpu(), cv.cpu()
    for s in range(inp.S):
        a0, a1, b0, b1 = ao[s], ao[s + 1], bo[s], bo[s + 1]
        wk, wv = oracle.merge(inp.a_keys[a0:a1], inp.a_vals[a0:a1], inp.b_keys[b0:b1], inp.b_vals[b0:b1], "u128",
                              descending=desc)
        c0 = a0 + b0
        _eq_keys(ck[c0:c0 + wk.size], wk)
        assert np.array_equal(oracle.vals_np(cv[c0:c0 + wk.size]), wv)


@pytest.mark.parametrize("desc", [False, True])
def test_u128_ranks(desc):
    sm = lib()
    inp = synth.merge_input(20011, 301, "u128", "tuple:50", seed=4, payload=False, descending=desc)
    X, keys = inp.a_keys, inp.b_keys
    for high in (False, True):
        got = sm.ranks_stable(X.cuda(), keys.cuda(), high, key_type="u128", descending=desc).cpu().tolist()
        f = oracle.rank_high if high else oracle.rank_low
        assert got == [f(x, X, "u128", descending=desc) for x in oracle.u128_ints(keys)]


@pytest.mark.parametrize("N", [0, 1, 4351, 4352, 4353, 5 * 4352 + 3, (1 << 20) + 5])
@pytest.mark.parametrize("dist", ["tuple:7", "full"])
@pytest.mark.parametrize("desc", [False, True])
def test_u128_sort(N, dist, desc):
    sm = lib()
    inp = synth.sort_input(N, "u128", dist, seed=N % 997 + 3)
    k, v = inp.keys.cuda(), inp.vals.cuda()
    sm.mergesort_stable(k, v, key_type="u128", descending=desc)
    torch.cuda.synchronize()
    wk, wv = oracle.sort(inp.keys, inp.vals, "u128", descending=desc)
    _eq_keys(k, wk)
    assert np.array_equal(oracle.vals_np(v.cpu()), wv)


def test_u128_wide_payload_merge_and_sort():
    sm = lib()
    inp = synth.merge_input(30011, 20011, "u128", "tuple:9", seed=6, payload=False)
    va = torch.randn(30011, 3, dtype=torch.float64)
    vb = torch.randn(20011, 3, dtype=torch.float64)
    ck, cv = sm.merge_stable(inp.a_keys.cuda(), va.cuda(), inp.b_keys.cuda(), vb.cuda(), key_type="u128")
    torch.cuda.synchronize()
    wk, wv = oracle.merge_wide(inp.a_keys, va.numpy(), inp.b_keys, vb.numpy(), "u128")
    _eq_keys(ck, wk)
    assert cv.cpu().numpy().tobytes() == wv.tobytes()
    s = synth.sort_input(50021, "u128", "tuple:9", seed=7, payload=False)
    vals = torch.randn(50021, 3, dtype=torch.float64)
    k, v = s.keys.cuda(), vals.cuda()
    sm.mergesort_stable(k, v, key_type="u128", descending=True)
    torch.cuda.synchronize()
    wk, wv = oracle.sort_wide(s.keys, vals.numpy(), "u128", descending=True)
    _eq_keys(k, wk)
    assert v.cpu().numpy().tobytes() == wv.tobytes()


@pytest.mark.parametrize("pApB", [(1, 1), (3, 3), (17, 5), (64, 64)])
def test_u128_plan(pApB):
    sm = lib()
    pA, pB = pApB
    inp = synth.merge_input(4001, 2999, "u128", "tuple:30", seed=pA, payload=False)
    a, b = oracle.u128_ints(inp.a_keys), oracle.u128_ints(inp.b_keys)
    _, _, oxbar, oybar, otasks = P.build_plan(a, b, pA, pB)
    xbar, ybar, tasks = sm.merge_plan(inp.a_keys.cuda(), inp.b_keys.cuda(), pA, pB, key_type="u128")
    assert xbar.tolist() == oxbar and ybar.tolist() == oybar
    assert np.array_equal(tasks.cpu().numpy(), P.task_table(otasks))


def test_u128_rejects_misaligned_keys():
    sm = lib()
    base = torch.zeros(2 * 100 + 1, dtype=torch.int64, device="cuda")
    mis = base[1:].view(100, 2)                       # 8-byte aligned only
    ok = torch.zeros(100, 2, dtype=torch.int64, device="cuda")
    with pytest.raises(sm.StableMergeError):
        sm.merge_stable(mis, None, ok, None, key_type="u128")
    with pytest.raises(ValueError):
        sm.merge_stable(ok, None, ok, None)          # 2-D keys need key_type="u128"
