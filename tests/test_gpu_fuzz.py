"""Seeded random sweep over the public API against the oracle (bit-exact):
key type x order x payload kind x size x distribution, for merge, batched
merge and sort -- combinations the targeted tests do not enumerate."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bit_exact, lib

pytestmark = pytest.mark.gpu

KTS = ["u32", "i32", "i64", "u64", "f32", "f64", "u128"]
DISTS = {"u32": ["bounded:3", "bounded:65536", "full"], "i32": ["full", "bounded:7"],
         "i64": ["bounded:1000", "full"], "u64": ["mostly:0x8000000000000000:9/10", "full"],
         "f32": ["special", "full"], "f64": ["special", "full"], "u128": ["tuple:5", "full"]}


def _cases(seed, count):
    rng = np.random.default_rng(seed)
    for i in range(count):
        kt = KTS[int(rng.integers(0, len(KTS)))]
        dist = DISTS[kt][int(rng.integers(0, len(DISTS[kt])))]
        size_class = int(rng.integers(0, 4))
        hi = [50, 5000, 200000, 3_000_000][size_class]
        n, m = int(rng.integers(0, hi)), int(rng.integers(0, hi))
        yield i, kt, dist, n, m, bool(rng.integers(0, 2)), int(rng.integers(0, 3))


def _keys_eq(got, want, kt):
    if kt == "u128":
        assert np.array_equal(oracle.as_np(got.cpu(), "u128").view(np.uint64), want.view(np.uint64))
    else:
        assert_bit_exact(got.cpu(), None, want, None, kt)


@pytest.mark.parametrize("chunk", range(10))
def test_fuzz_merge(chunk):
    sm = lib()
    for i, kt, dist, n, m, desc, pay in _cases(100 + chunk, 20):
        inp = synth.merge_input(n, m, kt, dist, seed=i + 1000 * chunk, payload=(pay == 1), descending=desc)
        d = inp.to("cuda")
        if pay == 2:                                  # 8-byte payload rows (fused 64-bit path)
            va = torch.arange(n, dtype=torch.int64) * 3 + 1
            vb = -torch.arange(m, dtype=torch.int64) - 1
            ck, cv = sm.merge_stable(d.a_keys, va.cuda(), d.b_keys, vb.cuda(), key_type=kt, descending=desc)
            wk, wv = oracle.merge_wide(inp.a_keys, va.numpy(), inp.b_keys, vb.numpy(), kt, descending=desc)
            _keys_eq(ck, wk, kt)
            assert np.array_equal(cv.cpu().numpy(), wv), (kt, dist, n, m, desc)
            continue
        ck, cv = sm.merge_stable(d.a_keys, d.a_vals, d.b_keys, d.b_vals, key_type=kt, descending=desc)
        wk, wv = oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, kt, descending=desc)
        _keys_eq(ck, wk, kt)
        if wv is not None:
            assert np.array_equal(oracle.vals_np(cv.cpu()), wv), (kt, dist, n, m, desc)


@pytest.mark.parametrize("chunk", range(5))
def test_fuzz_sort(chunk):
    sm = lib()
    for i, kt, dist, n, m, desc, pay in _cases(200 + chunk, 12):
        N = n + m
        inp = synth.sort_input(N, kt, dist, seed=i + 7 * chunk, payload=(pay != 0))
        k = inp.keys.cuda()
        v = None if inp.vals is None else inp.vals.cuda()
        sm.mergesort_stable(k, v, key_type=kt, descending=desc)
        wk, wv = oracle.sort(inp.keys, inp.vals, kt, descending=desc)
        _keys_eq(k, wk, kt)
        if wv is not None:
            assert np.array_equal(oracle.vals_np(v.cpu()), wv), (kt, dist, N, desc)


@pytest.mark.parametrize("chunk", range(2))
def test_fuzz_batched(chunk):
    sm = lib()
    rng = np.random.default_rng(300 + chunk)
    for i in range(8):
        kt = KTS[int(rng.integers(0, len(KTS)))]
        dist = DISTS[kt][0]
        S, mean = int(rng.integers(1, 400)), int(rng.integers(1, 3000))
        desc = bool(rng.integers(0, 2))
        inp = synth.batch_input(S, mean, kt, dist, seed=i + 11 * chunk, descending=desc)
        d = inp.to("cuda")
        ck, cv = sm.merge_stable_batched(d.a_keys, d.a_vals, d.a_offsets, d.b_keys, d.b_vals, d.b_offsets,
                                         key_type=kt, descending=desc)
        ao, bo = inp.a_offsets.tolist(), inp.b_offsets.tolist()
        ck, cv = ck.cpu(), cv.cpu()
        for s in range(S):
            a0, a1, b0, b1 = ao[s], ao[s + 1], bo[s], bo[s + 1]
            wk, wv = oracle.merge(inp.a_keys[a0:a1], inp.a_vals[a0:a1], inp.b_keys[b0:b1], inp.b_vals[b0:b1], kt,
                                  descending=desc)
            c0 = a0 + b0
            _keys_eq(ck[c0:c0 + (a1 - a0) + (b1 - b0)], wk, kt)
            assert np.array_equal(oracle.vals_np(cv[c0:c0 + (a1 - a0) + (b1 - b0)]), wv)
