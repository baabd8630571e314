"""GPU parity of the merge sort's phase 2 with two rounds per HBM pass
(sm_set_sort_ways(4), k4_* + k_tasks4; reading R20) against the
CPU oracle, and against the one-round-per-pass path (ways = 2).

The run length is forced small (sm_options.sort_run) so that many passes
-- an odd round first, then four-run passes whose blocks are longer, equal
to or shorter than a run -- run on inputs the oracle sorts in seconds."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bit_exact, lib

pytestmark = pytest.mark.gpu


def gpu_sort(sm, inp: synth.SortInput, ways: int, run=None, descending=False):
    k = inp.keys.cuda()
    v = None if inp.vals is None else inp.vals.cuda()
    sm.set_sort_ways(ways)
    try:
        sm.mergesort_stable(k, v, key_type=inp.key_type, run=run, descending=descending)
        torch.cuda.synchronize()
    finally:
        sm.set_sort_ways(0)
    return k.cpu(), (None if v is None else v.cpu())


@pytest.mark.parametrize("payload", [True, False])
@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
@pytest.mark.parametrize("run,N", [(16, 1), (16, 17), (16, 64), (16, 65), (16, 4097), (16, 20011), (64, 100003),
                                   (1008, 100003), (1008, 4 * 1008), (1008, 16 * 1008 + 1), (4096, 262147),
                                   (30000, 500001)])
def test_sort4_forced_runs(kt, payload, run, N):
    """Every pass count parity (odd: a plain round first), ragged last groups
    (1-3 runs, short last run), blocks longer than the runs (S > L)."""
    sm = lib()
    for dist in ("full", "bounded:3"):
        inp = synth.sort_input(N, kt, dist, seed=N + run, payload=payload)
        want = oracle.sort(inp.keys, inp.vals, kt)
        assert_bit_exact(*gpu_sort(sm, inp, 4, run=run), *want, kt)


@pytest.mark.parametrize("kt", ["u32", "i64", "f32"])
@pytest.mark.parametrize("dist", ["equal", "bounded:2", "special"])
def test_sort4_ties_and_specials(kt, dist):
    """All-equal keys and two-valued keys (every subproblem's ranges tie: the
    stable order is run index, then position), float specials (NaNs, signed
    zeros, infinities under totalOrder)."""
    if dist == "special" and not kt.startswith("f"):
        pytest.skip("float specials")
    sm = lib()
    for N, run in ((70001, 16), (70001, 1008), (300007, 2048)):
        inp = synth.sort_input(N, kt, dist, seed=N, payload=True)
        want = oracle.sort(inp.keys, inp.vals, kt)
        assert_bit_exact(*gpu_sort(sm, inp, 4, run=run), *want, kt)


@pytest.mark.parametrize("kt", ["u32", "i32", "u64", "f64"])
def test_sort4_descending(kt):
    sm = lib()
    for N, run in ((50003, 16), (200003, 1008)):
        inp = synth.sort_input(N, kt, "bounded:64", seed=N, payload=True)
        want = oracle.sort(inp.keys, inp.vals, kt, descending=True)
        assert_bit_exact(*gpu_sort(sm, inp, 4, run=run, descending=True), *want, kt)


@pytest.mark.parametrize("payload", [True, False])
@pytest.mark.parametrize("kt", ["u32", "i64"])
def test_sort4_default_run_matches_oracle(kt, payload):
    """Default phase 1 (one block per SM) and default passes at a size with an
    even and an odd round count."""
    sm = lib()
    for N in (1 << 22, 3 * (1 << 21) + 5):
        inp = synth.sort_input(N, kt, "bounded:1048576", seed=N, payload=payload)
        want = oracle.sort(inp.keys, inp.vals, kt)
        assert_bit_exact(*gpu_sort(sm, inp, 4), *want, kt)


def test_sort4_equals_two_way_full_c5():
    """BASELINE config 5 at full size (N = 2^28): two rounds per pass and one
    round per pass give the same bytes, and the result is sorted and stable
    (payload = original index, increasing within equal keys) and carries
    every key with its index (a permutation of the input)."""
    sm = lib()
    inp = synth.config_input(5)
    k4, v4 = gpu_sort(sm, inp, 4)
    k2, v2 = gpu_sort(sm, inp, 2)
    assert torch.equal(k4, k2) and torch.equal(v4, v2)
    k = k4.numpy().view(np.uint32)
    v = v4.numpy().view(np.uint32)
    assert np.all(k[1:] >= k[:-1])
    tie = k[1:] == k[:-1]
    assert np.all(v[1:][tie] > v[:-1][tie])
    src = inp.keys.numpy().view(np.uint32)
    assert np.array_equal(src[v], k)                  # a permutation carried with its keys


def test_sort_merge_passes_plan():
    """The pass plan the library reports (bench.py's algorithmic bytes use it):
    ceil(log2(N / R)) rounds, two per HBM pass where selected."""
    sm = lib()
    N = 1 << 28
    R = sm.sort_run("u32", True, N)
    rounds = 0
    while R << rounds < N:
        rounds += 1
    try:
        sm.set_sort_ways(2)
        assert sm.sort_merge_passes("u32", True, N) == rounds
        sm.set_sort_ways(4)
        assert sm.sort_merge_passes("u32", True, N) == rounds - rounds // 2
        assert sm.sort_merge_passes("u32", False, N) == rounds - rounds // 2
        r128 = 0
        while sm.sort_run("u128", True, 1 << 20) << r128 < 1 << 20:
            r128 += 1
        assert sm.sort_merge_passes("u128", True, 1 << 20) == r128   # 128-bit keys: one round per pass
        sm.set_sort_ways(0)                          # automatic: N >= ~1.5 M, but 4-byte keys alone < 2^28
        assert sm.sort_merge_passes("u32", True, N) == rounds - rounds // 2
        assert sm.sort_merge_passes("u32", False, N) == rounds
        for kt, payload, n in (("u32", False, 1 << 27), ("u64", True, 1 << 22), ("i64", False, 1 << 21)):
            r = 0
            while sm.sort_run(kt, payload, n) << r < n:
                r += 1
            assert sm.sort_merge_passes(kt, payload, n) == r - r // 2
        r_small = 0
        while sm.sort_run("u64", True, 1 << 20) << r_small < 1 << 20:
            r_small += 1
        assert sm.sort_merge_passes("u64", True, 1 << 20) == r_small
    finally:
        sm.set_sort_ways(0)
