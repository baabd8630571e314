"""GPU parity of the stable merge sort (rows a8-a9) against the CPU oracle."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bit_exact, lib

pytestmark = pytest.mark.gpu


def gpu_sort(sm, inp: synth.SortInput):
    k = inp.keys.cuda()
    v = None if inp.vals is None else inp.vals.cuda()
    sm.mergesort_stable(k, v, key_type=inp.key_type)
    torch.cuda.synchronize()
    return k.cpu(), (None if v is None else v.cpu())


@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
@pytest.mark.parametrize("N", [0, 1, 2, 3, 100, 1919, 1920, 1921, 3840, 5000, 65536, 100003, 1000001])
def test_sort_ragged(kt, N):
    sm = lib()
    for dist, payload in (("bounded:64", True), ("full", True), ("bounded:5", False)):
        inp = synth.sort_input(N, kt, dist, seed=N + 3, payload=payload)
        want = oracle.sort(inp.keys, inp.vals, kt)
        assert_bit_exact(*gpu_sort(sm, inp), *want, kt)


@pytest.mark.parametrize("payload", [True, False])
@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
def test_sort_run_boundaries(kt, payload):
    """Sizes around the block-sort run length R (which depends on the key +
    payload width) and its powers of two (the number of merge rounds changes
    there), full-range and narrow keys (the block sort skips digits all keys
    of a run share)."""
    sm = lib()
    R = sm.sort_run(kt, payload)
    for N in (R - 1, R, R + 1, 2 * R - 1, 2 * R + 3, 4 * R, 5 * R + 7):
        for dist in ("full", "bounded:3", "equal") + (("special",) if kt.startswith("f") else ()):
            inp = synth.sort_input(N, kt, dist, seed=N, payload=payload)
            want = oracle.sort(inp.keys, inp.vals, kt)
            assert_bit_exact(*gpu_sort(sm, inp), *want, kt)


def test_sort_signed_extremes():
    """Signed keys across zero and at both extremes (the block sort ranks the
    unsigned view with the sign bit flipped)."""
    sm = lib()
    for kt, dt in (("i32", np.int32), ("i64", np.int64)):
        info = np.iinfo(dt)
        rng = np.random.default_rng(7)
        vals = np.array([info.min, info.max, -1, 0, 1, info.min + 1, info.max - 1], dtype=dt)
        k = rng.choice(vals, size=20011).astype(dt)
        ct = torch.int32 if dt == np.int32 else torch.int64
        inp = synth.SortInput(kt, torch.from_numpy(k.view(np.int32 if dt == np.int32 else np.int64).copy()),
                              torch.arange(k.size, dtype=torch.int32))
        want = oracle.sort(inp.keys, inp.vals, kt)
        assert_bit_exact(*gpu_sort(sm, inp), *want, kt)


@pytest.mark.parametrize("pattern", ["sorted", "reversed", "all_equal", "sawtooth"])
def test_sort_patterns(pattern):
    sm = lib()
    N = 300007
    if pattern == "sorted":
        k = torch.arange(N, dtype=torch.int32)
    elif pattern == "reversed":
        k = torch.arange(N, 0, -1, dtype=torch.int32)
    elif pattern == "all_equal":
        k = torch.full((N,), 3, dtype=torch.int32)
    else:
        k = (torch.arange(N, dtype=torch.int32) % 1000)
    inp = synth.SortInput("i32", k, torch.arange(N, dtype=torch.int32))
    want = oracle.sort(inp.keys, inp.vals, "i32")
    got = gpu_sort(sm, inp)
    assert_bit_exact(*got, *want, "i32")
    if pattern in ("sorted", "all_equal"):
        assert torch.equal(got[1], torch.arange(N, dtype=torch.int32))


def test_sort_reduced_config5():
    sm = lib()
    inp = synth.config_input(5, scale=64)
    want = oracle.sort(inp.keys, inp.vals, "u32")
    assert_bit_exact(*gpu_sort(sm, inp), *want, "u32")


def test_sort_host_buffers():
    sm = lib()
    inp = synth.config_input(5, scale=4096)
    want = oracle.sort(inp.keys, inp.vals, "u32")
    k, v = inp.keys.clone(), inp.vals.clone()
    sm.mergesort_stable(k, v, key_type="u32")
    assert_bit_exact(k, v, *want, "u32")


def test_sort_full_size_config5():
    """N = 2^28 (BASELINE.json config 5), default launch configuration.  The
    stable sort of (key, original index) is unique, so the check is: keys
    non-decreasing, payload a permutation, out_key[t] == in_key[payload[t]],
    and equal keys in increasing payload order; plus
    the oracle's own sort on a 2^22 prefix-independent sample run."""
    sm = lib()
    dev = synth.config_input(5, device="cuda")
    k0 = dev.keys.clone()
    sm.mergesort_stable(dev.keys, dev.vals, key_type="u32")
    torch.cuda.synchronize()
    k, v = dev.keys, dev.vals.long()
    ku = k.long() & 0xFFFFFFFF
    assert bool((ku[1:] >= ku[:-1]).all())
    assert bool((torch.sort(v).values == torch.arange(v.numel(), device="cuda")).all())
    assert torch.equal(k, k0[v])
    ties = ku[1:] == ku[:-1]
    assert bool((v[1:][ties] > v[:-1][ties]).all())
    # bit-exact against the oracle on the full array
    want_k, want_v = oracle.sort(k0.cpu(), torch.arange(k0.numel(), dtype=torch.int32), "u32")
    assert_bit_exact(k.cpu(), dev.vals.cpu(), want_k, want_v, "u32")


@pytest.mark.parametrize("kt,N,payload,pinned", [("u32", (8 << 20) + 12345, True, True),
                                                  ("i64", (12 << 20) + 7, True, False),
                                                  ("u32", (20 << 20) + 3, False, True),
                                                  ("f32", (16 << 20) + 99, True, True)])
def test_sort_host_pipelined(kt, N, payload, pinned):
    """Host buffers of 64 MB or more: chunked uploads overlapped with the
    chunk sorts, and the last merge round cut by the coarse Steps 1-4 into
    sub-merges downloaded as they finish -- same bytes as the oracle."""
    sm = lib()
    inp = synth.sort_input(N, kt, "bounded:100000" if kt != "f32" else "special", seed=N % 101, payload=payload)
    want = oracle.sort(inp.keys, inp.vals, kt)
    k = inp.keys.clone()
    v = None if inp.vals is None else inp.vals.clone()
    if pinned:
        k = k.pin_memory()
        v = None if v is None else v.pin_memory()
    sm.mergesort_stable(k, v, key_type=kt)
    assert_bit_exact(k, v, *want, kt)


def test_host_pipelines_sort_then_merge_same_thread():
    """The sort's and the merge's host pipelines share one per-(thread,
    device) set of streams and events: a host-buffer sort (which grows one
    event list) followed by a pipelined host-buffer merge (which needs two)
    on the same thread -- a regression test for an event list read past its
    end -- both as the oracle."""
    sm = lib()
    s = synth.sort_input((20 << 20) + 3, "u32", "bounded:100000", seed=7, payload=False)
    k = s.keys.clone().pin_memory()
    sm.mergesort_stable(k, None, key_type="u32")
    assert_bit_exact(k, None, *oracle.sort(s.keys, None, "u32"), "u32")
    m = synth.merge_input(3 << 20, 3 << 20, "i64", "bounded:1000", seed=9, payload=True)
    ck, cv = sm.merge_stable(m.a_keys, m.a_vals, m.b_keys, m.b_vals, key_type="i64")
    assert_bit_exact(ck, cv, *oracle.merge(m.a_keys, m.a_vals, m.b_keys, m.b_vals, "i64"), "i64")


@pytest.mark.parametrize("kt,s", [("u32", 1), ("i64", 3), ("f64", 1)])
def test_sort_misaligned_views(kt, s):
    sm = lib()
    inp = synth.sort_input(100003, kt, "bounded:1000", seed=5)
    ct = synth.KEY_TYPES[kt][0]
    bk = torch.full((inp.N + s + 8,), -1, dtype=ct, device="cuda")
    bv = torch.full((inp.N + s + 8,), -1, dtype=torch.int32, device="cuda")
    k, v = bk[s:s + inp.N], bv[s:s + inp.N]
    k.copy_(inp.keys.cuda())
    v.copy_(inp.vals.cuda())
    sm.mergesort_stable(k, v, key_type=kt)
    torch.cuda.synchronize()
    assert_bit_exact(k.cpu(), v.cpu(), *oracle.sort(inp.keys, inp.vals, kt), kt)
    assert bool((bk[:s] == -1).all()) and bool((bk[s + inp.N:] == -1).all())


@pytest.mark.parametrize("payload", [True, False])
@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
def test_sort_blocks_per_sm(kt, payload):
    """Phase 1 with one CTA per block (k_block_sort_hbm), forced at small
    sizes through the run length: blocks of one element-tile and of several
    (ragged last tile, ragged last block), both parities of the round count
    (the pass plan takes one more pass, or copies an all-equal block, to land
    in the buffer the rounds start from), narrow and full-range keys (bytes
    all keys of a block share are skipped)."""
    sm = lib()
    dists = ("full", "bounded:3", "bounded:300", "equal") + (("special",) if kt.startswith("f") else ())
    for N, run in ((1000, 16), (5000, 1008), (20000, 8192 + 16), (40000, 20000), (70001, 70016),
                   (100003, 3 * 8192 + 48), (250000, 17008)):
        for dist in dists:
            inp = synth.sort_input(N, kt, dist, seed=N + run, payload=payload)
            want = oracle.sort(inp.keys, inp.vals, kt)
            k = inp.keys.cuda()
            v = None if inp.vals is None else inp.vals.cuda()
            sm.mergesort_stable(k, v, key_type=kt, run=run)
            torch.cuda.synchronize()
            assert_bit_exact(k.cpu(), None if v is None else v.cpu(), *want, kt)


@pytest.mark.parametrize("kt,payload", [("u32", True), ("i64", True), ("u64", False), ("f32", True)])
def test_sort_default_blocks_per_sm(kt, payload):
    """Sizes where the default phase 1 is one block per SM (sort_run(n) is
    not the shared-memory tile), checked against the oracle."""
    sm = lib()
    for N in (sm.sort_run(kt, payload) * 0 + 148 * (1 << 15) + 5, (12 << 20) + 77):
        assert sm.sort_run(kt, payload, N) != sm.sort_run(kt, payload)
        inp = synth.sort_input(N, kt, "bounded:100000" if kt != "f32" else "special", seed=N % 97, payload=payload)
        want = oracle.sort(inp.keys, inp.vals, kt)
        k = inp.keys.cuda()
        v = None if inp.vals is None else inp.vals.cuda()
        sm.mergesort_stable(k, v, key_type=kt)
        torch.cuda.synchronize()
        assert_bit_exact(k.cpu(), None if v is None else v.cpu(), *want, kt)


@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
def test_sort_blocks_per_sm_descending(kt):
    """The one-block-per-SM phase 1 under the reversed order (Desc<> keys:
    the complemented order view drives the radix digits), forced at small
    sizes, and at a size where it is the default: equal to the oracle's
    descending stable sort."""
    sm = lib()
    cases = [(30001, 8192 + 16, "bounded:300"), (50000, 4096, "full"), (9000, 16, "equal")]
    if kt in ("u32", "f32"):
        cases.append((148 * (1 << 15) + 3, None, "bounded:100000" if kt == "u32" else "special"))
    for N, run, dist in cases:
        inp = synth.sort_input(N, kt, dist if not (kt.startswith("f") and dist == "full") else "special",
                               seed=N + 1, payload=True)
        want = oracle.sort(inp.keys, inp.vals, kt, descending=True)
        k, v = inp.keys.cuda(), inp.vals.cuda()
        sm.mergesort_stable(k, v, key_type=kt, descending=True, run=run)
        torch.cuda.synchronize()
        assert_bit_exact(k.cpu(), v.cpu(), *want, kt)


@pytest.mark.parametrize("dist,desc", [("bounded:3", False), ("equal", False), ("full", True), ("bounded:3", True)])
def test_sort_rounds_ties_across_chunks(dist, desc):
    """A 12.6 M sort (one block per SM in phase 1, then eight rounds whose runs
    grow past 255 blocks per side): heavy ties, all-equal keys, both orders --
    the oracle's stable sort.  (A shared-memory-sample cross-rank kernel for
    these rounds was measured slower than the plain searches: DESIGN §12.)"""
    sm = lib()
    N = (12 << 20) + 77
    inp = synth.sort_input(N, "u32", dist, seed=N % 89, payload=True)
    want = oracle.sort(inp.keys, inp.vals, "u32", descending=desc)
    k, v = inp.keys.cuda(), inp.vals.cuda()
    sm.mergesort_stable(k, v, key_type="u32", descending=desc)
    torch.cuda.synchronize()
    assert_bit_exact(k.cpu(), v.cpu(), *want, "u32")
