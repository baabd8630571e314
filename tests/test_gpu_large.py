"""Merges and sorts of 2^31 elements or more (the kernels index 32-bit; the
library adds the paper's Steps 1-4 at coarse granularity on top, see
merge_large_device / sort_large_device).  At this size the oracle is checked
through properties that pin the stable merge / sort exactly (PAPER.md
L158-166): the output is non-decreasing, each input's elements appear in
their input order (source-index payloads), equal keys put A first, and the
keys travel with their payloads.  Needs ~60 GB of device memory."""
import pytest
import torch

import synth
from gpu_util import lib

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _free():
    yield
    torch.cuda.empty_cache()


def test_merge_above_2e31_elements():
    sm = lib()
    n, m = (1 << 30) + 12345, (1 << 30) + 999
    inp = synth.merge_input(n, m, "i32", "bounded:100000", seed=3, payload=True, device="cuda")
    ck, cv = sm.merge_stable(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, key_type="i32")
    torch.cuda.synchronize()
    assert ck.numel() == n + m > (1 << 31)
    assert bool((ck[1:] >= ck[:-1]).all())                             # non-decreasing
    from_a = cv >= 0                                                    # payload bit 31: B
    assert int(from_a.sum()) == n
    assert torch.equal(cv[from_a], inp.a_vals) and torch.equal(ck[from_a], inp.a_keys)   # A in order
    del from_a
    from_b = cv < 0
    assert torch.equal(cv[from_b], inp.b_vals) and torch.equal(ck[from_b], inp.b_keys)   # B in order
    tie = ck[1:] == ck[:-1]
    assert not bool((tie & from_b[:-1] & ~from_b[1:]).any())            # equal keys: A before B


def test_sort_above_2e31_elements():
    sm = lib()
    N = (1 << 31) + 777
    keys = synth._keys("bounded:1048576", "u32", 9, synth.STREAM_SORT, N, "cuda")
    vals = torch.arange(N, dtype=torch.int64, device="cuda").to(torch.int32)   # uint32 bits
    k, v = keys.clone(), vals.clone()
    sm.mergesort_stable(k, v, key_type="u32")
    torch.cuda.synchronize()
    ku = k.to(torch.int64) & 0xFFFFFFFF                                 # unsigned order
    vi = v.to(torch.int64) & 0xFFFFFFFF
    assert bool((ku[1:] >= ku[:-1]).all())
    tie = ku[1:] == ku[:-1]
    assert bool((vi[1:][tie] > vi[:-1][tie]).all())                     # stable: input order on ties
    del tie
    seen = torch.zeros(N, dtype=torch.bool, device="cuda")
    seen[vi] = True
    assert bool(seen.all())                                             # payloads: a permutation
    del seen
    assert torch.equal(k, keys[vi])                                     # keys travel with payloads
