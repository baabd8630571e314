"""GPU parity of the batched stable merge: S
independent merges in one call, each checked bit-exact against the oracle's
merge of that pair (oracle.merge), the outputs laid end to end."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bit_exact, lib

pytestmark = pytest.mark.gpu

NP = {"u32": np.uint32, "i32": np.int32, "i64": np.int64, "u64": np.uint64, "f32": np.float32, "f64": np.float64}
CARRIER = {"u32": np.int32, "i32": np.int32, "i64": np.int64, "u64": np.int64, "f32": np.int32, "f64": np.int64}


def _segments(lengths, kt, dist, seed, stream):
    """Concatenated, per-segment sorted keys drawn from synth's generator."""
    total = int(sum(lengths))
    bits = synth._keys(dist, kt, seed, stream, total, "cpu")
    off = np.zeros(len(lengths) + 1, dtype=np.int64)
    off[1:] = np.cumsum(lengths)
    order = synth.KEY_TYPES[kt][1]
    seg = torch.repeat_interleave(torch.arange(len(lengths)), torch.as_tensor(np.asarray(lengths, dtype=np.int64)))
    idx = torch.sort(synth._order_key(bits, order), stable=True).indices       # library sort by key,
    idx = idx[torch.sort(seg[idx], stable=True).indices]                        # then by segment
    return oracle.as_np(bits[idx], kt).copy(), off


def _case(S, la, lb, kt, dist, payload, seed):
    a, aoff = _segments(la, kt, dist, seed, 1)
    b, boff = _segments(lb, kt, dist, seed, 2)
    va = np.arange(a.size, dtype=np.uint32) if payload else None
    vb = (np.arange(b.size, dtype=np.uint32) | np.uint32(1 << 31)) if payload else None
    want_k, want_v = [], []
    for s in range(S):
        k, v = oracle.merge(a[aoff[s]:aoff[s + 1]], None if va is None else va[aoff[s]:aoff[s + 1]],
                            b[boff[s]:boff[s + 1]], None if vb is None else vb[boff[s]:boff[s + 1]], kt)
        want_k.append(k)
        if payload:
            want_v.append(v)
    want_k = np.concatenate(want_k) if want_k else np.zeros(0, NP[kt])
    want_v = (np.concatenate(want_v) if want_v else np.zeros(0, np.uint32)) if payload else None
    t = lambda x: None if x is None else torch.from_numpy(x.view(CARRIER[kt]) if x.dtype == NP[kt] else
                                                         x.view(np.int32)).cuda()
    return (t(a), t(va), torch.from_numpy(aoff).cuda(), t(b), t(vb), torch.from_numpy(boff).cuda(), want_k, want_v)


def _run(sm, case, kt):
    a, va, aoff, b, vb, boff, want_k, want_v = case
    ck, cv = sm.merge_stable_batched(a, va, aoff, b, vb, boff, key_type=kt)
    torch.cuda.synchronize()
    assert_bit_exact(ck.cpu(), None if cv is None else cv.cpu(), want_k, want_v, kt)


@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
@pytest.mark.parametrize("payload", [True, False])
def test_batched_random_lengths(kt, payload):
    sm = lib()
    rng = np.random.default_rng(11)
    for S, hi in ((1, 50000), (7, 20000), (300, 3000), (3000, 100)):
        la = rng.integers(0, hi, S)
        lb = rng.integers(0, hi, S)
        la[rng.random(S) < 0.1] = 0               # empty A segments
        lb[rng.random(S) < 0.1] = 0               # empty B segments
        for dist in ("bounded:5", "full"):
            _run(sm, _case(S, la, lb, kt, dist, payload, seed=S + hi), kt)


def test_batched_many_segments_and_long_ones():
    sm = lib()
    rng = np.random.default_rng(3)
    S = 20000
    la = rng.integers(0, 40, S)
    lb = rng.integers(0, 40, S)
    la[5] = 100000                                 # spans many blocks
    lb[17] = 65537
    _run(sm, _case(S, la, lb, "u32", "bounded:100", True, seed=9), "u32")


def test_batched_equals_single_merge():
    """S = 1 is the plain merge (same bytes as merge_stable)."""
    sm = lib()
    inp = synth.config_input(1, scale=8).to("cuda")
    z = torch.zeros(1, dtype=torch.int64, device="cuda")
    aoff = torch.cat([z, torch.tensor([inp.n], device="cuda")])
    boff = torch.cat([z, torch.tensor([inp.m], device="cuda")])
    k1, v1 = sm.merge_stable(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, key_type="u32")
    k2, v2 = sm.merge_stable_batched(inp.a_keys, inp.a_vals, aoff, inp.b_keys, inp.b_vals, boff, key_type="u32")
    assert torch.equal(k1, k2) and torch.equal(v1, v2)


def test_batched_degenerate():
    sm = lib()
    e = torch.empty(0, dtype=torch.int32, device="cuda")
    z = torch.zeros(4, dtype=torch.int64, device="cuda")
    k, v = sm.merge_stable_batched(e, e, z, e, e, z)            # three empty segments
    assert k.numel() == 0
    a = torch.arange(10, dtype=torch.int32, device="cuda")
    aoff = torch.tensor([0, 0, 10, 10], dtype=torch.int64, device="cuda")
    boff = torch.zeros(4, dtype=torch.int64, device="cuda")
    k, _ = sm.merge_stable_batched(a, None, aoff, e, None, boff)  # B empty: C = A
    assert torch.equal(k, a)


def test_batched_malformed_offsets_stay_inside_output():
    """Precondition violated (decreasing / out-of-range offsets): the output
    is unspecified, but nothing outside C may be written."""
    sm = lib()
    a = torch.arange(1000, dtype=torch.int32, device="cuda")
    b = torch.arange(500, dtype=torch.int32, device="cuda")
    aoff = torch.tensor([0, 700, 300, 5000], dtype=torch.int64, device="cuda")
    boff = torch.tensor([-7, 400, 100, 500], dtype=torch.int64, device="cuda")
    guard = torch.full((1500 + 4096,), -12345, dtype=torch.int32, device="cuda")
    out = guard[:1500]
    sm.merge_stable_batched(a, None, aoff, b, None, boff, out_keys=out)
    torch.cuda.synchronize()
    assert bool((guard[1500:] == -12345).all())


@pytest.mark.parametrize("kt,payload", [("u32", True), ("i64", False), ("f32", True)])
def test_batched_segments_at_the_tile_boundary(kt, payload):
    """Segments whose n + m is just below, at and just above the tile
    capacity: the first two are single tasks (reading R19), the rest go
    through cross ranks and cases (a)-(e)."""
    sm = lib()
    nv = sm.tile_capacity(kt, payload)
    tot = np.array([nv - 1, nv, nv + 1, 2 * nv, 1, 0, nv - 2, nv + 7] * 5)
    rng = np.random.default_rng(21)
    la = np.array([int(rng.integers(0, t + 1)) for t in tot])
    lb = tot - la
    for dist in ("bounded:5", "full"):
        _run(sm, _case(len(tot), la, lb, kt, dist, payload, seed=7), kt)
