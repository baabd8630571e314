"""GPU parity of the wide / struct-payload entry points (SURVEY.md §8(f)
row 2) against the oracle's merge_wide / sort_wide, bit-exact: payload rows
of 5 to 64 bytes and several dtypes, ascending and descending, ragged sizes
across tiles, misaligned rows, the batched merge and the sort."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bit_exact, lib

pytestmark = pytest.mark.gpu

DIST = {"u32": "bounded:50", "i32": "full", "i64": "bounded:1000", "u64": "mostly:0x8000000000000000:9/10",
        "f32": "special", "f64": "full"}
# payload row kinds: (torch dtype, trailing shape)
ROWS = {"i64": (torch.int64, ()), "f64x3": (torch.float64, (3,)), "u8x5": (torch.uint8, (5,)),
        "i16x3": (torch.int16, (3,)), "f32x4": (torch.float32, (4,)), "i32x16": (torch.int32, (16,))}


def _rows(kind, count, seed):
    dt, shp = ROWS[kind]
    g = torch.Generator().manual_seed(seed)
    raw = torch.randint(0, 256, (count * max(1, int(np.prod(shp))) * torch.tensor([], dtype=dt).element_size(),),
                        generator=g, dtype=torch.uint8)
    return raw.view(dt).reshape((count,) + shp)


def _bits(t):
    return t.cpu().contiguous().view(torch.uint8).numpy().tobytes()


CASES = [(kind, nm) for kind in ROWS for nm in [(0, 0), (1, 0), (5003, 2999), (70001, 33)]] + \
        [(kind, ((1 << 20) + 3, (1 << 19) + 7)) for kind in ("i64", "u8x5")]


@pytest.mark.parametrize("kt", ["u32", "i32", "i64", "u64", "f32", "f64"])
@pytest.mark.parametrize("kind,nm", CASES)
@pytest.mark.parametrize("desc", [False, True])
def test_wide_merge(kt, kind, nm, desc):
    sm = lib()
    n, m = nm
    inp = synth.merge_input(n, m, kt, DIST[kt], seed=n % 89 + 3, payload=False, descending=desc)
    va, vb = _rows(kind, n, 1), _rows(kind, m, 2)
    ck, cv = sm.merge_stable(inp.a_keys.cuda(), va.cuda(), inp.b_keys.cuda(), vb.cuda(), key_type=kt,
                             descending=desc)
    torch.cuda.synchronize()
    wk, wv = oracle.merge_wide(inp.a_keys, va.numpy(), inp.b_keys, vb.numpy(), kt, descending=desc)
    assert_bit_exact(ck.cpu(), None, wk, None, kt)
    assert cv.shape == (n + m,) + ROWS[kind][1] and cv.dtype == ROWS[kind][0]
    assert _bits(cv) == wv.tobytes()


def test_wide_merge_misaligned_rows():
    """Rows starting at odd addresses (a uint8 row view at offset 1): the
    gather falls back to byte words."""
    sm = lib()
    inp = synth.merge_input(9001, 4003, "u32", "bounded:50", seed=4, payload=False)
    base_a = _rows("u8x5", 9002, 5).cuda()
    base_b = _rows("u8x5", 4004, 6).cuda()
    va = base_a.view(-1)[1:1 + 9001 * 5].view(9001, 5)
    vb = base_b.view(-1)[3:3 + 4003 * 5].view(4003, 5)
    ck, cv = sm.merge_stable(inp.a_keys.cuda(), va, inp.b_keys.cuda(), vb, key_type="u32")
    torch.cuda.synchronize()
    wk, wv = oracle.merge_wide(inp.a_keys, va.cpu().numpy(), inp.b_keys, vb.cpu().numpy(), "u32")
    assert _bits(cv) == wv.tobytes()


@pytest.mark.parametrize("kt", ["u32", "i64", "f64"])
@pytest.mark.parametrize("desc", [False, True])
@pytest.mark.parametrize("kind", ["f64x3", "i64"])          # i64: the fused 8-byte path
def test_wide_batched(kt, desc, kind):
    sm = lib()
    inp = synth.batch_input(257, 2600, kt, DIST[kt], seed=31, payload=False, descending=desc)
    va, vb = _rows(kind, inp.n, 7), _rows(kind, inp.m, 8)
    d = inp.to("cuda")
    ck, cv = sm.merge_stable_batched(d.a_keys, va.cuda(), d.a_offsets, d.b_keys, vb.cuda(), d.b_offsets,
                                     key_type=kt, descending=desc)
    torch.cuda.synchronize()
    ao, bo = inp.a_offsets.tolist(), inp.b_offsets.tolist()
    cvb = cv.cpu()
    for s in range(inp.S):
        a0, a1, b0, b1 = ao[s], ao[s + 1], bo[s], bo[s + 1]
        wk, wv = oracle.merge_wide(inp.a_keys[a0:a1], va[a0:a1].numpy(), inp.b_keys[b0:b1], vb[b0:b1].numpy(),
                                   kt, descending=desc)
        c0 = a0 + b0
        assert_bit_exact(ck[c0:c0 + wk.size].cpu(), None, wk, None, kt)
        assert _bits(cvb[c0:c0 + wk.size]) == wv.tobytes()


@pytest.mark.parametrize("kt", ["u32", "i32", "u64", "f32"])
@pytest.mark.parametrize("kind", ["i64", "u8x5", "i32x16"])
@pytest.mark.parametrize("N", [0, 1, 4353, 5 * 4352 + 3, (1 << 20) + 5])
@pytest.mark.parametrize("desc", [False, True])
def test_wide_sort(kt, kind, N, desc):
    sm = lib()
    inp = synth.sort_input(N, kt, DIST[kt], seed=N % 1000 + 2, payload=False)
    vals = _rows(kind, N, 9)
    k, v = inp.keys.cuda(), vals.cuda()
    sm.mergesort_stable(k, v, key_type=kt, descending=desc)
    torch.cuda.synchronize()
    wk, wv = oracle.sort_wide(inp.keys, vals.numpy(), kt, descending=desc)
    assert_bit_exact(k.cpu(), None, wk, None, kt)
    assert _bits(v) == wv.tobytes()


def test_wide_rejects_host_and_bad_rows():
    sm = lib()
    a = torch.arange(10, dtype=torch.int32)
    with pytest.raises(ValueError):
        sm.merge_stable(a, torch.zeros(10, 2, dtype=torch.int64), a, torch.zeros(10, 2, dtype=torch.int64))
    with pytest.raises(ValueError):
        sm.merge_stable(a.cuda(), torch.zeros(10, 2, dtype=torch.int64).cuda(), a.cuda(),
                        torch.zeros(10, 3, dtype=torch.int64).cuda())
