"""Helpers shared by the -m gpu parity tests (no method arithmetic here)."""
import numpy as np
import pytest
import torch

import oracle
import synth


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def lib():
    need_gpu()
    import paper_1202_6575_b200 as sm
    return sm


def gpu_merge(sm, inp: synth.MergeInput, **kw):
    d = inp.to("cuda")
    ck, cv = sm.merge_stable(d.a_keys, d.a_vals, d.b_keys, d.b_vals, key_type=inp.key_type, **kw)
    torch.cuda.synchronize()
    return ck.cpu(), (None if cv is None else cv.cpu())


def oracle_merge(inp: synth.MergeInput):
    return oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, inp.key_type)


def assert_bit_exact(got_k, got_v, want_k, want_v, key_type):
    gk = oracle.as_np(got_k, key_type)
    assert gk.shape == want_k.shape
    if gk.dtype.kind == "f":           # bit patterns: NaN payloads, signed zeros
        ui = np.uint32 if gk.dtype.itemsize == 4 else np.uint64
        gk, want_k = gk.view(ui), np.ascontiguousarray(want_k).view(ui)
    if not np.array_equal(gk, want_k):
        bad = np.flatnonzero(gk != want_k)
        raise AssertionError(f"{bad.size} key mismatches, first at {bad[:8].tolist()}: "
                             f"got {gk[bad[:4]].tolist()} want {want_k[bad[:4]].tolist()}")
    if want_v is not None:
        gv = oracle.vals_np(got_v)
        if not np.array_equal(gv, want_v):
            bad = np.flatnonzero(gv != want_v)
            raise AssertionError(f"{bad.size} payload mismatches, first at {bad[:8].tolist()}")
    else:
        assert got_v is None
