"""CUDA-graph capture of the device-pointer calls (include/stablemerge.h,
"Device"): a merge, a batched merge and a merge sort captured once into a
torch.cuda.CUDAGraph, then replayed on fresh inputs copied into the captured
buffers; every replay bit-exact against the CPU oracle.  Also: a call leaves
the calling thread's current device as it found it."""
import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bit_exact, lib
from test_gpu_batched import _case

pytestmark = pytest.mark.gpu


def _capture(fn):
    """Warm up on a side stream (one-time setup stays outside the capture),
    then capture fn into a graph."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        out = fn()
    return g, out


@pytest.mark.parametrize("kt,payload,n,m", [("u32", True, (1 << 20) + 3, (1 << 19) + 11),
                                            ("i32", False, 100_003, 7), ("i64", True, 65_537, 65_536),
                                            ("f32", True, 40_001, 50_003)])
def test_merge_graph_replay(kt, payload, n, m):
    sm = lib()
    st = synth.merge_input(n, m, kt, "full", seed=1, payload=payload).to("cuda")   # captured buffers
    g, (ck, cv) = _capture(lambda: sm.merge_stable(st.a_keys, st.a_vals, st.b_keys, st.b_vals, key_type=kt))
    for seed in (2, 3):
        inp = synth.merge_input(n, m, kt, "bounded:1000" if seed == 3 else "full", seed=seed, payload=payload)
        for dst, src in ((st.a_keys, inp.a_keys), (st.b_keys, inp.b_keys), (st.a_vals, inp.a_vals),
                         (st.b_vals, inp.b_vals)):
            if dst is not None:
                dst.copy_(src)
        g.replay()
        torch.cuda.synchronize()
        assert_bit_exact(ck.cpu(), None if cv is None else cv.cpu(),
                         *oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, kt), kt)


def test_batched_graph_replay():
    sm = lib()
    rng = np.random.default_rng(5)
    S = 300
    la, lb = rng.integers(0, 9000, S), rng.integers(0, 9000, S)
    a, va, aoff, b, vb, boff, wk, wv = _case(S, la, lb, "u32", "full", True, 11)
    g, (ck, cv) = _capture(lambda: sm.merge_stable_batched(a, va, aoff, b, vb, boff, key_type="u32"))
    a2, va2, _, b2, vb2, _, wk2, wv2 = _case(S, la, lb, "u32", "bounded:50", True, 12)
    for src, want_k, want_v in (((a, va, b, vb), wk, wv), ((a2, va2, b2, vb2), wk2, wv2)):
        for dst, x in zip((a, va, b, vb), src):
            if dst is not x:
                dst.copy_(x)
        g.replay()
        torch.cuda.synchronize()
        assert_bit_exact(ck.cpu(), cv.cpu(), want_k, want_v, "u32")


@pytest.mark.parametrize("kt,payload,N", [("u32", True, 300_007), ("i64", False, 50_001)])
def test_sort_graph_replay(kt, payload, N):
    sm = lib()
    st = synth.sort_input(N, kt, "full", seed=3, payload=payload, device="cuda")
    g, _ = _capture(lambda: sm.mergesort_stable(st.keys, st.vals, key_type=kt))
    for seed in (4, 5):
        inp = synth.sort_input(N, kt, "bounded:100" if seed == 5 else "full", seed=seed, payload=payload)
        st.keys.copy_(inp.keys)
        if payload:
            st.vals.copy_(inp.vals)
        g.replay()
        torch.cuda.synchronize()
        assert_bit_exact(st.keys.cpu(), st.vals.cpu() if payload else None,
                         *oracle.sort(inp.keys, inp.vals, kt), kt)


def test_call_keeps_current_device_and_runs_on_stream_device():
    sm = lib()
    inp = synth.merge_input(10_007, 9_001, "u32", "full", seed=9, payload=True).to("cuda")
    dev = torch.cuda.current_device()
    s = torch.cuda.Stream()
    ck, cv = sm.merge_stable(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, key_type="u32", stream=s)
    s.synchronize()
    assert torch.cuda.current_device() == dev
    cpu = inp.to("cpu")
    assert_bit_exact(ck.cpu(), cv.cpu(), *oracle.merge(cpu.a_keys, cpu.a_vals, cpu.b_keys, cpu.b_vals, "u32"),
                     "u32")


@pytest.mark.parametrize("kind", ["merge", "sort"])
def test_graph_replay_dynamic_task_assignment(kind):
    """Sizes where K2 hands its tasks out from a task counter (more than 8 tasks
    per resident CTA): the counter lives in the call's scratch and is zeroed
    by the kernel launched before K2 -- inside the graph, so every replay
    starts from zero -- each replay the oracle's result."""
    sm = lib()
    if kind == "merge":
        n = m = (1 << 23) + 17
        st = synth.merge_input(n, m, "i32", "full", seed=1, payload=False).to("cuda")
        g, (ck, _) = _capture(lambda: sm.merge_stable(st.a_keys, None, st.b_keys, None, key_type="i32"))
        for seed in (2, 3, 4):
            inp = synth.merge_input(n, m, "i32", "bounded:1000" if seed == 3 else "full", seed=seed, payload=False)
            st.a_keys.copy_(inp.a_keys)
            st.b_keys.copy_(inp.b_keys)
            g.replay()
            torch.cuda.synchronize()
            assert_bit_exact(ck.cpu(), None, *oracle.merge(inp.a_keys, None, inp.b_keys, None, "i32"), "i32")
    else:
        N = (12 << 20) + 5
        st = synth.sort_input(N, "u32", "full", seed=3, payload=True, device="cuda")
        g, _ = _capture(lambda: sm.mergesort_stable(st.keys, st.vals, key_type="u32"))
        for seed in (4, 5):
            inp = synth.sort_input(N, "u32", "bounded:100" if seed == 5 else "full", seed=seed, payload=True)
            st.keys.copy_(inp.keys)
            st.vals.copy_(inp.vals)
            g.replay()
            torch.cuda.synchronize()
            assert_bit_exact(st.keys.cpu(), st.vals.cpu(), *oracle.sort(inp.keys, inp.vals, "u32"), "u32")
