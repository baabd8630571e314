"""The seeded input generators (synth/): known answer, determinism, recipe."""
import numpy as np
import torch

import synth


def test_splitmix64_known_answer():
    # SplitMix64 from state 0: first output is 0xE220A8397B1DCDAF (the
    # published reference sequence of the generator).
    g = 0x9E3779B97F4A7C15
    assert synth._mix64_int(g) == 0xE220A8397B1DCDAF
    t = synth._mix64(torch.tensor([synth._s64(g)]))
    assert (t.item() & ((1 << 64) - 1)) == 0xE220A8397B1DCDAF


def test_stream_deterministic_and_offsettable():
    a = synth.splitmix_stream(5, 1, 1000)
    b = synth.splitmix_stream(5, 1, 1000)
    assert torch.equal(a, b)
    c = synth.splitmix_stream(5, 1, 400, start=600)
    assert torch.equal(a[600:], c)
    assert not torch.equal(a, synth.splitmix_stream(5, 2, 1000))


def test_bounded_range():
    r = synth.splitmix_stream(1, 1, 100000)
    v = synth.bounded(r, 1000)
    assert int(v.min()) >= 0 and int(v.max()) == 999
    # roughly uniform
    h = torch.bincount(v, minlength=1000)
    assert int(h.min()) > 50 and int(h.max()) < 160


def test_config_recipes_small_scale():
    for cfg in (1, 2, 3, 4):
        inp = synth.config_input(cfg, scale=1 << 10)
        kt = inp.key_type
        dt = {"u32": np.uint32, "i32": np.int32, "i64": np.int64, "u64": np.uint64}[kt]
        a = inp.a_keys.numpy().view(dt)
        b = inp.b_keys.numpy().view(dt)
        assert np.all(a[1:] >= a[:-1]) and np.all(b[1:] >= b[:-1])
        if inp.a_vals is not None:
            assert np.array_equal(inp.a_vals.numpy().view(np.uint32), np.arange(inp.n, dtype=np.uint32))
            assert np.array_equal(inp.b_vals.numpy().view(np.uint32),
                                  (np.arange(inp.m) | (1 << 31)).astype(np.uint32))
    c2 = synth.config_input(2, scale=1 << 10)
    assert int(c2.a_keys.min()) < 0 < int(c2.a_keys.max())           # signed full range
    c4 = synth.config_input(4, scale=1 << 8)
    a = c4.a_keys.numpy().view(np.uint64)
    frac = float(np.mean(a == np.uint64(1 << 63)))
    assert 0.87 < frac < 0.93
    s = synth.config_input(5, scale=1 << 12)
    assert s.keys.numel() == (1 << 16) and int(s.keys.max()) < (1 << 20)
    assert torch.equal(s.vals, torch.arange(1 << 16, dtype=torch.int32))
