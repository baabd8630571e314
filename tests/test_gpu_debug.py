"""The SM_DEBUG build (lib/libstablemerge_debug.so): the paper's
disjoint-write invariant checked on the device.  Every
K2 store must fall inside its task's output range and inside C, every K3 /
K3H store inside its run (else the kernel traps), and K2 must store every
output element exactly once -- counted per element by the debug build's
coverage counters (sm_debug_cover).  Runs in a subprocess: a trap would end
the CUDA context of the process that hit it.  The outputs are also compared
with the oracle, so the debug build is parity-tested too."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, ROOT)
sys.path.insert(0, ROOT + "/tests")
import numpy as np, torch
import oracle, synth
import paper_1202_6575_b200 as sm
from gpu_util import assert_bit_exact
assert sm.is_debug_build()
dev = "cuda"
def covered(n_out, fn):
    cover = torch.zeros(n_out, dtype=torch.int32, device=dev)
    sm.debug_cover(cover)
    out = fn()
    torch.cuda.synchronize()
    sm.debug_cover(None)
    return cover, out
# merges of every BASELINE merge config's distribution, reduced, several tiles + ragged tails
for cfg, scale in ((1, 16), (2, 256), (3, 512), (4, 256)):
    inp = synth.config_input(cfg, scale=scale)
    d = inp.to(dev)
    for blk in (None, 500):
        kw = {} if blk is None else dict(block=blk)
        cover, (ck, cv) = covered(inp.n + inp.m, lambda: sm.merge_stable(d.a_keys, d.a_vals, d.b_keys, d.b_vals,
                                                                        key_type=inp.key_type, **kw))
        assert bool((cover == 1).all()), ("merge coverage", cfg, blk, int(cover.min()), int(cover.max()))
        want = oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, inp.key_type)
        assert_bit_exact(ck.cpu(), None if cv is None else cv.cpu(), *want, inp.key_type)
# batched merges
b = synth.batch_input(300, 700, "u32", "bounded:1000", seed=3)
db = b.to(dev)
cover, (ck, cv) = covered(b.n + b.m, lambda: sm.merge_stable_batched(db.a_keys, db.a_vals, db.a_offsets, db.b_keys,
                                                                     db.b_vals, db.b_offsets, key_type="u32"))
assert bool((cover == 1).all()), "batched coverage"
# sorts: the shared-memory block sort and the one-block-per-SM phase 1; every
# merge pass stores every element once
for kt, N, run in (("u32", 300007, None), ("i64", 200003, 16400), ("f32", 150001, 8192 + 16), ("u64", 70001, 1008)):
    s = synth.sort_input(N, kt, "bounded:100000" if kt != "f32" else "special", seed=N, payload=True)
    k, v = s.keys.to(dev), s.vals.to(dev)
    R = run or sm.sort_run(kt, True, N)
    rounds = 0
    L = R
    while L < N:
        rounds += 1
        L *= 2
    # one store per element per HBM pass: two rounds per pass (k_tasks4,
    # ways 4, an odd round on its own) or one (ways 2)
    for ways in (4, 2):
        k, v = s.keys.to(dev), s.vals.to(dev)
        sm.set_sort_ways(ways)
        cover, _ = covered(N, lambda: sm.mergesort_stable(k, v, key_type=kt, run=run))
        sm.set_sort_ways(0)
        passes = rounds - (rounds // 2 if ways == 4 else 0)
        assert bool((cover == passes).all()), ("sort coverage", kt, N, ways, passes, int(cover.min()),
                                               int(cover.max()))
        assert_bit_exact(k.cpu(), v.cpu(), *oracle.sort(s.keys, s.vals, kt), kt)
print("debug build: store ranges and exact coverage ok")
"""


def test_debug_build_store_ranges_and_exact_coverage():
    import build_native
    lib = build_native.build_debug()
    env = dict(os.environ, SM_LIB_PATH=lib)
    r = subprocess.run([sys.executable, "-c", SCRIPT.replace("ROOT", repr(ROOT))], env=env, capture_output=True,
                       text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "exact coverage ok" in r.stdout
