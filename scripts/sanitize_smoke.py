"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every entry point at sizes that span several tasks, stages and
sort rounds, results checked against the oracle."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import paper_1202_6575_b200 as sm  # noqa: E402
import synth  # noqa: E402

ok = True
for kt, payload in (("u32", True), ("i32", False), ("i64", True), ("u64", False), ("f32", True)):
    inp = synth.merge_input(30011, 17003, kt, "bounded:50" if kt != "f32" else "special", seed=3, payload=payload)
    d = inp.to("cuda")
    wk, wv = oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, kt)
    for mp in (False, True):
        ck, cv = sm.merge_stable(d.a_keys, d.a_vals, d.b_keys, d.b_vals, key_type=kt, merge_path=mp)
        torch.cuda.synchronize()
        ok &= np.array_equal(oracle.as_np(ck.cpu(), kt).view(np.uint8), wk.view(np.uint8))
        if payload:
            ok &= np.array_equal(oracle.vals_np(cv.cpu()), wv)
    s = synth.sort_input(50000, kt, "bounded:100" if kt != "f32" else "special", seed=4, payload=payload)
    k, v = s.keys.cuda(), (s.vals.cuda() if s.vals is not None else None)
    sm.mergesort_stable(k, v, key_type=kt)
    torch.cuda.synchronize()
    sk, sv = oracle.sort(s.keys, s.vals, kt)
    ok &= np.array_equal(oracle.as_np(k.cpu(), kt).view(np.uint8), sk.view(np.uint8))
b = synth.batch_input(300, 100, "u32", "bounded:1000", seed=5).to("cuda")
ck, cv = sm.merge_stable_batched(b.a_keys, b.a_vals, b.a_offsets, b.b_keys, b.b_vals, b.b_offsets, key_type="u32")
torch.cuda.synchronize()
print("sanitize smoke", "OK" if ok else "MISMATCH")
sys.exit(0 if ok else 1)
