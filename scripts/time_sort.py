"""Device time of one stable merge sort (CUDA events, inputs restored between
calls outside the timed region): python scripts/time_sort.py KT N PAYLOAD DIST [WAYS]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1202_6575_b200 as sm  # noqa: E402
import synth  # noqa: E402

kt, N, payload, dist = sys.argv[1], int(sys.argv[2]), sys.argv[3] == "1", sys.argv[4] if len(sys.argv) > 4 else "full"
ways = int(sys.argv[5]) if len(sys.argv) > 5 else 4
sm.set_sort_ways(ways)
inp = synth.sort_input(N, kt, dist, seed=1, payload=payload, device="cuda")
k, v = inp.keys.clone(), None if inp.vals is None else inp.vals.clone()
ts = []
for i in range(13):
    k.copy_(inp.keys)
    if v is not None:
        v.copy_(inp.vals)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sm.mergesort_stable(k, v, key_type=kt)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1))
ts.sort()
print(f"sort {kt} N={N} payload={payload} {dist} ways={ways}: median {ts[len(ts) // 2]:.3f} ms")
