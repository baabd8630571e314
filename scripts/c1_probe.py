"""C1 launch-overhead probe (experiments): per-call device time of the C1
merge (a) back to back, (b) after an L2-flushing torch kernel (the bench's
per-step flush), (c) after the flush and then a small kernel; small-merge
one-launch on and off."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1202_6575_b200 as sm  # noqa: E402

dev = torch.device("cuda", 0)
wl = bench.make_workload(1, bench.rank_seed(1, 0), dev, sm)
flush = torch.empty(2 * bench.L2_BYTES // 4, dtype=torch.int32, device=dev)
small = torch.zeros(1024, dtype=torch.int32, device=dev)
st = torch.cuda.current_stream(dev)
for fuse in (True, False):
    sm.set_small_fuse(fuse)
    for mode in ("b2b", "flush", "flush+small"):
        for _ in range(5):
            wl.call()
        torch.cuda.synchronize()
        evs = []
        for _ in range(200):
            if mode != "b2b":
                flush.add_(1)
            if mode == "flush+small":
                small.add_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            wl.call()
            e1.record(st)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
        print(f"small_fuse={fuse} {mode:12s} median {ts[len(ts) // 2]:.2f} us  p10 {ts[len(ts) // 10]:.2f}  p90 {ts[9 * len(ts) // 10]:.2f}", flush=True)
sm.set_small_fuse(True)
