"""A/B timing of library builds (experiments): for each config, time K
steps of the bench workload with CUDA events (L2 flushed between steps for
the small ones, as bench.py does), the per-kernel times from the library's
event profiler, and a checksum of the output (every variant must agree).

    SM_LIB_PATH=<variant .so> python scripts/ab_time.py [--configs 1,2,3,4,5] [--steps 20]
"""
import argparse
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
import paper_1202_6575_b200 as sm  # noqa: E402


def digest(ts):
    h = hashlib.sha1()
    for t in ts:
        if t is not None:
            h.update(t.detach().contiguous().view(torch.uint8).cpu().numpy().tobytes())
    return h.hexdigest()[:12]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("SM_LIB_PATH", "default")))
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    flush = torch.empty(2 * bench.L2_BYTES // 4, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    for cfg in [int(x) for x in a.configs.split(",")]:
        wl = bench.make_workload(cfg, bench.rank_seed(cfg, 0), dev, sm)
        small = wl.c["kind"] == "sort" or wl.step_bytes() < 4 * bench.L2_BYTES
        for _ in range(a.warmup):
            wl.prep()
            wl.call()
        torch.cuda.synchronize()
        tot = 0.0
        for _ in range(a.steps):                    # timed (PDL on)
            wl.prep()
            if small:
                flush.add_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            wl.call()
            e1.record(stream)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        sm.profile_enable(True)                     # per-kernel times (the profiler turns PDL off)
        for _ in range(a.steps):
            wl.prep()
            if small:
                flush.add_(1)
            wl.call()
        torch.cuda.synchronize()
        k = {n: sm.profile_read(p) for n, p in (("K1", sm.PROF_K1), ("K2", sm.PROF_K2), ("K3", sm.PROF_K3))}
        sm.profile_enable(False)
        if wl.c["kind"] == "sort":
            outs = (wl.work_k, wl.work_v)
        else:
            outs = (wl.out_k, wl.out_v)
        ms = tot / a.steps
        gbs = wl.step_bytes() / (ms * 1e-3) / 1e9
        per = {n: round(v[0] / max(1, a.steps), 4) for n, v in k.items() if v[1]}
        print(json.dumps({"tag": a.tag, "cfg": cfg, "ms": round(ms, 4), "GBs": round(gbs), "kernels_ms_per_step": per,
                          "digest": digest(outs)}), flush=True)
        del wl
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
