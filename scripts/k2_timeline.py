"""K2 per-CTA timeline (experiments): with an SM_K2_TSTAMP build of the
library, run each config's bench workload back to back and report, for one
call, when the CTAs entered, issued their first stage, finished producing
and finished storing (us from the earliest entry) -- startup latency and
tail imbalance of the persistent grid.

    SM_LIB_PATH=<tstamp build> python scripts/k2_timeline.py [--configs 2,1,3,4]
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1202_6575_b200 as sm  # noqa: E402


def pct(x, q):
    return round(float(np.percentile(x, q)), 2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,1,3,4")
    ap.add_argument("--tag", default=os.path.basename(os.environ.get("SM_LIB_PATH", "default")))
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    fn = sm._lib.sm_debug_k2_timestamps
    fn.argtypes = [ctypes.c_void_p]
    ts = torch.zeros(16 * 4096, dtype=torch.int64, device=dev)
    for cfg in [int(x) for x in a.configs.split(",")]:
        wl = bench.make_workload(cfg, bench.rank_seed(cfg, 0), dev, sm)
        for _ in range(5):
            wl.prep()
            wl.call()
        ts.zero_()
        torch.cuda.synchronize()
        fn(ctypes.c_void_p(ts.data_ptr()))
        wl.prep()
        wl.call()           # the previous call's K2 is still draining when this one's starts (PDL)
        torch.cuda.synchronize()
        fn(None)
        allt = ts.view(-1, 8).cpu().numpy().astype(np.float64)
        k3 = allt[4096:]
        k3 = k3[k3[:, 0] > 0]
        if k3.size:                                  # the sort's phase 1 (K3H): entry, pre-pass, passes
            r3 = (k3 - k3[:, 0].min()) / 1e3
            print(json.dumps({"tag": a.tag, "cfg": cfg, "k3h_ctas": int(k3.shape[0]),
                              **{f"k3h_slot{s}": {"p50": pct(r3[:, s][k3[:, s] > 0], 50),
                                                  "max": pct(r3[:, s][k3[:, s] > 0], 100)}
                                 for s in range(8) if (k3[:, s] > 0).any()}}), flush=True)
        t = allt[:4096]
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        out = {"tag": a.tag, "cfg": cfg, "ctas": int(t.shape[0])}
        for name, k in (("entry", 0), ("first_issue", 1), ("prod_done", 2), ("store_done", 3), ("ranker_done", 4),
                        ("first_queued", 5)):
            col = rel[:, k][t[:, k] > 0]
            if col.size:
                out[name] = {"min": pct(col, 0), "p50": pct(col, 50), "p90": pct(col, 90), "max": pct(col, 100)}
        sd = rel[:, 3]
        out["tail_us(max-p50 store_done)"] = round(float(sd.max() - np.median(sd)), 2)
        print(json.dumps(out), flush=True)
        del wl
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
