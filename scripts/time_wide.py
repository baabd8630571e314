"""Time wide-payload merges and sorts (index payload + row gather) against
the same keys with uint32 payloads: python scripts/time_wide.py"""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1202_6575_b200 as sm


def timed(f, reps=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


n = m = 1 << 25
inp = synth.merge_input(n, m, "u32", "full", seed=1, payload=True).to("cuda")
for name, (dt, shp) in {"u32 payload (fused)": (None, None), "int64 rows": (torch.int64, ()),
                        "16-byte rows": (torch.int32, (4,)), "24-byte rows": (torch.float64, (3,))}.items():
    if dt is None:
        va, vb, pb = inp.a_vals, inp.b_vals, 4
    else:
        va = torch.zeros((n,) + shp, dtype=dt, device="cuda")
        vb = torch.zeros((m,) + shp, dtype=dt, device="cuda")
        pb = va.element_size() * (va[0].numel() if shp else 1)
    ms = timed(lambda: sm.merge_stable(inp.a_keys, va, inp.b_keys, vb, key_type="u32"))
    gbs = 2 * (n + m) * (4 + pb) / ms / 1e6
    print(f"merge 2^25+2^25 u32 keys + {name}: {ms:.3f} ms, {gbs:.0f} GB/s algorithmic")

N = 1 << 26
src = synth.sort_input(N, "u32", "bounded:1048576", seed=2, payload=True)
k0 = src.keys.cuda()
for name, vals0 in (("u32 payload", src.vals.cuda()), ("int64 rows", src.vals.cuda().to(torch.int64))):
    k, v = k0.clone(), vals0.clone()

    def run():
        k.copy_(k0)
        v.copy_(vals0)
        sm.mergesort_stable(k, v, key_type="u32")
    ms = timed(run, 5)
    print(f"sort 2^26 u32 keys + {name}: {ms:.3f} ms (incl. two input copies)")
