"""K1 latency against the number of searches (experiments): C2's arrays,
merge_plan with p_A = p_B = p (the cross ranks only), CUDA events around K1
through the library's profiler."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1202_6575_b200 as sm  # noqa: E402
import synth  # noqa: E402

inp = synth.config_input(2, device="cuda")
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for p in (256, 1024, 2048, 4096, 8192, 16580, 33160):
    for _ in range(3):
        sm.merge_plan(inp.a_keys, inp.b_keys, p, p, key_type="i32")
    torch.cuda.synchronize()
    sm.profile_enable(True)
    for _ in range(20):
        flush.add_(1)
        sm.merge_plan(inp.a_keys, inp.b_keys, p, p, key_type="i32")
    torch.cuda.synchronize()
    t, n = sm.profile_read(sm.PROF_K1)
    sm.profile_enable(False)
    print(f"p={p:6d} searches={2 * p + 2:6d} K1 {t / max(n, 1) * 1e3:7.2f} us", flush=True)
