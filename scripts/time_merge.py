"""Time one merge shape through the binding (CUDA events, inputs resident):
python scripts/time_merge.py KEY_TYPE N M [payload 0/1] [dist]"""
import sys
import torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import synth
import paper_1202_6575_b200 as sm

kt, n, m = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
payload = len(sys.argv) > 4 and sys.argv[4] == "1"
dist = sys.argv[5] if len(sys.argv) > 5 else "full"
inp = synth.merge_input(n, m, kt, dist, seed=1, payload=payload).to("cuda")
ck = torch.empty_like(torch.cat([inp.a_keys, inp.b_keys]))
cv = None if not payload else torch.empty(n + m, dtype=torch.int32, device="cuda")
f = lambda: sm.merge_stable(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, ck, cv, key_type=kt)
for _ in range(5):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 100
e0.record()
for _ in range(K):
    f()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
eb = ck.element_size() * (ck.numel() // (n + m)) + (4 if payload else 0)
print(f"{kt} n={n} m={m} payload={payload} {ms:.4f} ms  {2 * (n + m) * eb / ms / 1e6:.0f} GB/s")
