"""Host issue time of one small merge call vs its GPU time (is a small merge
launch/host bound?), and the same call replayed from a CUDA graph."""
import os
import sys
import time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1202_6575_b200 as sm

for (n, kt, pay) in ((1 << 15, "i32", False), (1 << 20, "u32", True)):
    inp = synth.merge_input(n, n, kt, "bounded:65536", seed=1, payload=pay).to("cuda")
    ck = torch.empty(2 * n, dtype=inp.a_keys.dtype, device="cuda")
    cv = torch.empty(2 * n, dtype=torch.int32, device="cuda") if pay else None
    f = lambda: sm.merge_stable(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, ck, cv, key_type=kt)
    for _ in range(10):
        f()
    torch.cuda.synchronize()
    K = 500
    t0 = time.perf_counter()
    for _ in range(K):
        f()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{kt} n=m={n}: host issue {1e6 * (t1 - t0) / K:.1f} us/call, wall incl. drain {1e6 * (t2 - t0) / K:.1f} us/call")
    # CUDA graph of the call
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        f()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(g):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(K):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"   graph replay: {1e3 * e0.elapsed_time(e1) / K:.1f} us/call")
    except Exception as ex:
        print("   graph capture failed:", repr(ex)[:200])

# the C ABI alone (ctypes, arguments prepared once)
n = 1 << 15
inp = synth.merge_input(n, n, "i32", "bounded:65536", seed=1, payload=False).to("cuda")
ck = torch.empty(2 * n, dtype=torch.int32, device="cuda")
fn = sm._lib.merge_stable_i32
args = (inp.a_keys.data_ptr(), None, n, inp.b_keys.data_ptr(), None, n, ck.data_ptr(), None,
        torch.cuda.current_stream().cuda_stream)
for _ in range(10):
    fn(*args)
torch.cuda.synchronize()
K = 2000
t0 = time.perf_counter()
for _ in range(K):
    fn(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"C ABI only (ctypes): {1e6 * (t1 - t0) / K:.1f} us/call")
import ctypes
cudart = ctypes.CDLL("libcudart.so") if False else None
