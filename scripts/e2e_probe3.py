import os, time, torch, sys, ctypes
sys.path.insert(0, os.getcwd())
import synth, paper_1202_6575_b200 as sm
inp = synth.merge_input(1 << 26, 1 << 26, "i32", "full", 7, payload=False)
a, b = inp.a_keys.pin_memory(), inp.b_keys.pin_memory()
out = torch.empty(a.numel() + b.numel(), dtype=torch.int32).pin_memory()
lib = sm._lib
for r in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st = lib.merge_stable_i32(a.data_ptr(), None, a.numel(), b.data_ptr(), None, b.numel(), out.data_ptr(), None, None)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"status {st} call returned after {1e3*(t1-t0):.2f} ms, done after {1e3*(t2-t0):.2f} ms")
print("pinned?", a.is_pinned(), b.is_pinned(), out.is_pinned())
