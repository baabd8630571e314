import os, time, torch, sys
sys.path.insert(0, os.getcwd())
import synth, paper_1202_6575_b200 as sm
inp = synth.merge_input(1 << 26, 1 << 26, "i32", "full", 7, payload=False)
a, b = inp.a_keys.pin_memory(), inp.b_keys.pin_memory()
out = torch.empty(a.numel() + b.numel(), dtype=torch.int32).pin_memory()
for _ in range(2):
    sm.merge_stable(a, None, b, None, out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    sm.merge_stable(a, None, b, None, out)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 5
print(os.environ.get("SM_HOST_BLOCKS"), f"{dt*1e3:.2f} ms per call, {2*out.numel()*4/dt/1e9:.1f} GB/s H2D+D2H")
