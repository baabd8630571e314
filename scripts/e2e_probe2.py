import os, time, torch, sys
sys.path.insert(0, os.getcwd())
import synth, paper_1202_6575_b200 as sm
n = 1 << 26
inp = synth.merge_input(n, n, "i32", "full", 7, payload=False)
a, b = inp.a_keys.pin_memory(), inp.b_keys.pin_memory()
out = torch.empty(2 * n, dtype=torch.int32).pin_memory()
da, db, dc = torch.empty_like(a, device="cuda"), torch.empty_like(b, device="cuda"), torch.empty_like(out, device="cuda")
s = [torch.cuda.Stream(), torch.cuda.Stream()]
P = 16
ch = n // P
def run(merge=True):
    for k in range(P):
        st = s[k & 1]
        with torch.cuda.stream(st):
            da[k*ch:(k+1)*ch].copy_(a[k*ch:(k+1)*ch], non_blocking=True)
            db[k*ch:(k+1)*ch].copy_(b[k*ch:(k+1)*ch], non_blocking=True)
            if merge:
                sm.merge_stable(da[k*ch:(k+1)*ch], None, db[k*ch:(k+1)*ch], None, dc[2*k*ch:2*(k+1)*ch])
            out[2*k*ch:2*(k+1)*ch].copy_(dc[2*k*ch:2*(k+1)*ch], non_blocking=True)
for merge in (False, True):
    run(merge); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): run(merge)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print("merge" if merge else "copies only", f"{dt*1e3:.2f} ms, {4*out.numel()*2/dt/1e9:.1f} GB/s")
