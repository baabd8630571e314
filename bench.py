#!/usr/bin/env python
"""Benchmark of the B200 stable merge (arXiv 1202.6575) -- driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

A step is one pass of the hot path over one batch of synthetic input: for the
default workload (BASELINE.json configs[1], the one its metric is quoted on:
stable merge keys-only, n = m = 2^26 int32 full range) a step is one
merge_stable call = K1 cross ranks + K2 classify/copy/merge (rows a0-a7).
--config 5 benches the merge sort (rows a8-a9); configs 1, 3, 4 the other
merges.  Inputs are seeded and synthetic (synth/), resident in HBM before the
timed region.  Multi-GPU (torchrun): every rank merges its own replica
(different seed), no collective on the data path ("replicas only",
DESIGN.md); value = all ranks' elements / max-over-ranks time.

Rank 0 prints ONE JSON line.  `roofline` is for the dominant kernel (K2,
k_tasks), timed live with CUDA events on its launch stream (sm_profile_*);
`cpu_baseline` is the CPU oracle (oracle/, single thread) on a bounded sample
of the same workload; `e2e` is the same metric through the C ABI with pinned
HOST buffers (host->device and device->host copies inside the timed region).
`--impl reference` times the oracle instead (the reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402

CONFIG_NAMES = {
    1: "C1 stable merge n=m=2^20 u32 keys in [0,2^16) + u32 source-index payload (BASELINE.json configs[0])",
    2: "C2 stable merge keys-only n=m=2^26 int32 full range (BASELINE.json configs[1])",
    3: "C3 unbalanced stable merge n=2^28 m=2^16 int64 keys in [0,1000) + u32 payload (BASELINE.json configs[2])",
    4: "C4 adversarial stable merge n=2^27 m=2^25 u64 90% one value + u32 payload (BASELINE.json configs[3])",
    5: "C5 stable merge sort N=2^28 u32 keys in [0,2^20) + u32 original-index payload (BASELINE.json configs[4])",
}
L2_BYTES = 126 * 1024 * 1024
FALLBACK_HBM_GBS = 6650.0


def load_json(name):
    p = os.path.join(ROOT, name)
    return json.load(open(p)) if os.path.exists(p) else None


def hbm_peak():
    mp = load_json("MEASURED_PEAKS.json")
    if mp and mp.get("hbm_gbs"):
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy_ R+W)"
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def args_():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, choices=[1, 2, 3, 4, 5], default=2)
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded CPU-oracle sample budget")
    ap.add_argument("--no-extras", action="store_true", help="timed loop only (for ncu launch lists)")
    return ap.parse_args()


# --------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and clock-event reasons via NVML every ~5 ms."""
    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
             0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples = []
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                clk = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
                try:
                    rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    rs = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.samples.append((time.time(), clk, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.ok:
            self._t.start()
        return self

    def stop(self):
        self._stop.set()
        if self.ok:
            self._t.join(timeout=1)

    def summary(self, t0, t1):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "nvml unavailable"}
        win = [s for s in self.samples if t0 <= s[0] <= t1]
        note = "samples inside the timed region"
        if not win:
            win = self.samples[-20:]
            note = "timed region shorter than the sampling period: last samples of the run"
        mask = 0
        for s in win:
            mask |= s[2]
        reasons = [n for b, n in self.NAMES.items() if mask & b and b != 0x1]
        return {"sm_mhz": statistics.median([s[1] for s in win]) if win else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(win), "note": note}


# ---------------------------------------------------------------- helpers
def dist_setup(gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world, device="cuda"):
    """Max of a per-rank scalar (the timed region's device time) over ranks:
    the job is as slow as its slowest replica.  `device` is cuda under NCCL,
    cpu under gloo (tests)."""
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def rank_seed(cfg, rank):
    """Replicas only: each rank merges its own seeded replica."""
    return synth.BASE_SEED + cfg + 1000 * rank


def aggregate_value(elems_per_rank, world, steps, t_ms_max):
    """Whole-job throughput: the elements all ranks processed over the
    max-over-ranks time of the timed region."""
    return world * elems_per_rank * steps / (t_ms_max / 1e3)


def elements_of(cfg):
    c = synth.CONFIGS[cfg]
    return c["N"] if c["kind"] == "sort" else c["n"] + c["m"]


def step_bytes(cfg):
    """Algorithmic HBM bytes of one launch of the dominant kernel (K2) per
    SURVEY.md §8(d): read A+B + write C, keys + payload."""
    c = synth.CONFIGS[cfg]
    eb = synth.elem_bytes(c["key_type"], c["payload"])
    return 2 * elements_of(cfg) * eb


def sort_passes(cfg):
    """Passes of the merge sort over HBM: the block sort (row a8) plus
    ceil(log2(N / R)) merge rounds (row a9), R = the library's run length."""
    import math
    import paper_1202_6575_b200 as sm
    c = synth.CONFIGS[cfg]
    R = sm.sort_run(c["key_type"], c["payload"])
    return 1 + max(0, math.ceil(math.log2(c["N"] / R)))


def step_alg_bytes(cfg):
    """Algorithmic HBM bytes of one whole step: a merge reads A+B and writes C
    once; the sort reads and writes the array once per pass."""
    c = synth.CONFIGS[cfg]
    return step_bytes(cfg) * (sort_passes(cfg) if c["kind"] == "sort" else 1)


def traffic_from_profiles(cfg):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p)).get(str(cfg))
    if not d:
        return None, None
    return d.get("dram_bytes_per_launch"), d.get("source")


# ------------------------------------------------------------------ ours
def run_ours(a, world, rank, local):
    import paper_1202_6575_b200 as sm

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = a.config
    c = synth.CONFIGS[cfg]
    kt = c["key_type"]
    seed = rank_seed(cfg, rank)
    clocks = ClockSampler(local).start()

    # ---- inputs resident in HBM
    if c["kind"] == "merge":
        inp = synth.merge_input(c["n"], c["m"], kt, c["dist"], seed, c["payload"], device=dev)
        n, m = inp.n, inp.m
        out_k = torch.empty(n + m, dtype=inp.a_keys.dtype, device=dev)
        out_v = torch.empty(n + m, dtype=torch.int32, device=dev) if c["payload"] else None

        def call():
            sm.merge_stable(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, out_k, out_v, key_type=kt)
        in_bytes = step_bytes(cfg) // 2
    else:
        src = synth.sort_input(c["N"], kt, c["dist"], seed, c["payload"], device=dev)
        work_k = src.keys.clone()
        work_v = src.vals.clone() if src.vals is not None else None

        def call():
            sm.mergesort_stable(work_k, work_v, key_type=kt)
        in_bytes = step_bytes(cfg) // 2
    elems = elements_of(cfg)
    per_step_events = c["kind"] == "sort" or in_bytes * 2 < 4 * L2_BYTES
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev) if per_step_events else None

    def prep():
        if c["kind"] == "sort":                       # restore the unsorted input (untimed)
            work_k.copy_(src.keys)
            if work_v is not None:
                work_v.copy_(src.vals)
        if flush is not None:
            flush.add_(1)                             # write > L2 between timed steps

    stream = torch.cuda.current_stream(dev)
    for _ in range(a.warmup):
        prep()
        call()
    call()
    launches_per_step = sm.last_launch_count()
    torch.cuda.synchronize(dev)
    barrier(world)
    torch.cuda.synchronize(dev)

    t_wall0 = time.time()
    if not per_step_events:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(a.steps):
            call()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t_ms = e0.elapsed_time(e1)
    else:
        evs = []
        for _ in range(a.steps):
            prep()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            call()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize(dev)
        t_ms = sum(x.elapsed_time(y) for x, y in evs)
    t_wall1 = time.time()
    barrier(world)
    t_ms = max_over_ranks(t_ms, world)
    clk = clocks.summary(t_wall0, t_wall1)

    value = aggregate_value(elems, world, a.steps, t_ms)
    ms_per_step = t_ms / a.steps
    res = dict(value=value, ms_per_step=ms_per_step, launches=launches_per_step * a.steps, clocks=clk,
               per_step_events=per_step_events)
    if a.no_extras:
        clocks.stop()
        return res

    # ---- per-kernel durations (CUDA events on the launch stream)
    prof_steps = max(3, min(a.steps, 50 if c["kind"] == "sort" else 200))
    sm.profile_enable(True)
    for _ in range(prof_steps):
        prep()
        call()
    torch.cuda.synchronize(dev)
    k1 = sm.profile_read(sm.PROF_K1)
    k2 = sm.profile_read(sm.PROF_K2)
    k3 = sm.profile_read(sm.PROF_K3)
    sm.profile_enable(False)
    res["kernels"] = {"k_cross_ranks": k1, "k_tasks": k2, "k_block_sort": k3, "steps": prof_steps}

    # ---- end to end through the C ABI with pinned host buffers
    if c["kind"] == "merge":
        h = inp.to("cpu")
        pin = lambda t: None if t is None else t.pin_memory()
        ha, hav, hb, hbv = pin(h.a_keys), pin(h.a_vals), pin(h.b_keys), pin(h.b_vals)
        hok = torch.empty(n + m, dtype=h.a_keys.dtype).pin_memory()
        hov = torch.empty(n + m, dtype=torch.int32).pin_memory() if c["payload"] else None

        def e2e_call():
            sm.merge_stable(ha, hav, hb, hbv, hok, hov, key_type=kt, stream=stream)
        h2d = in_bytes
        d2h = in_bytes
    else:
        hk = src.keys.cpu().pin_memory()
        hv = src.vals.cpu().pin_memory() if src.vals is not None else None
        hwk, hwv = hk.clone().pin_memory(), (hv.clone().pin_memory() if hv is not None else None)

        def e2e_call():
            sm.mergesort_stable(hwk, hwv, key_type=kt, stream=stream)
        h2d = d2h = in_bytes
    e2e_call()
    torch.cuda.synchronize(dev)
    e2e_ms = 0.0
    for _ in range(a.e2e_steps):
        if c["kind"] == "sort":
            hwk.copy_(hk)
            if hwv is not None:
                hwv.copy_(hv)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        e2e_call()     # binding synchronises the stream for host outputs
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms += e0.elapsed_time(e1)
    e2e_ms = max_over_ranks(e2e_ms, world)
    res["e2e"] = {"value": world * elems * a.e2e_steps / (e2e_ms / 1e3), "unit": "elements/s",
                  "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": a.e2e_steps,
                  "path": "C ABI with pinned host buffers (library stages H2D, kernels, D2H)"}
    res["host_input"] = (h if c["kind"] == "merge" else (hk, hv))
    clocks.stop()
    return res


def cpu_oracle_sample(cfg, host_input, budget_s):
    """The oracle as it stands, single thread, on a bounded sample of the
    workload: whole-workload calls repeated for ~budget_s, or a prefix sample
    if one call would exceed it."""
    import oracle
    c = synth.CONFIGS[cfg]
    kt = c["key_type"]
    reps, elems, t = 0, 0, 0.0
    if c["kind"] == "merge":
        h = host_input
        frac = 1.0
        t0 = time.perf_counter()
        oracle.merge(h.a_keys[:1 << 16], None if h.a_vals is None else h.a_vals[:1 << 16],
                     h.b_keys[:1 << 16], None if h.b_vals is None else h.b_vals[:1 << 16], kt)
        est = (time.perf_counter() - t0) / (1 << 17) * (h.n + h.m)
        if est > budget_s:
            frac = budget_s / est
        na, nb = max(1, int(h.n * frac)), max(1, int(h.m * frac))
        A, AV = h.a_keys[:na], None if h.a_vals is None else h.a_vals[:na]
        B, BV = h.b_keys[:nb], None if h.b_vals is None else h.b_vals[:nb]
        while t < budget_s or reps == 0:
            t0 = time.perf_counter()
            oracle.merge(A, AV, B, BV, kt)
            t += time.perf_counter() - t0
            reps += 1
            elems += na + nb
        sample = (f"oracle_merge (two-pointer, 1 thread) on {'the full workload' if frac == 1.0 else f'prefixes A[:{na}], B[:{nb}] of the workload'}"
                  f", {reps} repetition(s), {t:.1f} s")
    else:
        hk, hv = host_input
        N = hk.numel()
        Ns = min(N, 1 << 22)
        while t < budget_s or reps == 0:
            t0 = time.perf_counter()
            oracle.sort(hk[:Ns], None if hv is None else hv[:Ns], kt)
            t += time.perf_counter() - t0
            reps += 1
            elems += Ns
        sample = (f"oracle_sort (bottom-up stable merge sort, 1 thread) on the first {Ns} of {N} input elements, "
                  f"{reps} repetition(s), {t:.1f} s (sort cost grows as N log N: this per-element rate "
                  f"over-states the full-size CPU rate)")
    return {"value": elems / t, "unit": "elements/s", "cores": 1, "kind": "oracle", "sample": sample,
            "host_cores_available": os.cpu_count()}


# ------------------------------------------------------------- reference
def run_reference(a):
    """Reference arm of this tier: the CPU oracle, as it stands, each step a
    bounded sample of the workload sized so the whole run takes ~1-2 min."""
    import oracle
    oracle.build()
    cfg = a.config
    c = synth.CONFIGS[cfg]
    kt = c["key_type"]
    total_budget = 90.0
    per_step = total_budget / max(1, a.steps + a.warmup)
    if c["kind"] == "merge":
        h = synth.merge_input(c["n"], c["m"], kt, c["dist"], synth.BASE_SEED + cfg, c["payload"])
        t0 = time.perf_counter()
        oracle.merge(h.a_keys[:1 << 16], None if h.a_vals is None else h.a_vals[:1 << 16], h.b_keys[:1 << 16],
                     None if h.b_vals is None else h.b_vals[:1 << 16], kt)
        ns = (time.perf_counter() - t0) / (1 << 17)
        frac = min(1.0, per_step / (ns * (h.n + h.m)))
        na, nb = max(1, int(h.n * frac)), max(1, int(h.m * frac))
        args = (h.a_keys[:na], None if h.a_vals is None else h.a_vals[:na], h.b_keys[:nb],
                None if h.b_vals is None else h.b_vals[:nb], kt)
        fn = lambda: oracle.merge(*args)
        elems = na + nb
        sample = f"oracle_merge on prefixes A[:{na}], B[:{nb}] of the workload per step"
    else:
        s = synth.sort_input(c["N"], kt, c["dist"], synth.BASE_SEED + cfg, c["payload"])
        Ns = 1 << 16
        t0 = time.perf_counter()
        oracle.sort(s.keys[:Ns], None if s.vals is None else s.vals[:Ns], kt)
        ns = (time.perf_counter() - t0) / Ns
        Ns = int(max(1 << 12, min(c["N"], per_step / ns)))
        args = (s.keys[:Ns], None if s.vals is None else s.vals[:Ns], kt)
        fn = lambda: oracle.sort(*args)
        elems = Ns
        sample = f"oracle_sort on the first {Ns} of {c['N']} input elements per step"
    for _ in range(a.warmup):
        fn()
    t = 0.0
    for _ in range(a.steps):
        t0 = time.perf_counter()
        fn()
        t += time.perf_counter() - t0
    value = elems * a.steps / t
    return {
        "impl": "reference",
        "metric": load_json("BASELINE.json")["metric"],
        "value": value, "unit": "elements/s", "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": 1e3 * t / a.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": kt, "data": "synthetic",
        "config": {"workload": CONFIG_NAMES[cfg], "elements_per_step_sampled": elems},
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "elements/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    a = args_()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if a.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(a)), flush=True)
        return
    world, rank, local = dist_setup(a.gpus)
    r = run_ours(a, world, rank, local)
    if rank != 0:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    cfg = a.config
    c = synth.CONFIGS[cfg]
    peak, peak_src = hbm_peak()
    elems = elements_of(cfg)
    alg = step_bytes(cfg)
    line = {
        "metric": load_json("BASELINE.json")["metric"],
        "value": r["value"], "unit": "elements/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": c["key_type"] + ("+u32" if c["payload"] else ""), "data": "synthetic",
        "config": {"workload": CONFIG_NAMES[cfg], "elements_per_gpu_step": elems, "key_type": c["key_type"],
                   "payload": c["payload"], "dist": c["dist"], "seed": f"{synth.BASE_SEED + cfg:#x} + 1000*rank",
                   "l2": ("per-step events, L2 flushed (2x L2 write) and sort input restored between timed steps"
                          if r["per_step_events"] else
                          f"inputs+output {alg / 1e9:.2f} GB > 126 MB L2: no flush, back-to-back steps"),
                   "parallelism": f"replicas x{world}" if world > 1 else "1 GPU"},
        "achieved_hbm_gbs": step_alg_bytes(cfg) / (r["ms_per_step"] * 1e-3) / 1e9,
        "algorithmic_bytes_per_step": step_alg_bytes(cfg),
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
    }
    line["achieved_hbm_frac"] = line["achieved_hbm_gbs"] / peak
    if "kernels" in r:
        k2_ms, k2_n = r["kernels"]["k_tasks"]
        k1_ms, k1_n = r["kernels"]["k_cross_ranks"]
        k3_ms, k3_n = r["kernels"]["k_block_sort"]
        if c["kind"] == "sort":
            per_launch_bytes = 2 * elems * synth.elem_bytes(c["key_type"], c["payload"])
        else:
            per_launch_bytes = alg
        k2_avg = k2_ms / max(1, k2_n)
        achieved = per_launch_bytes / (k2_avg * 1e-3) / 1e9
        traffic, tsrc = traffic_from_profiles(cfg)
        line["roofline"] = {"bound": "hbm", "kernel": "k_tasks (K2: classify + copy/merge)",
                            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                            "traffic": traffic, "traffic_source": tsrc, "peak_source": peak_src,
                            "algorithmic_bytes_per_launch": per_launch_bytes,
                            "avg_launch_ms": k2_avg,
                            "share_of_step": k2_ms / max(1e-9, k1_ms + k2_ms + k3_ms),
                            "k_cross_ranks_avg_ms": k1_ms / max(1, k1_n),
                            "k_cross_ranks_ms_per_step": k1_ms / r["kernels"]["steps"],
                            "k_tasks_ms_per_step": k2_ms / r["kernels"]["steps"],
                            "k_block_sort_avg_ms": (k3_ms / k3_n) if k3_n else None}
    if "e2e" in r:
        line["e2e"] = r["e2e"]
    if world == 1 and not a.no_extras:
        line["cpu_baseline"] = cpu_oracle_sample(cfg, r["host_input"], a.cpu_seconds)
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
