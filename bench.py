#!/usr/bin/env python
"""Benchmark of the B200 stable merge (arXiv 1202.6575) -- driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 2]

A step is one pass of the hot path over one batch of synthetic input.  The
headline workload (--config 2, the default) is BASELINE.json configs[1],
the configuration this tier's bench convention designates (BASELINE.json's
metric names no config itself): stable merge keys-only, n = m = 2^26 int32
full range; a step is one merge_stable call = K1 cross ranks + K2
classify/copy/merge (rows a0-a7).  --config 5 benches the merge sort (rows
a8-a9); configs 1, 3, 4 the other merges.  Inputs are seeded and synthetic
(synth/), resident in HBM before the timed region.  In the same run, after
the headline, `per_config` measures all five BASELINE configs (ms per step,
elements/s, achieved GB/s, the dominant kernels' per-launch times and
roofline fractions, clocks) -- skipped with --no-per-config / --no-extras.

Multi-GPU (torchrun, N > 1): the paper's BSP form (§3,
SURVEY §8(e)) -- rank r holds block r of A and of B (C2-class shards,
2^26 + 2^26 int32 per rank, so the global merge grows with N: weak
scaling), and a step is one distributed.merge_stable_sharded call: one
all-gather of block-start keys, the local rank kernels, ONE all-reduce (the
single synchronisation), the task plan, one NCCL exchange of each task's
foreign range, the local merges.  value = all ranks' elements / the
max-over-ranks device time.

Rank 0 prints ONE JSON line.  `roofline` is for the dominant kernel (K2,
k_tasks; K3H k_block_sort_hbm for the sort when it dominates), timed live
with CUDA events on its launch stream (sm_profile_*); `cpu_baseline` is the
CPU oracle (oracle/, single thread) on a bounded sample of the same
workload; `e2e` is the same metric through the C ABI with pinned HOST
buffers (host->device and device->host copies inside the timed region).
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
    6: "B1 batched stable merges: 2^16 pairs, lengths uniform in [0,2^11) per side, u32 keys in [0,2^16) + u32 "
       "payload (SURVEY.md §8(f) row 1; not a BASELINE.json config)",
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
    ap.add_argument("--config", type=int, choices=sorted(synth.CONFIGS), default=2,
                    help="1-5: BASELINE.json configs[0..4] (2 = the metric's workload); 6: batched merges (NEXT row)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="bounded CPU-oracle sample budget")
    ap.add_argument("--no-extras", action="store_true", help="timed loop only (for ncu launch lists)")
    ap.add_argument("--no-per-config", action="store_true", help="skip the per-config measurements of C1-C5")
    ap.add_argument("--peer-access", action="store_true",
                    help="N > 1: the sharded merge reads foreign ranges through CUDA IPC instead of the NCCL exchange")
    ap.add_argument("--sort-ways", type=int, choices=[0, 2, 4], default=0,
                    help="merge sort phase 2: 0 = automatic (default), 4 = two merge rounds per HBM pass, "
                         "2 = one round per pass")
    ap.add_argument("--merge-path", action="store_true",
                    help="merges only: time the equal-output merge-path COMPARISON instead of the paper's method")
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


def traffic_from_profiles(cfg):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p)).get(str(cfg))
    if not d:
        return None, None
    return d.get("dram_bytes_per_launch"), d.get("source")


# -------------------------------------------------------------- workloads
class Workload:
    """One bench workload: its inputs resident in HBM, the timed call, the
    algorithmic bytes, the end-to-end (host-buffer) call and the bounded CPU
    oracle sample."""

    def __init__(self, cfg, seed, dev):
        self.cfg, self.c, self.dev = cfg, synth.CONFIGS[cfg], dev
        self.kt = self.c["key_type"]
        self.eb = synth.elem_bytes(self.kt, self.c["payload"])

    passes = 1                                  # HBM passes of the algorithmic bytes

    def k2_launch_bytes(self):  # noqa: E301
        """Algorithmic bytes of one launch of the dominant kernel K2 (SURVEY
        §8(d): read A+B + write C, keys + payload)."""
        return 2 * self.elems * self.eb

    def step_bytes(self):
        return self.k2_launch_bytes() * self.passes

    def prep(self):
        pass


class MergeWork(Workload):
    def __init__(self, cfg, seed, dev, sm):
        super().__init__(cfg, seed, dev)
        c, kt = self.c, self.kt
        self.inp = synth.merge_input(c["n"], c["m"], kt, c["dist"], seed, c["payload"], device=dev)
        n, m = self.inp.n, self.inp.m
        self.elems = n + m
        self.out_k = torch.empty(n + m, dtype=self.inp.a_keys.dtype, device=dev)
        self.out_v = torch.empty(n + m, dtype=torch.int32, device=dev) if c["payload"] else None
        self.sm = sm

    merge_path = False

    def call(self):
        i = self.inp
        self.sm.merge_stable(i.a_keys, i.a_vals, i.b_keys, i.b_vals, self.out_k, self.out_v, key_type=self.kt,
                             merge_path=self.merge_path)

    def e2e_setup(self, stream):
        h = self.host = self.inp.to("cpu")
        pin = lambda t: None if t is None else t.pin_memory()
        self.h_args = (pin(h.a_keys), pin(h.a_vals), pin(h.b_keys), pin(h.b_vals),
                       torch.empty(self.elems, dtype=h.a_keys.dtype).pin_memory(),
                       torch.empty(self.elems, dtype=torch.int32).pin_memory() if self.c["payload"] else None)
        self.stream = stream
        return self.elems * self.eb, self.elems * self.eb       # H2D, D2H bytes

    def e2e_call(self):
        self.sm.merge_stable(*self.h_args, key_type=self.kt, stream=self.stream)

    def oracle_sample(self, budget_s):
        import oracle
        h, kt = self.host, self.kt
        t0 = time.perf_counter()
        oracle.merge(h.a_keys[:1 << 16], None if h.a_vals is None else h.a_vals[:1 << 16],
                     h.b_keys[:1 << 16], None if h.b_vals is None else h.b_vals[:1 << 16], kt)
        est = (time.perf_counter() - t0) / (1 << 17) * (h.n + h.m)
        frac = min(1.0, budget_s / est) if est > 0 else 1.0
        na, nb = max(1, int(h.n * frac)), max(1, int(h.m * frac))
        args = (h.a_keys[:na], None if h.a_vals is None else h.a_vals[:na],
                h.b_keys[:nb], None if h.b_vals is None else h.b_vals[:nb], kt)
        what = "the full workload" if frac == 1.0 else f"prefixes A[:{na}], B[:{nb}] of the workload"
        return lambda: oracle.merge(*args), na + nb, f"oracle_merge (two-pointer, 1 thread) on {what}"


class SortWork(Workload):
    def __init__(self, cfg, seed, dev, sm):
        super().__init__(cfg, seed, dev)
        c, kt = self.c, self.kt
        self.src = synth.sort_input(c["N"], kt, c["dist"], seed, c["payload"], device=dev)
        self.elems = c["N"]
        self.work_k = self.src.keys.clone()
        self.work_v = self.src.vals.clone() if self.src.vals is not None else None
        self.sm = sm
        import math
        R = sm.sort_run(kt, c["payload"], c["N"])     # phase 1's run length for this N
        self.rounds = max(0, math.ceil(math.log2(c["N"] / R)))      # the paper's merge rounds
        # HBM passes: the block sort + one per merge pass (the library's plan:
        # two rounds per pass where sm_set_sort_ways selects it)
        self.merge_passes = sm.sort_merge_passes(kt, c["payload"], c["N"])
        self.passes = 1 + self.merge_passes

    def prep(self):                              # restore the unsorted input (untimed)
        self.work_k.copy_(self.src.keys)
        if self.work_v is not None:
            self.work_v.copy_(self.src.vals)

    def call(self):
        self.sm.mergesort_stable(self.work_k, self.work_v, key_type=self.kt)

    def e2e_setup(self, stream):
        self.hk = self.src.keys.cpu().pin_memory()
        self.hv = self.src.vals.cpu().pin_memory() if self.src.vals is not None else None
        self.hwk = self.hk.clone().pin_memory()
        self.hwv = self.hv.clone().pin_memory() if self.hv is not None else None
        self.stream = stream
        return self.elems * self.eb, self.elems * self.eb

    def e2e_prep(self):
        self.hwk.copy_(self.hk)
        if self.hwv is not None:
            self.hwv.copy_(self.hv)

    def e2e_call(self):
        self.sm.mergesort_stable(self.hwk, self.hwv, key_type=self.kt, stream=self.stream)

    def oracle_sample(self, budget_s):
        import oracle
        N = self.hk.numel()
        Ns = min(N, 1 << 22)
        args = (self.hk[:Ns], None if self.hv is None else self.hv[:Ns], self.kt)
        return (lambda: oracle.sort(*args), Ns,
                f"oracle_sort (bottom-up stable merge sort, 1 thread) on the first {Ns} of {N} input elements "
                f"(sort cost grows as N log N: this per-element rate over-states the full-size CPU rate)")


class BatchWork(Workload):
    def __init__(self, cfg, seed, dev, sm):
        super().__init__(cfg, seed, dev)
        c, kt = self.c, self.kt
        self.inp = synth.batch_input(c["S"], c["mean"], kt, c["dist"], seed, c["payload"], device=dev)
        self.elems = self.inp.n + self.inp.m
        self.out_k = torch.empty(self.elems, dtype=self.inp.a_keys.dtype, device=dev)
        self.out_v = torch.empty(self.elems, dtype=torch.int32, device=dev) if c["payload"] else None
        self.sm = sm

    def call(self):
        i = self.inp
        self.sm.merge_stable_batched(i.a_keys, i.a_vals, i.a_offsets, i.b_keys, i.b_vals, i.b_offsets,
                                     self.out_k, self.out_v, key_type=self.kt)

    def e2e_setup(self, stream):
        # the batched entry takes device buffers: e2e = pinned H2D copies of
        # the inputs and offsets, the call, and the D2H copy of the output
        self.host = self.inp.to("cpu")
        h = self.host
        pin = lambda t: None if t is None else t.pin_memory()
        self.h_in = [pin(t) for t in (h.a_keys, h.a_vals, h.a_offsets, h.b_keys, h.b_vals, h.b_offsets)]
        self.d_in = [None if t is None else torch.empty_like(t, device=self.dev) for t in self.h_in]
        self.h_out = [torch.empty(self.elems, dtype=h.a_keys.dtype).pin_memory(),
                      torch.empty(self.elems, dtype=torch.int32).pin_memory() if self.c["payload"] else None]
        self.stream = stream
        h2d = sum(t.numel() * t.element_size() for t in self.h_in if t is not None)
        d2h = sum(t.numel() * t.element_size() for t in self.h_out if t is not None)
        return h2d, d2h

    def e2e_call(self):
        with torch.cuda.stream(self.stream):
            for d, h in zip(self.d_in, self.h_in):
                if d is not None:
                    d.copy_(h, non_blocking=True)
            ak, av, ao, bk, bv, bo = self.d_in
            self.sm.merge_stable_batched(ak, av, ao, bk, bv, bo, self.out_k, self.out_v, key_type=self.kt)
            self.h_out[0].copy_(self.out_k, non_blocking=True)
            if self.out_v is not None:
                self.h_out[1].copy_(self.out_v, non_blocking=True)
        self.stream.synchronize()

    def oracle_sample(self, budget_s):
        import oracle
        h, kt = self.host, self.kt
        ao, bo = h.a_offsets.numpy(), h.b_offsets.numpy()
        S = len(ao) - 1
        # a prefix of the segments, ~budget_s of per-segment oracle merges
        t0 = time.perf_counter()
        k = min(S, 64)
        for s in range(k):
            oracle.merge(h.a_keys[ao[s]:ao[s + 1]], None if h.a_vals is None else h.a_vals[ao[s]:ao[s + 1]],
                         h.b_keys[bo[s]:bo[s + 1]], None if h.b_vals is None else h.b_vals[bo[s]:bo[s + 1]], kt)
        est = (time.perf_counter() - t0) / k * S
        ks = max(1, min(S, int(S * budget_s / max(est, 1e-9))))

        def fn():
            for s in range(ks):
                oracle.merge(h.a_keys[ao[s]:ao[s + 1]], None if h.a_vals is None else h.a_vals[ao[s]:ao[s + 1]],
                             h.b_keys[bo[s]:bo[s + 1]], None if h.b_vals is None else h.b_vals[bo[s]:bo[s + 1]],
                             kt)
        elems = int(ao[ks] + bo[ks])
        return fn, elems, f"oracle_merge per segment (1 thread) on the first {ks} of {S} segments"


def make_workload(cfg, seed, dev, sm):
    kind = synth.CONFIGS[cfg]["kind"]
    return {"merge": MergeWork, "sort": SortWork, "batch": BatchWork}[kind](cfg, seed, dev, sm)


# ------------------------------------------------------------ N > 1: sharded
class ShardedMergeWork(Workload):
    """N > 1: the paper's BSP form (§3).  Rank
    r holds block r of A and of B (C2-class: n_per = 2^26 int32 full-range
    keys per array per rank; the global merge is n = m = world * n_per); one
    step is one distributed.merge_stable_sharded call.  `ops` is the test
    seam of distributed.py (None: the CUDA library); `peer_access` selects
    the CUDA-IPC path instead of the NCCL exchange."""

    def __init__(self, rank, world, dev, n_per=1 << 26, ops=None, peer_access=False, group=None):
        from paper_1202_6575_b200 import distributed as D
        self.cfg, self.c, self.dev = 2, dict(synth.CONFIGS[2]), dev
        self.kt = "i32"
        self.eb = synth.elem_bytes("i32", False)
        self.rank, self.world, self.n_per = rank, world, n_per
        a, b = synth.sharded_merge_blocks(n_per, world, rank, synth.BASE_SEED + 2, device=dev)
        self.a_keys, self.b_keys = a, b
        self.n = self.m = n_per * world
        self.elems = 2 * n_per                      # per rank
        self.ops = ops if ops is not None else D.CudaOps("i32")
        self.peer_access, self.group = peer_access, group
        self.pieces, self.stats = [], {}

    def call(self):
        from paper_1202_6575_b200 import distributed as D
        self.stats = {}
        self.pieces = D.merge_stable_sharded(self.a_keys, None, self.b_keys, None, self.n, self.m, key_type=self.kt,
                                             ops=self.ops, peer_access=self.peer_access, group=self.group,
                                             stats=self.stats)


# ------------------------------------------------------------------ ours
def _time_steps(wl, steps, stream, dev, prep, per_step_events, world):
    """Device time of `steps` steps (CUDA events on the launch stream),
    max over ranks; back-to-back when the inputs exceed L2, else one event
    pair per step with L2 flushed in between (prep)."""
    barrier(world)
    torch.cuda.synchronize(dev)
    t_wall0 = time.time()
    if not per_step_events:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            wl.call()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t_ms = e0.elapsed_time(e1)
    else:
        evs = []
        for _ in range(steps):
            prep()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            wl.call()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize(dev)
        t_ms = sum(x.elapsed_time(y) for x, y in evs)
    t_wall1 = time.time()
    barrier(world)
    return max_over_ranks(t_ms, world), t_wall0, t_wall1


def _kernel_profile(wl, sm, steps, prep, dev):
    """Per-kernel durations (the library's CUDA-event profiler, events on
    each kernel's own launch stream; profiling turns PDL off)."""
    sm.profile_enable(True)
    for _ in range(steps):
        prep()
        wl.call()
    torch.cuda.synchronize(dev)
    k = {"k_cross_ranks": sm.profile_read(sm.PROF_K1), "k_tasks": sm.profile_read(sm.PROF_K2),
         "k_block_sort": sm.profile_read(sm.PROF_K3), "steps": steps}
    sm.profile_enable(False)
    return k


def _roofline(wl, kernels, peak, peak_src, cfg):
    """The dominant kernel's roofline: algorithmic bytes per launch (SURVEY
    §8(d): read + write, keys + payload) over its average launch time."""
    k2_ms, k2_n = kernels["k_tasks"]
    k1_ms, k1_n = kernels["k_cross_ranks"]
    k3_ms, k3_n = kernels["k_block_sort"]
    steps = kernels["steps"]
    per_launch_bytes = wl.k2_launch_bytes()
    k2_avg = k2_ms / max(1, k2_n)
    achieved = per_launch_bytes / (k2_avg * 1e-3) / 1e9
    traffic, tsrc = traffic_from_profiles(cfg)
    out = {"bound": "hbm", "kernel": "k_tasks (K2: classify + copy/merge)",
           "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
           "traffic": traffic, "traffic_source": tsrc, "peak_source": peak_src,
           "algorithmic_bytes_per_launch": per_launch_bytes,
           "avg_launch_ms": k2_avg,
           "share_of_step": k2_ms / max(1e-9, k1_ms + k2_ms + k3_ms),
           "k_cross_ranks_avg_ms": k1_ms / max(1, k1_n),
           "k_cross_ranks_ms_per_step": k1_ms / steps,
           "k_tasks_ms_per_step": k2_ms / steps,
           "k_block_sort_avg_ms": (k3_ms / k3_n) if k3_n else None}
    if k3_n:
        # phase 1 (row a8): its algorithmic bytes are one read + one write of
        # the input (its radix passes move more: that is the kernel's cost)
        k3_avg = k3_ms / k3_n
        b3 = 2 * wl.elems * wl.eb
        out["k_block_sort"] = {"avg_launch_ms": k3_avg, "algorithmic_bytes_per_launch": b3,
                               "achieved": b3 / (k3_avg * 1e-3) / 1e9, "frac": b3 / (k3_avg * 1e-3) / 1e9 / peak}
    return out


def _measure_config(cfg, sm, dev, stream, steps, warmup, peak, peak_src, clocks):
    """One BASELINE config at N = 1 (per_config): time, kernels, roofline."""
    wl = make_workload(cfg, rank_seed(cfg, 0), dev, sm)
    per_step_events = wl.c["kind"] == "sort" or wl.step_bytes() < 4 * L2_BYTES
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev) if per_step_events else None

    def prep():
        wl.prep()
        if flush is not None:
            flush.add_(1)

    for _ in range(warmup):
        prep()
        wl.call()
    t_ms, w0, w1 = _time_steps(wl, steps, stream, dev, prep, per_step_events, 1)
    kern = _kernel_profile(wl, sm, max(3, steps), prep, dev)
    ms = t_ms / steps
    roof = _roofline(wl, kern, peak, peak_src, cfg)
    out = {"workload": CONFIG_NAMES[cfg], "steps": steps, "ms_per_step": ms,
           "elements_per_s": wl.elems / (ms * 1e-3),
           "achieved_hbm_gbs": wl.step_bytes() / (ms * 1e-3) / 1e9,
           "achieved_hbm_frac": wl.step_bytes() / (ms * 1e-3) / 1e9 / peak,
           "algorithmic_bytes_per_step": wl.step_bytes(),
           "k_tasks_avg_ms": roof["avg_launch_ms"], "k_tasks_frac": roof["frac"],
           "k_tasks_ms_per_step": roof["k_tasks_ms_per_step"],
           "k_cross_ranks_ms_per_step": roof["k_cross_ranks_ms_per_step"],
           "clocks": clocks.summary(w0, w1)}
    if "k_block_sort" in roof:
        out["k_block_sort_ms"] = roof["k_block_sort"]["avg_launch_ms"]
        out["merge_rounds"] = wl.rounds
        out["merge_passes"] = wl.merge_passes
    del wl, flush
    torch.cuda.empty_cache()
    return out


def run_ours(a, world, rank, local):
    import paper_1202_6575_b200 as sm
    sm.set_sort_ways(a.sort_ways)

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = a.config
    clocks = ClockSampler(local).start()
    if world > 1:
        wl = ShardedMergeWork(rank, world, dev, peer_access=a.peer_access)   # inputs resident in HBM
    else:
        wl = make_workload(cfg, rank_seed(cfg, rank), dev, sm)
        wl.merge_path = a.merge_path
    per_step_events = world == 1 and (wl.c["kind"] == "sort" or wl.step_bytes() < 4 * L2_BYTES)
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev) if per_step_events else None

    def prep():
        wl.prep()
        if flush is not None:
            flush.add_(1)                             # write > L2 between timed steps

    stream = torch.cuda.current_stream(dev)
    for _ in range(a.warmup):
        prep()
        wl.call()
    if world > 1:
        l0 = wl.ops.launches
        wl.call()
        launches_per_step = wl.ops.launches - l0     # this rank's library launches in one sharded step
    else:
        wl.call()
        launches_per_step = sm.last_launch_count()
    torch.cuda.synchronize(dev)
    t_ms, t_wall0, t_wall1 = _time_steps(wl, a.steps, stream, dev, prep, per_step_events, world)
    clk = clocks.summary(t_wall0, t_wall1)

    res = dict(value=aggregate_value(wl.elems, world, a.steps, t_ms), ms_per_step=t_ms / a.steps,
               launches=None if launches_per_step is None else launches_per_step * a.steps, clocks=clk,
               per_step_events=per_step_events, wl=wl)
    if world > 1:
        # exchange volume of the sharded merge: max over ranks, against the
        # ~half-of-the-local-input bound of the paper's one exchange step
        st = wl.stats
        res["sharded"] = {"recv_bytes_max": int(max_over_ranks(float(st.get("recv_bytes", 0)), world)),
                          "local_input_bytes": int(st.get("local_bytes", 0)), "tasks": st.get("tasks"),
                          "peer_access": bool(a.peer_access),
                          "global_n": wl.n, "global_m": wl.m}
        clocks.stop()
        return res
    if a.no_extras:
        clocks.stop()
        return res

    res["kernels"] = _kernel_profile(wl, sm, max(3, min(a.steps, 50 if wl.c["kind"] == "sort" else 200)), prep, dev)

    # ---- end to end through the public API with pinned host buffers
    h2d, d2h = wl.e2e_setup(stream)
    wl.e2e_call()
    torch.cuda.synchronize(dev)
    e2e_ms = 0.0
    for _ in range(a.e2e_steps):
        if hasattr(wl, "e2e_prep"):
            wl.e2e_prep()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        wl.e2e_call()     # host outputs are ready when the call returns
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms += e0.elapsed_time(e1)
    res["e2e"] = {"value": aggregate_value(wl.elems, world, a.e2e_steps, e2e_ms), "unit": "elements/s",
                  "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": a.e2e_steps,
                  "path": "public API with pinned host buffers (H2D, kernels, D2H inside the timed region)"}
    res["cpu_baseline"] = cpu_oracle_sample(wl, a.cpu_seconds)

    # ---- every BASELINE config in the same run (per_config)
    if not a.no_per_config:
        peak, peak_src = hbm_peak()
        for attr in ("inp", "src", "work_k", "work_v", "out_k", "out_v", "h_args", "host", "hk", "hv", "hwk", "hwv"):
            if hasattr(wl, attr):
                setattr(wl, attr, None)
        del flush
        torch.cuda.empty_cache()
        per = {}
        for c in (1, 2, 3, 4, 5):
            steps = 5 if synth.CONFIGS[c]["kind"] == "sort" else 20
            per[f"C{c}"] = _measure_config(c, sm, dev, stream, steps, 3, peak, peak_src, clocks)
        res["per_config"] = per
    clocks.stop()
    return res


def cpu_oracle_sample(wl, budget_s):
    """The oracle as it stands, single thread, on a bounded sample of the
    workload (whole-workload calls, or a prefix if one call exceeds the
    budget), repeated for ~budget_s."""
    fn, elems, what = wl.oracle_sample(budget_s)
    reps, t = 0, 0.0
    while t < budget_s or reps == 0:
        t0 = time.perf_counter()
        fn()
        t += time.perf_counter() - t0
        reps += 1
    return {"value": elems * reps / t, "unit": "elements/s", "cores": 1, "kind": "oracle",
            "sample": f"{what}, {reps} repetition(s), {t:.1f} s", "host_cores_available": os.cpu_count()}


# ------------------------------------------------------------- reference
class _HostOnly:
    """Workload inputs on the host only (the reference arm has no GPU path)."""


def run_reference(a):
    """Reference arm of this tier: the CPU oracle, as it stands, each step a
    bounded sample of the workload sized so the whole run takes ~1-2 min."""
    import oracle
    oracle.build()
    cfg = a.config
    c = synth.CONFIGS[cfg]
    kt = c["key_type"]
    per_step = 90.0 / max(1, a.steps + a.warmup)
    wl = _HostOnly()
    wl.kt, wl.c = kt, c
    if c["kind"] == "merge":
        wl.host = synth.merge_input(c["n"], c["m"], kt, c["dist"], synth.BASE_SEED + cfg, c["payload"])
        fn, elems, what = MergeWork.oracle_sample(wl, per_step)
    elif c["kind"] == "batch":
        wl.host = synth.batch_input(c["S"], c["mean"], kt, c["dist"], synth.BASE_SEED + cfg, c["payload"])
        fn, elems, what = BatchWork.oracle_sample(wl, per_step)
    else:
        src = synth.sort_input(c["N"], kt, c["dist"], synth.BASE_SEED + cfg, c["payload"])
        Ns = 1 << 16
        t0 = time.perf_counter()
        oracle.sort(src.keys[:Ns], None if src.vals is None else src.vals[:Ns], kt)
        ns = (time.perf_counter() - t0) / Ns
        Ns = int(max(1 << 12, min(c["N"], per_step / ns)))
        args = (src.keys[:Ns], None if src.vals is None else src.vals[:Ns], kt)
        fn, elems, what = (lambda: oracle.sort(*args)), Ns, f"oracle_sort on the first {Ns} of {c['N']} elements"
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
        "cpu_baseline": {"value": value, "unit": "elements/s", "cores": 1, "kind": "oracle",
                         "sample": f"{what} per step"},
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
    wl = r["wl"]
    c = wl.c
    peak, peak_src = hbm_peak()
    sharded = "sharded" in r
    if sharded:
        parallelism = (f"sharded over {world} ranks: the paper's BSP form (rank r holds block r of A and B, "
                       f"one all-reduce of cross ranks, one {'CUDA-IPC' if a.peer_access else 'NCCL'} exchange)")
        workload = (f"C2-class sharded stable merge keys-only: n = m = {world} x 2^26 int32 full range "
                    f"(each rank: its 2^26 + 2^26 block pair)")
    else:
        parallelism = "1 GPU"
        workload = CONFIG_NAMES[cfg]
    line = {
        "metric": load_json("BASELINE.json")["metric"],
        "value": r["value"], "unit": "elements/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": c["key_type"] + ("+u32" if c["payload"] else ""), "data": "synthetic",
        "config": {"workload": workload, "elements_per_gpu_step": wl.elems, "key_type": c["key_type"],
                   "payload": c["payload"], "dist": c["dist"], "seed": f"{synth.BASE_SEED + cfg:#x} + 1000*rank",
                   "l2": ("per-step events, L2 flushed (2x L2 write) and sort input restored between timed steps"
                          if r["per_step_events"] else
                          f"inputs+output {wl.step_bytes() / 1e9:.2f} GB > 126 MB L2: no flush, back-to-back steps"),
                   "parallelism": parallelism,
                   "method": ("merge-path comparison (equal output tiles; NOT the paper's method)" if a.merge_path
                              else "paper: cross ranks + cases (a)-(e)")},
        "achieved_hbm_gbs": wl.step_bytes() / (r["ms_per_step"] * 1e-3) / 1e9,
        "algorithmic_bytes_per_step": wl.step_bytes(),
        "gpu_launches": r["launches"],
        "clocks": r["clocks"],
    }
    line["achieved_hbm_frac"] = line["achieved_hbm_gbs"] / peak
    if sharded:
        line["sharded"] = r["sharded"]
        line["achieved_hbm_gbs_note"] = "per GPU: local elements x 8 B / max-over-ranks step time"
    if "kernels" in r:
        line["roofline"] = _roofline(wl, r["kernels"], peak, peak_src, cfg)
    for key in ("e2e", "cpu_baseline", "per_config"):
        if key in r:
            line[key] = r[key]
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
