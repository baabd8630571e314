"""Sharded multi-GPU merge and sort timing, for a
multi-GPU node:

    torchrun --standalone --nproc-per-node N scripts/bench_sharded.py [--what merge|sort]
             [--elements 2^28] [--peer 0|1] [--steps 10]

Each rank holds the paper's block r of A and B (merge) or of the input
(sort), generated on its GPU; the timed region is the sharded call, max over
ranks of the CUDA-event time, barrier and synchronise on both sides.  Prints
one JSON line on rank 0.  Not part of the driver's bench contract."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_1202_6575_b200 import distributed as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="merge", choices=["merge", "sort"])
    ap.add_argument("--elements", type=int, default=1 << 28, help="elements per input array (merge) / in total (sort)")
    ap.add_argument("--peer", type=int, default=1, help="1: CUDA-IPC peer access, 0: NCCL point-to-point")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p, r = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cuda", local)
    if a.what == "merge":
        inp = synth.merge_input(a.elements, a.elements, "i32", "full", seed=7, payload=False, device=dev)
        x = D.block_starts(a.elements, p)
        ak, bk = inp.a_keys[x[r]:x[r + 1]].contiguous(), inp.b_keys[x[r]:x[r + 1]].contiguous()
        del inp
        call = lambda: D.merge_stable_sharded(ak, None, bk, None, a.elements, a.elements, key_type="i32", peer_access=bool(a.peer))
        elems, nbytes = 2 * a.elements, 2 * 2 * a.elements * 4
    else:
        xs = D.block_starts(a.elements, p)
        src = synth.sort_input(a.elements, "u32", "bounded:1048576", seed=7, payload=True, device=dev)
        k0, v0 = src.keys[xs[r]:xs[r + 1]].contiguous(), src.vals[xs[r]:xs[r + 1]].contiguous()
        del src
        call = lambda: D.mergesort_stable_sharded(k0.clone(), v0.clone(), a.elements, key_type="u32",
                                                  peer_access=bool(a.peer))
        elems, nbytes = a.elements, None
    for _ in range(2):
        call()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        call()
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1) / a.steps], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if r == 0:
        ms = float(t.item())
        line = {"what": f"sharded {a.what}", "n_gpus": p, "peer_access": bool(a.peer), "ms_per_call": ms,
                "elements_per_s": elems / (ms * 1e-3)}
        if nbytes:
            line["algorithmic_gbs"] = nbytes / (ms * 1e-3) / 1e9
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
