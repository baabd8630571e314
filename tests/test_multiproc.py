"""N>1 host logic of bench.py on CPU with the gloo backend (world size 2).

bench.py at N>1 runs the sharded merge of the paper's BSP form (DESIGN.md
§8): rank r holds block r of A and B, one all-reduce of cross ranks, one
exchange; the reported value is all ranks' elements over the max-over-ranks
device time.  These tests cover that logic without a GPU (the oracle's
primitives stand in for the library), plus the max-over-ranks and
whole-job aggregation helpers with per-rank replicas.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench
import oracle
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # per-rank device time: the job value must use the slowest rank
        t_ms = 10.0 * (rank + 1)
        t_max = bench.max_over_ranks(t_ms, world, device="cpu")
        # replicas: distinct seeded inputs, each merged independently
        seed = bench.rank_seed(2, rank)
        inp = synth.merge_input(3000, 2000, "i32", "full", seed, payload=True)
        ck, cv = oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, "i32")
        digest = torch.tensor([int(np.int64(ck.astype(np.int64).sum()))], dtype=torch.int64)
        gathered = [torch.zeros_like(digest) for _ in range(world)]
        dist.all_gather(gathered, digest)
        dist.barrier()
        out.put((rank, t_max, seed, [int(g.item()) for g in gathered],
                 bool(np.all(ck[1:] >= ck[:-1])), int(cv.size)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_gloo_world2_replicas_and_max_over_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=150) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [20.0, 20.0]                 # max over ranks, seen by every rank
    assert res[0][2] != res[1][2]                              # distinct replica seeds
    assert res[0][3] == res[1][3] and res[0][3][0] != res[0][3][1]   # distinct replicas, same view
    assert all(r[4] and r[5] == 5000 for r in res)


def test_aggregate_value_is_whole_job():
    # 2 ranks x 1000 elements x 10 steps in 20 ms (max over ranks) = 1e6 elements/s
    assert bench.aggregate_value(1000, 2, 10, 20.0) == pytest.approx(1e6)
    assert bench.max_over_ranks(3.5, 1) == 3.5


def test_reference_arm_prints_one_json_line():
    """`bench.py --impl reference` (the CPU oracle as the reference arm) runs
    without a GPU and prints the contract's JSON line."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "1",
                        "--warmup", "1"], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["higher_is_better"] is True


def _sharded_worker(rank, world, port, out):
    """bench.py's N > 1 step (ShardedMergeWork -> distributed.merge_stable_sharded)
    on CPU with gloo, the oracle's primitives standing in for the library."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from test_distributed import OracleOps
        wl = bench.ShardedMergeWork(rank, world, torch.device("cpu"), n_per=3000, ops=OracleOps("i32"))
        for _ in range(2):                               # steps are repeatable
            wl.call()
        pieces = [(p.offset, p.keys) for p in wl.pieces]
        blocks = [None] * world
        dist.all_gather_object(blocks, (wl.a_keys, wl.b_keys))
        allp = [None] * world
        dist.all_gather_object(allp, pieces)
        recv_max = bench.max_over_ranks(float(wl.stats["recv_bytes"]), world, device="cpu")
        if rank == 0:
            A = torch.cat([b[0] for b in blocks])
            B = torch.cat([b[1] for b in blocks])
            want, _ = oracle.merge(A, None, B, None, "i32")
            ps = sorted((pc for g in allp for pc in g), key=lambda t: t[0])
            tiled = all(ps[i][0] + ps[i][1].numel() == ps[i + 1][0] for i in range(len(ps) - 1)) and ps[0][0] == 0
            got = oracle.as_np(torch.cat([p[1] for p in ps]), "i32")
            out.put((tiled, bool(np.array_equal(got, want)), wl.elems, wl.n, recv_max, wl.stats["local_bytes"]))
        else:
            out.put(None)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(180)
def test_gloo_world2_bench_sharded_step():
    """The N > 1 bench step is the sharded merge of the paper's BSP form
    (§3): rank r holds block r of A and B, the pieces of
    both ranks tile [0, n+m) and equal the oracle's merge of the global
    arrays; per-rank work is fixed (weak scaling), and the exchange volume
    (max over ranks) stays below the local input."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=150) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    tiled, equal, elems, n, recv_max, local = next(r for r in res if r is not None)
    assert tiled and equal
    assert elems == 6000 and n == 6000
    assert 0 <= recv_max < local
