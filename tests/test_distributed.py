"""The sharded multi-GPU merge (paper_1202_6575_b200.distributed; SURVEY.md
§8(e), §8(f) row 3) on CPU with the gloo backend: the host logic -- block
starts, the all-reduce of partial ranks (the single synchronisation), the
2p-task plan, the one exchange round -- at world sizes 2-4, with the oracle's
rank and merge standing in for the two local GPU primitives (test seam only).
The concatenated pieces must be the oracle's global stable merge."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth


class OracleOps:
    """CPU stand-ins for the two local primitives (tests only)."""

    def __init__(self, kt):
        self.kt = kt

    def ranks(self, X, keys, high):
        f = oracle.rank_high if high else oracle.rank_low
        xs = oracle.as_np(X, self.kt)
        ks = oracle.as_np(keys, self.kt)
        return torch.tensor([f(k, xs, self.kt) for k in ks], dtype=torch.int64)

    def merge(self, ak, av, bk, bv):
        ck, cv = oracle.merge(ak, av, bk, bv, self.kt)
        ct = synth.KEY_TYPES[self.kt][0]
        keys = torch.from_numpy(ck.view(np.int32 if ct == torch.int32 else np.int64).copy())
        return keys, (None if cv is None else torch.from_numpy(cv.view(np.int32).copy()))


def _worker(rank, world, port, cases, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        for case in cases:
            _one(rank, world, case, out)
    finally:
        dist.destroy_process_group()


def _one(rank, world, case, out):
    if True:
        from paper_1202_6575_b200 import distributed as D
        n, m, kt, dist_name, payload = case
        inp = synth.merge_input(n, m, kt, dist_name, seed=n * 7 + m, payload=payload)
        x, y = D.block_starts(n, world), D.block_starts(m, world)
        ak, bk = inp.a_keys[x[rank]:x[rank + 1]], inp.b_keys[y[rank]:y[rank + 1]]
        av = None if inp.a_vals is None else inp.a_vals[x[rank]:x[rank + 1]]
        bv = None if inp.b_vals is None else inp.b_vals[y[rank]:y[rank + 1]]
        pieces = D.merge_stable_sharded(ak, av, bk, bv, n, m, ops=OracleOps(kt))
        gathered = [None] * world
        dist.all_gather_object(gathered, [(p.offset, p.keys, p.vals) for p in pieces])
        if rank == 0:
            allp = sorted((pc for g in gathered for pc in g), key=lambda t: t[0])
            keys = torch.cat([t[1] for t in allp]) if allp else inp.a_keys[:0]
            offs_ok = all(allp[i][0] + allp[i][1].numel() == allp[i + 1][0] for i in range(len(allp) - 1))
            vals = torch.cat([t[2] for t in allp]) if (allp and payload) else None
            wk, wv = oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, kt)
            ok = offs_ok and (not allp or allp[0][0] == 0)
            ok = ok and np.array_equal(oracle.as_np(keys, kt).view(np.uint8), wk.view(np.uint8))
            if payload:
                ok = ok and np.array_equal(oracle.vals_np(vals), wv)
            out.put((case, ok))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CASES = [
    (5000, 3000, "i32", "bounded:20", True),
    (4097, 9001, "u64", "mostly:0x8000000000000000:9/10", True),
    (6000, 6000, "f32", "special", False),
    (2, 7, "i32", "bounded:3", True),        # n < p: empty A blocks
    (3000, 0, "u32", "full", True),          # B empty
    (2000, 2500, "i64", "equal", True),      # all keys equal: C = A || B
]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3, 4])
def test_sharded_merge_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=250) for _ in CASES]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for case, ok in results:
        assert ok, (world, case)


def test_plan_tasks_tile_the_output():
    """The distributed plan (the library's host Steps 3-4, sm_plan_tasks) tiles
    [0, n+m) and partitions A and B, checked against the ranks of the oracle."""
    from paper_1202_6575_b200 import distributed as D
    for n, m, p in ((18, 15, 5), (1000, 37, 4), (7, 2000, 3), (0, 5, 2), (3, 1, 8)):
        inp = synth.merge_input(max(n, 1), max(m, 1), "i32", "bounded:5", seed=n + m)
        a = oracle.as_np(inp.a_keys, "i32")[:n]
        b = oracle.as_np(inp.b_keys, "i32")[:m]
        x, y = D.block_starts(n, p), D.block_starts(m, p)
        xbar = [oracle.rank_low(a[x[i]], b, "i32") if x[i] < n else m for i in range(p)] + [m]
        ybar = [oracle.rank_high(b[y[j]], a, "i32") if y[j] < m else n for j in range(p)] + [n]
        tasks = D.plan_tasks(n, m, p, xbar, ybar)
        spans = sorted((a0 + b0, a1 - a0 + b1 - b0) for _, a0, a1, b0, b1 in tasks)
        pos = 0
        for off, ln in spans:
            assert off == pos
            pos += ln
        assert pos == n + m
