"""The sharded multi-GPU merge sort (paper_1202_6575_b200.distributed.
mergesort_stable_sharded) on CPU with the gloo
backend at world sizes 2-5 (powers of two and not: odd trailing runs,
unequal p_A / p_B, empty blocks), with the oracle's rank / merge / sort
standing in for the local GPU primitives (test seam only).  The ranks'
output blocks, concatenated, must be the oracle's stable sort of the whole
array, keys and payloads, and rank r must hold exactly block r."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from test_distributed import OracleOps, _free_port


class OracleSortOps(OracleOps):
    def __init__(self, kt, descending=False):
        super().__init__(kt)
        self.desc = descending

    def ranks(self, X, keys, high):
        f = oracle.rank_high if high else oracle.rank_low
        xs = oracle.as_np(X, self.kt)
        ks = oracle.u128_ints(keys) if self.kt == "u128" else oracle.as_np(keys, self.kt)
        return torch.tensor([f(k, xs, self.kt, descending=self.desc) for k in ks], dtype=torch.int64)

    def merge(self, ak, av, bk, bv):
        ck, cv = oracle.merge(ak, av, bk, bv, self.kt, descending=self.desc)
        return self._t(ck), (None if cv is None else torch.from_numpy(cv.view(np.int32).copy()))

    def sort(self, keys, vals):
        sk, sv = oracle.sort(keys, vals, self.kt, descending=self.desc)
        return self._t(sk), (None if sv is None else torch.from_numpy(sv.view(np.int32).copy()))

    def _t(self, k):
        if self.kt == "u128":
            return torch.from_numpy(np.ascontiguousarray(k).view(np.int64).reshape(-1, 2).copy())
        ct = synth.KEY_TYPES[self.kt][0]
        return torch.from_numpy(np.ascontiguousarray(k).view(np.int32 if ct == torch.int32 else np.int64).copy())


def _worker(rank, world, port, cases, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1202_6575_b200 import distributed as D
        for case in cases:
            N, kt, dname, payload, desc = case
            inp = synth.sort_input(N, kt, dname, seed=N + world, payload=payload)
            xs = D.block_starts(N, world)
            k = inp.keys[xs[rank]:xs[rank + 1]].clone()
            v = None if inp.vals is None else inp.vals[xs[rank]:xs[rank + 1]].clone()
            sk, sv = D.mergesort_stable_sharded(k, v, N, key_type=kt, descending=desc,
                                                ops=OracleSortOps(kt, desc))
            got = [None] * world
            dist.all_gather_object(got, (sk, sv))
            if rank == 0:
                ok = all(got[q][0].shape[0] == xs[q + 1] - xs[q] for q in range(world))
                keys = torch.cat([g[0] for g in got])
                wk, wv = oracle.sort(inp.keys, inp.vals, kt, descending=desc)
                ok = ok and np.array_equal(oracle.as_np(keys, kt).view(np.uint8), wk.view(np.uint8))
                if payload:
                    vals = torch.cat([g[1] for g in got])
                    ok = ok and np.array_equal(oracle.vals_np(vals), wv)
                out.put((case, ok))
    finally:
        dist.destroy_process_group()


CASES = [(0, "u32", "bounded:5", True, False), (1, "u32", "bounded:5", True, False),
         (3, "i32", "full", True, False), (257, "u32", "bounded:7", True, False),
         (1000, "i64", "bounded:3", True, False), (999, "u64", "full", False, False),
         (777, "f32", "special", True, False), (1001, "i32", "bounded:9", True, True),
         (513, "u128", "tuple:4", True, False), (640, "u128", "tuple:4", True, True)]


@pytest.mark.parametrize("world", [2, 3, 4, 5])
def test_sharded_sort_gloo(world):
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    mp.spawn(_worker, args=(world, _free_port(), CASES, out), nprocs=world, join=True)
    res = [out.get(timeout=5) for _ in CASES]
    bad = [c for c, ok in res if not ok]
    assert not bad, bad
