"""The sharded merge on the GPU with the library's kernels (world size 1 over
NCCL: the collectives and the CUDA rank/merge primitives; the multi-rank
exchange is covered on CPU by tests/test_distributed.py -- one GPU here)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

import oracle
import synth
from gpu_util import assert_bit_exact, lib

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl1():
    lib()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()), RANK="0", WORLD_SIZE="1")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("kt,dist_name", [("i32", "full"), ("u64", "mostly:0x8000000000000000:9/10"),
                                          ("f32", "special")])
def test_sharded_merge_world1_cuda(nccl1, kt, dist_name):
    from paper_1202_6575_b200 import distributed as D
    inp = synth.merge_input(300001, 200003, kt, dist_name, seed=5, payload=True)
    d = inp.to("cuda")
    pieces = D.merge_stable_sharded(d.a_keys, d.a_vals, d.b_keys, d.b_vals, inp.n, inp.m, key_type=kt)
    pieces.sort(key=lambda p: p.offset)
    keys = torch.cat([p.keys for p in pieces]).cpu()
    vals = torch.cat([p.vals for p in pieces]).cpu()
    assert_bit_exact(keys, vals, *oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, kt), kt)


def test_ranks_stable_matches_oracle():
    sm = lib()
    for kt, dist_name in (("i32", "bounded:50"), ("u64", "full"), ("f64", "special")):
        inp = synth.merge_input(100003, 5000, kt, dist_name, seed=8, payload=False)
        X, keys = inp.a_keys.cuda(), inp.b_keys.cuda()
        lo = sm.ranks_stable(X, keys, False, key_type=kt).cpu().numpy()
        hi = sm.ranks_stable(X, keys, True, key_type=kt).cpu().numpy()
        xs, ks = oracle.as_np(inp.a_keys, kt), oracle.as_np(inp.b_keys, kt)
        sample = range(0, ks.size, 97)
        assert [lo[i] for i in sample] == [oracle.rank_low(ks[i], xs, kt) for i in sample]
        assert [hi[i] for i in sample] == [oracle.rank_high(ks[i], xs, kt) for i in sample]


@pytest.mark.parametrize("kt,dist_name,desc", [("u32", "bounded:1048576", False), ("i64", "bounded:1000", True),
                                               ("u128", "tuple:50", False)])
def test_sharded_sort_world1_cuda(nccl1, kt, dist_name, desc):
    """World size 1: phase 1 only (the library's sort through CudaOps); the
    multi-rank rounds are covered on CPU by tests/test_distributed_sort.py."""
    from paper_1202_6575_b200 import distributed as D
    inp = synth.sort_input(200003, kt, dist_name, seed=3)
    k, v = D.mergesort_stable_sharded(inp.keys.cuda(), inp.vals.cuda(), inp.N, key_type=kt, descending=desc)
    wk, wv = oracle.sort(inp.keys, inp.vals, kt, descending=desc)
    assert np.array_equal(oracle.as_np(k.cpu(), kt).view(np.uint8), wk.view(np.uint8))
    assert np.array_equal(oracle.vals_np(v.cpu()), wv)


def _peer_worker(rank, world, port, cases, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1202_6575_b200 import distributed as D
        for case in cases:
            n, m, kt, dist_name = case
            inp = synth.merge_input(n, m, kt, dist_name, seed=n + m, payload=True)
            x, y = D.block_starts(n, world), D.block_starts(m, world)
            ak = inp.a_keys[x[rank]:x[rank + 1]].cuda()
            av = inp.a_vals[x[rank]:x[rank + 1]].cuda()
            bk = inp.b_keys[y[rank]:y[rank + 1]].cuda()
            bv = inp.b_vals[y[rank]:y[rank + 1]].cuda()
            pieces = D.merge_stable_sharded(ak, av, bk, bv, n, m, key_type=kt, peer_access=True)
            got = [None] * world
            dist.all_gather_object(got, [(pc.offset, pc.keys.cpu(), pc.vals.cpu()) for pc in pieces])
            if rank == 0:
                allp = sorted((t for g in got for t in g), key=lambda t: t[0])
                keys = torch.cat([t[1] for t in allp])
                vals = torch.cat([t[2] for t in allp])
                wk, wv = oracle.merge(inp.a_keys, inp.a_vals, inp.b_keys, inp.b_vals, kt)
                ok = np.array_equal(oracle.as_np(keys, kt).view(np.uint8), wk.view(np.uint8)) and \
                    np.array_equal(oracle.vals_np(vals), wv)
                out.put((case, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_merge_peer_access_ipc(world):
    """peer_access=True: the merge kernel reads each task's foreign range
    straight from the holder rank's shard through CUDA IPC (no exchange
    step).  Functional check with `world` processes sharing cuda:0 (gloo for
    the small collectives); on a node every rank has its own GPU and the
    reads go over NVLink."""
    lib()
    import torch.multiprocessing as mp
    cases = [(300001, 200003, "i32", "full"), (100000, 7, "u64", "mostly:0x8000000000000000:9/10"),
             (5, 90001, "f32", "special")]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    mp.spawn(_peer_worker, args=(world, _port(), cases, out), nprocs=world, join=True)
    res = [out.get(timeout=5) for _ in cases]
    assert all(ok for _, ok in res), res


def _peer_sort_worker(rank, world, port, cases, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1202_6575_b200 import distributed as D
        for case in cases:
            N, kt, dist_name = case
            inp = synth.sort_input(N, kt, dist_name, seed=N + world, payload=True)
            xs = D.block_starts(N, world)
            k = inp.keys[xs[rank]:xs[rank + 1]].cuda()
            v = inp.vals[xs[rank]:xs[rank + 1]].cuda()
            sk, sv = D.mergesort_stable_sharded(k, v, N, key_type=kt, peer_access=True)
            got = [None] * world
            dist.all_gather_object(got, (sk.cpu(), sv.cpu()))
            if rank == 0:
                keys = torch.cat([g[0] for g in got])
                vals = torch.cat([g[1] for g in got])
                wk, wv = oracle.sort(inp.keys, inp.vals, kt)
                ok = all(got[q][0].shape[0] == xs[q + 1] - xs[q] for q in range(world))
                ok = ok and np.array_equal(oracle.as_np(keys, kt).view(np.uint8), wk.view(np.uint8)) and \
                    np.array_equal(oracle.vals_np(vals), wv)
                out.put((case, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_sort_peer_access_ipc(world):
    """peer_access=True for the sharded sort: foreign task inputs read in
    place and merged pieces copied straight into the destination ranks'
    next blocks through CUDA IPC (processes sharing cuda:0, gloo for the
    small collectives)."""
    lib()
    import torch.multiprocessing as mp
    cases = [(300001, "u32", "bounded:1048576"), (100003, "i64", "bounded:50"), (77777, "f32", "special")]
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    mp.spawn(_peer_sort_worker, args=(world, _port(), cases, out), nprocs=world, join=True)
    res = [out.get(timeout=5) for _ in cases]
    assert all(ok for _, ok in res), res
