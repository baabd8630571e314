"""Sharded stable merge over several GPUs.

The paper's own remark (§3): the method suits distributed
(BSP) machines because the merge of distinguished elements of earlier
algorithms is gone -- one exchange step remains.  Here the p processing
elements ARE the ranks (one GPU each, torch.distributed over NCCL):

  blocks     rank r holds block r of A and block r of B, blocks exactly as
             PAPER.md L168-182 with p = world size
             (x_r = r*ceil(n/p) for r < n mod p, else r*floor(n/p) + n mod p)
  Steps 1-2  every rank ranks all p A-block starts in its B shard (rank_low)
             and all p B-block starts in its A shard (rank_high) with the
             library's rank kernel; the cross rank of a block start is the
             sum of its ranks over the shards (the shards partition B / A in
             order), so ONE all-reduce of 2p integers gives every x̄_q, ȳ_q --
             the single synchronisation of L373-375 (plus one all-gather of
             the 2p block-start keys before it)
  Steps 3-4  every rank classifies all 2p tasks (cases (a)-(e), O(p) host
             work); rank q owns A-side task q and B-side task q
  exchange   each task's A range lies in one A block and its B range in one
             B block (the paper's containment argument, L343-361), so each
             task needs at most one foreign range, from one rank: one round
             of point-to-point sends (batch_isend_irecv)
  merge      each rank merges its two tasks with the library's device merge

The output is left where the tasks computed it: a list of (global offset,
keys, payloads) pieces per rank, the pieces of all ranks tiling [0, n+m).
Every computation step runs in the CUDA library (`ranks_stable`,
`merge_stable`); the collectives are NCCL.  `ops` exists only so that the
multi-process host logic can be tested on CPU (gloo) with another local
implementation of the two primitives.
"""
from __future__ import annotations

from typing import List, NamedTuple, Optional, Sequence

import torch
import torch.distributed as dist


class Piece(NamedTuple):
    offset: int                     # global output index of keys[0]
    keys: torch.Tensor
    vals: Optional[torch.Tensor]


class CudaOps:
    """The two local primitives on this rank's GPU (the library's kernels)."""

    def __init__(self, key_type: Optional[str] = None):
        from . import merge_stable, ranks_stable
        self._merge, self._ranks, self.key_type = merge_stable, ranks_stable, key_type

    def ranks(self, X: torch.Tensor, keys: torch.Tensor, high: bool) -> torch.Tensor:
        if X.numel() == 0 or keys.numel() == 0:
            return torch.zeros(keys.numel(), dtype=torch.int64, device=keys.device)
        return self._ranks(X, keys, high, key_type=self.key_type)

    def merge(self, ak, av, bk, bv):
        return self._merge(ak, av, bk, bv, key_type=self.key_type)


def block_starts(length: int, p: int) -> List[int]:
    """x_0..x_p (x_p = length at L293)."""
    q, r = divmod(length, p)
    return [i * (q + 1) if i < r else i * q + r for i in range(p)] + [length]


def block_of(k: int, length: int, p: int) -> int:
    """Block of index k (L294-300); block_of(length) = p (reading R3)."""
    if k >= length:
        return p
    q, r = divmod(length, p)
    big = r * (q + 1)
    return k // (q + 1) if k < big else (k - big) // q + r


def plan_tasks(n: int, m: int, p: int, xbar: Sequence[int], ybar: Sequence[int]):
    """Steps 3-4 (L310-340; readings R1, R8): the 2p tasks as
    (owner, a0, a1, b0, b1), A-side task q then B-side task q for every q."""
    x, y = block_starts(n, p), block_starts(m, p)
    tasks = []
    for i in range(p):
        if xbar[i] == xbar[i + 1]:
            t = (x[i], x[i + 1], xbar[i], xbar[i])
        else:
            j = block_of(xbar[i], m, p)
            if xbar[i] == y[j]:
                t = (x[i], ybar[j], xbar[i], xbar[i])
            elif block_of(xbar[i + 1], m, p) == j:
                t = (x[i], x[i + 1], xbar[i], xbar[i + 1])
            elif xbar[i + 1] == y[j + 1]:
                t = (x[i], x[i + 1], xbar[i], y[j + 1])
            else:
                t = (x[i], ybar[j + 1], xbar[i], y[j + 1])
        tasks.append((i,) + t)
    for j in range(p):
        if ybar[j] == ybar[j + 1]:
            t = (ybar[j], ybar[j], y[j], y[j + 1])
        else:
            i = block_of(ybar[j], n, p)
            if ybar[j] == x[i]:
                t = (ybar[j], ybar[j], y[j], xbar[i])
            elif block_of(ybar[j + 1], n, p) == i:
                t = (ybar[j], ybar[j + 1], y[j], y[j + 1])
            elif ybar[j + 1] == x[i + 1]:
                t = (ybar[j], x[i + 1], y[j], y[j + 1])
            else:
                t = (ybar[j], x[i + 1], y[j], xbar[i + 1])
        tasks.append((j,) + t)
    return tasks


def _holder(lo: int, hi: int, length: int, p: int) -> int:
    """The rank holding the non-empty range [lo, hi) (one block, L343-361)."""
    return block_of(lo, length, p) if hi > lo else -1


def merge_stable_sharded(a_keys: torch.Tensor, a_vals: Optional[torch.Tensor], b_keys: torch.Tensor,
                         b_vals: Optional[torch.Tensor], n: int, m: int, *, group=None,
                         key_type: Optional[str] = None, ops=None) -> List[Piece]:
    """Stable merge (ties: A first) of A (n) and B (m) sharded over the ranks
    of `group`: this rank passes its blocks A[x_r, x_{r+1}) and B[y_r, y_{r+1})
    (PAPER.md block partition, p = world size).  Returns this rank's output
    pieces."""
    p = dist.get_world_size(group)
    r = dist.get_rank(group)
    ops = ops or CudaOps(key_type)
    x, y = block_starts(n, p), block_starts(m, p)
    if a_keys.numel() != x[r + 1] - x[r] or b_keys.numel() != y[r + 1] - y[r]:
        raise ValueError("shards must be the paper's blocks: A[x_r, x_r+1) and B[y_r, y_r+1)")
    if (a_vals is None) != (b_vals is None):
        raise ValueError("payloads must be given for both inputs or neither")
    dev = a_keys.device
    # block-start keys of every rank: one all-gather of (A[x_r], B[y_r])
    mine = torch.zeros(2, dtype=a_keys.dtype, device=dev)
    if a_keys.numel():
        mine[0] = a_keys[0]
    if b_keys.numel():
        mine[1] = b_keys[0]
    starts = torch.empty(2 * p, dtype=a_keys.dtype, device=dev)
    dist.all_gather_into_tensor(starts, mine, group=group)
    sa, sb = starts[0::2].contiguous(), starts[1::2].contiguous()
    # Steps 1-2: ranks in the local shards; empty block starts rank as the
    # sentinel (their sum is the full length, reading R4)
    part = torch.empty(2 * p, dtype=torch.int64, device=dev)
    part[:p] = ops.ranks(b_keys, sa, False)                  # rank_low(A[x_q], B_r)
    part[p:] = ops.ranks(a_keys, sb, True)                   # rank_high(B[y_q], A_r)
    empty_a = torch.tensor([x[q] >= n for q in range(p)], device=dev)
    empty_b = torch.tensor([y[q] >= m for q in range(p)], device=dev)
    part[:p] = torch.where(empty_a, torch.full_like(part[:p], b_keys.numel()), part[:p])
    part[p:] = torch.where(empty_b, torch.full_like(part[p:], a_keys.numel()), part[p:])
    dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)  # the single synchronisation (L373-375)
    ranks = part.cpu().tolist()
    xbar = ranks[:p] + [m]
    ybar = ranks[p:] + [n]
    tasks = plan_tasks(n, m, p, xbar, ybar)

    # exchange: every task's foreign range from its single holder
    ops_list, recv = [], {}
    for k, (owner, a0, a1, b0, b1) in enumerate(tasks):
        for side, lo, hi, length, starts_, keys_, vals_ in (("A", a0, a1, n, x, a_keys, a_vals),
                                                             ("B", b0, b1, m, y, b_keys, b_vals)):
            h = _holder(lo, hi, length, p)
            if h < 0 or h == owner:
                continue
            if owner == r:                                   # receive [lo, hi) from rank h
                kt = torch.empty(hi - lo, dtype=a_keys.dtype, device=dev)
                ops_list.append(dist.P2POp(dist.irecv, kt, h, group=group))
                vt = None
                if vals_ is not None:
                    vt = torch.empty(hi - lo, dtype=a_vals.dtype, device=dev)
                    ops_list.append(dist.P2POp(dist.irecv, vt, h, group=group))
                recv[(k, side)] = (kt, vt)
            elif h == r:                                     # send my slice to the owner
                s0, s1 = lo - starts_[r], hi - starts_[r]
                ops_list.append(dist.P2POp(dist.isend, keys_[s0:s1].contiguous(), owner, group=group))
                if vals_ is not None:
                    ops_list.append(dist.P2POp(dist.isend, vals_[s0:s1].contiguous(), owner, group=group))
    if ops_list:
        for w in dist.batch_isend_irecv(ops_list):
            w.wait()

    # merge this rank's tasks on its GPU
    pieces = []
    for k, (owner, a0, a1, b0, b1) in enumerate(tasks):
        if owner != r or a1 - a0 + b1 - b0 == 0:
            continue

        def local(side, lo, hi, starts_, keys_, vals_):
            if (k, side) in recv:
                return recv[(k, side)]
            s0, s1 = lo - starts_[r], hi - starts_[r]
            return keys_[s0:s1], (None if vals_ is None else vals_[s0:s1])

        ak, av = local("A", a0, a1, x, a_keys, a_vals)
        bk, bv = local("B", b0, b1, y, b_keys, b_vals)
        ck, cv = ops.merge(ak.contiguous(), None if av is None else av.contiguous(), bk.contiguous(),
                           None if bv is None else bv.contiguous())
        pieces.append(Piece(a0 + b0, ck, cv))
    return pieces
