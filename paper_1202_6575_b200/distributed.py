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
    """The local primitives on this rank's GPU (the library's kernels)."""

    def __init__(self, key_type: Optional[str] = None, descending: bool = False):
        from . import last_launch_count, merge_stable, mergesort_stable, ranks_stable
        self._merge, self._ranks, self._sort = merge_stable, ranks_stable, mergesort_stable
        self._count = last_launch_count
        self.key_type, self.descending = key_type, descending
        self.launches = 0                          # the library's kernel launches through this object

    def ranks(self, X: torch.Tensor, keys: torch.Tensor, high: bool) -> torch.Tensor:
        if X.numel() == 0 or keys.numel() == 0:
            return torch.zeros(keys.numel(), dtype=torch.int64, device=keys.device)
        r = self._ranks(X, keys, high, key_type=self.key_type, descending=self.descending)
        self.launches += self._count()
        return r

    def merge(self, ak, av, bk, bv):
        r = self._merge(ak, av, bk, bv, key_type=self.key_type, descending=self.descending)
        self.launches += self._count()
        return r

    def sort(self, keys, vals):
        keys = keys.clone()
        vals = None if vals is None else vals.clone()
        r = self._sort(keys, vals, key_type=self.key_type, descending=self.descending)
        self.launches += self._count()
        return r


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


def plan_tasks(n: int, m: int, p: int, xbar: Sequence[int], ybar: Sequence[int], pB: Optional[int] = None):
    """Steps 3-4 (L310-340; readings R1, R8): the p_A + p_B tasks as
    (owner, a0, a1, b0, b1), A-side task q then B-side task q for every q
    (p_A = p, p_B = pB or p: reading R7) -- the library's classification
    (sm_plan_tasks, the same code as the device's K2), on the host."""
    from . import plan_tasks as _plan
    pA, pB = p, (p if pB is None else pB)
    rows = _plan(n, m, pA, pB, xbar, ybar)
    return [(i,) + rows[i] for i in range(pA)] + [(j,) + rows[pA + j] for j in range(pB)]


def _holder(lo: int, hi: int, length: int, p: int) -> int:
    """The rank holding the non-empty range [lo, hi) (one block, L343-361)."""
    return block_of(lo, length, p) if hi > lo else -1


def _coll_device(t: torch.Tensor, group) -> torch.device:
    """Where the small collectives run: the tensors' device, or the host for
    a gloo group (CPU tests; several ranks sharing one GPU)."""
    return torch.device("cpu") if dist.get_backend(group) == "gloo" else t.device


def _share(t: Optional[torch.Tensor]):
    """A picklable CUDA IPC handle of t (torch's own IPC reduction)."""
    if t is None:
        return None
    from torch.multiprocessing.reductions import reduce_tensor
    return reduce_tensor(t.contiguous())


def _open(shared) -> Optional[torch.Tensor]:
    if shared is None:
        return None
    fn, args = shared
    return fn(*args)


def merge_stable_sharded(a_keys: torch.Tensor, a_vals: Optional[torch.Tensor], b_keys: torch.Tensor,
                         b_vals: Optional[torch.Tensor], n: int, m: int, *, group=None,
                         key_type: Optional[str] = None, ops=None,
                         peer_access: bool = False, stats: Optional[dict] = None) -> List[Piece]:
    """Stable merge (ties: A first) of A (n) and B (m) sharded over the ranks
    of `group`: this rank passes its blocks A[x_r, x_{r+1}) and B[y_r, y_{r+1})
    (PAPER.md block partition, p = world size).  Returns this rank's output
    pieces.  `stats` (optional dict) receives this rank's exchange volume:
    recv_bytes (foreign input ranges this rank's tasks read) and
    local_bytes (its own shards).

    peer_access (opt-in; CUDA shards in an NCCL group, all ranks' GPUs
    peer-accessible): no exchange step at all -- every rank maps the other
    ranks' shards (CUDA IPC handles, one all-gather) and the merge kernel's
    TMA loads read each task's foreign range straight from the holder's
    memory over NVLink, so the transfer overlaps the merge stage by stage
    inside ONE kernel; a barrier before the merges (inputs complete) and
    after them (no rank frees its shard while peers read it).  A mapped
    shard that does not land on this rank's device (torch opens an IPC
    handle on the sender's device index) makes the call fall back to the
    NCCL exchange: the library launches on the inputs' device only.  The
    NVLink path has been exercised with processes sharing one GPU only."""
    p = dist.get_world_size(group)
    r = dist.get_rank(group)
    ops = ops or CudaOps(key_type)
    custom_ops = not isinstance(ops, CudaOps)
    x, y = block_starts(n, p), block_starts(m, p)
    if a_keys.numel() != x[r + 1] - x[r] or b_keys.numel() != y[r + 1] - y[r]:
        raise ValueError("shards must be the paper's blocks: A[x_r, x_r+1) and B[y_r, y_r+1)")
    if (a_vals is None) != (b_vals is None):
        raise ValueError("payloads must be given for both inputs or neither")
    dev = a_keys.device
    cdev = _coll_device(a_keys, group)
    # block-start keys of every rank: one all-gather of (A[x_r], B[y_r])
    mine = torch.zeros(2, dtype=a_keys.dtype, device=dev)
    if a_keys.numel():
        mine[0] = a_keys[0]
    if b_keys.numel():
        mine[1] = b_keys[0]
    starts = torch.empty(2 * p, dtype=a_keys.dtype, device=cdev)
    dist.all_gather_into_tensor(starts, mine.to(cdev), group=group)
    starts = starts.to(dev)
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
    part = part.to(cdev)
    dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)  # the single synchronisation (L373-375)
    ranks = part.cpu().tolist()
    xbar = ranks[:p] + [m]
    ybar = ranks[p:] + [n]
    tasks = plan_tasks(n, m, p, xbar, ybar)

    if stats is not None:
        eb = a_keys.element_size() + (0 if a_vals is None else a_vals.element_size())
        fb = b_keys.element_size() + (0 if b_vals is None else b_vals.element_size())
        recv = 0
        for (owner, a0, a1, b0, b1) in tasks:
            if owner != r:
                continue
            if a1 > a0 and _holder(a0, a1, n, p) != r:
                recv += (a1 - a0) * eb
            if b1 > b0 and _holder(b0, b1, m, p) != r:
                recv += (b1 - b0) * fb
        stats.update(recv_bytes=recv, local_bytes=a_keys.numel() * eb + b_keys.numel() * fb, tasks=len(tasks))
    peer_access = bool(peer_access) and a_keys.is_cuda and b_keys.is_cuda and not custom_ops
    if peer_access and p > 1:
        pieces = _merge_tasks_peer(tasks, r, p, n, m, x, y, a_keys, a_vals, b_keys, b_vals, ops, group)
        if pieces is not None:
            return pieces

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


def _merge_tasks_peer(tasks, r, p, n, m, x, y, a_keys, a_vals, b_keys, b_vals, ops, group) -> List[Piece]:
    """The merges of merge_stable_sharded(peer_access=True): foreign ranges
    are read in place from the peers' shards (CUDA IPC mappings)."""
    torch.cuda.synchronize(a_keys.device)               # this rank's shards are complete ...
    handles = [None] * p
    dist.all_gather_object(handles, [_share(a_keys), _share(a_vals), _share(b_keys), _share(b_vals)], group=group)
    mapped = {}                                          # ... and every rank's, after the all-gather

    def shard(q):
        if q == r:
            return a_keys, a_vals, b_keys, b_vals
        if q not in mapped:
            mapped[q] = [_open(h) for h in handles[q]]
        return mapped[q]

    # every rank must be able to read every peer shard on its own device
    ok = all(t is None or t.device == a_keys.device for q in range(p) for t in shard(q))
    flags = torch.tensor([1 if ok else 0], dtype=torch.int32, device=_coll_device(a_keys, group))
    dist.all_reduce(flags, op=dist.ReduceOp.MIN, group=group)
    if not int(flags.item()):
        mapped.clear()
        dist.barrier(group=group)
        return None                                      # the caller takes the NCCL exchange

    pieces = []
    for k, (owner, a0, a1, b0, b1) in enumerate(tasks):
        if owner != r or a1 - a0 + b1 - b0 == 0:
            continue
        ha, hb = _holder(a0, a1, n, p), _holder(b0, b1, m, p)
        ak = a_keys[:0] if ha < 0 else shard(ha)[0][a0 - x[ha]:a1 - x[ha]]
        av = None if a_vals is None else (a_vals[:0] if ha < 0 else shard(ha)[1][a0 - x[ha]:a1 - x[ha]])
        bk = b_keys[:0] if hb < 0 else shard(hb)[2][b0 - y[hb]:b1 - y[hb]]
        bv = None if b_vals is None else (b_vals[:0] if hb < 0 else shard(hb)[3][b0 - y[hb]:b1 - y[hb]])
        ck, cv = ops.merge(ak, av, bk, bv)           # the kernel reads peer memory directly
        pieces.append(Piece(a0 + b0, ck, cv))
    torch.cuda.synchronize(a_keys.device)               # done reading the peers' shards
    mapped.clear()                                      # release the IPC mappings before the owners may free
    dist.barrier(group=group)
    return pieces


# ------------------------------------------------------------ sharded sort
# SURVEY.md §8(f) row 3 (merge SORT over the GPUs), the paper's merge sort
# (§3) with the ranks as processing elements:
#   phase 1  each rank sorts its block of the input (the library's sort:
#            "sorting sequentially in parallel p consecutive blocks", L406-407)
#   phase 2  ceil(log2 p) rounds; round i merges run pairs (2k, 2k+1), a run
#            being the sorted union of 2^i consecutive ranks' blocks, held
#            block-partitioned over those ranks (rank j of the run holds its
#            block j, PAPER.md L168-182 with p = the run's rank count).  One
#            pair is one sharded merge with p_A, p_B = the two runs' rank
#            counts (reading R7): one all-gather of block-start keys, local
#            ranks summed by ONE all-reduce (the single synchronisation,
#            L373-375), the p_A + p_B task plan (Steps 3-4), one round of
#            point-to-point sends of each task's foreign range (one block,
#            L343-361), local merges, and one round of sends that re-blocks
#            the merged run over its ranks.  All pairs of a round share the
#            same collectives; an odd trailing run waits (L409-410).
# Result: rank r holds block r of the stably sorted whole (equal keys keep
# their global input order: left runs play A).

def _reblock_peer(plans, pieces, mypair, keys, vals, r, p, group):
    """Sort round, peer access: every rank allocates its next-round block and
    shares it (CUDA IPC); task owners copy their merged pieces' segments
    straight into the destination blocks; a barrier ends the round."""
    dev = keys.device
    nk, nv = keys[:0], (None if vals is None else vals[:0])
    if mypair is not None:
        a0, b0, b1, n, m, x, y, owned = mypair
        z = block_starts(n + m, b1 - a0)
        L = z[r - a0 + 1] - z[r - a0]
        nk = torch.empty((L,) + tuple(keys.shape[1:]), dtype=keys.dtype, device=dev)
        nv = None if vals is None else torch.empty(L, dtype=vals.dtype, device=dev)
    else:
        nk, nv = keys, vals                           # odd trailing run: the block stays
    torch.cuda.synchronize(dev)                       # this rank's merged pieces are complete
    handles = [None] * p
    dist.all_gather_object(handles, [_share(nk), _share(nv)] if mypair is not None else None, group=group)
    for (a0, b0, b1, n, m, x, y, owned) in plans:
        z = block_starts(n + m, b1 - a0)
        for k, (owner, (ta0, ta1, tb0, tb1)) in enumerate(owned):
            if owner != r:
                continue
            off, L = ta0 + tb0, ta1 - ta0 + tb1 - tb0
            if L == 0:
                continue
            ck, cv = next((pk, pv) for (po, pk, pv) in pieces if po == off)
            for blk in range(b1 - a0):
                lo, hi = max(off, z[blk]), min(off + L, z[blk + 1])
                if hi <= lo:
                    continue
                dest = a0 + blk
                dk, dv = (nk, nv) if dest == r else [_open(h) for h in handles[dest]]
                dk[lo - z[blk]:hi - z[blk]].copy_(ck[lo - off:hi - off])       # peer-to-peer over NVLink
                if cv is not None:
                    dv[lo - z[blk]:hi - z[blk]].copy_(cv[lo - off:hi - off])
    torch.cuda.synchronize(dev)                       # every copy into the peers' blocks done
    dist.barrier(group=group)
    return nk, nv


def _cat(parts, like):
    parts = [t for t in parts if t is not None and t.shape[0] > 0]
    if not parts:
        return like[:0]
    return torch.cat(parts) if len(parts) > 1 else parts[0]


def mergesort_stable_sharded(keys: torch.Tensor, vals: Optional[torch.Tensor], N: int, *, group=None,
                             key_type: Optional[str] = None, descending: bool = False, ops=None,
                             peer_access: bool = False):
    """Stable sort of an array of N keys (+ uint32 payloads) sharded over the
    ranks of `group`: this rank passes block r of the input (PAPER.md block
    partition, p = world size) and gets back block r of the sorted array.
    Returns (keys, vals).

    peer_access (opt-in, CUDA shards): both exchange steps of a round go
    through CUDA IPC mappings instead of NCCL sends -- the merges read their
    foreign ranges in place from the holders' blocks, and each task owner
    copies its merged piece straight into the destination ranks' next-round
    blocks (peer-to-peer copies over NVLink).  If a mapped block does not
    land on this rank's device, the sort continues with the NCCL exchange."""
    p = dist.get_world_size(group)
    r = dist.get_rank(group)
    peer_access = bool(peer_access) and keys.is_cuda and ops is None and p > 1   # one rank: nothing to exchange
    ops = ops or CudaOps(key_type, descending)
    xs = block_starts(N, p)
    if keys.shape[0] != xs[r + 1] - xs[r]:
        raise ValueError("the shard must be the paper's block r of the input: [x_r, x_r+1)")
    if vals is not None and vals.shape[0] != keys.shape[0]:
        raise ValueError("vals must have one entry per key")
    dev = keys.device
    sizes = [xs[q + 1] - xs[q] for q in range(p)]      # run length = sum of its ranks' input blocks
    if keys.shape[0] > 1:
        keys, vals = ops.sort(keys, vals)                # phase 1
    h = 1
    while h < p:                                         # phase 2: round with runs of h ranks
        # block-start key of every rank's current block (one all-gather)
        mine = torch.zeros((1,) + tuple(keys.shape[1:]), dtype=keys.dtype, device=dev)
        if keys.shape[0]:
            mine[0] = keys[0]
        cdev = _coll_device(keys, group)
        starts = torch.empty((p,) + tuple(keys.shape[1:]), dtype=keys.dtype, device=cdev)
        dist.all_gather_into_tensor(starts, mine.to(cdev), group=group)
        starts = starts.to(dev)
        part = torch.zeros(2 * p, dtype=torch.int64, device=dev)
        pairs = []
        for a0 in range(0, p, 2 * h):
            b0, b1 = a0 + h, min(a0 + 2 * h, p)
            if b0 >= p:
                continue                                 # odd trailing run: unchanged this round
            pA, pB = h, b1 - b0
            n, m = sum(sizes[a0:b0]), sum(sizes[b0:b1])
            pairs.append((a0, b0, b1, n, m))
            x, y = block_starts(n, pA), block_starts(m, pB)
            if b0 <= r < b1:                             # B rank: rank_low(A[x_q], my B block)
                loc = ops.ranks(keys, starts[a0:b0].contiguous(), False)
                loc = torch.where(torch.tensor([x[q] >= n for q in range(pA)], device=dev),
                                  torch.full_like(loc, keys.shape[0]), loc)    # empty block start: m (R4)
                part[a0:b0] = loc
            elif a0 <= r < b0:                           # A rank: rank_high(B[y_q], my A block)
                loc = ops.ranks(keys, starts[b0:b1].contiguous(), True)
                loc = torch.where(torch.tensor([y[q] >= m for q in range(pB)], device=dev),
                                  torch.full_like(loc, keys.shape[0]), loc)
                part[p + b0:p + b1] = loc
        part = part.to(cdev)
        dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)   # the single synchronisation
        ranks = part.cpu().tolist()
        ops_list, recv, mypair = [], {}, None
        plans = []
        if peer_access:                                  # map every rank's current block (CUDA IPC)
            torch.cuda.synchronize(dev)
            handles = [None] * p
            dist.all_gather_object(handles, [_share(keys), _share(vals)], group=group)
            peers = {q: [_open(h) for h in handles[q]] for q in range(p) if q != r}
            peers[r] = [keys, vals]
            ok = all(t is None or t.device == dev for q in range(p) for t in peers[q])
            flags = torch.tensor([1 if ok else 0], dtype=torch.int32, device=_coll_device(keys, group))
            dist.all_reduce(flags, op=dist.ReduceOp.MIN, group=group)
            if not int(flags.item()):                    # mapped on another device: NCCL from here on
                peers = None
                peer_access = False
                dist.barrier(group=group)
        for (a0, b0, b1, n, m) in pairs:
            pA, pB = b0 - a0, b1 - b0
            xbar = ranks[a0:b0] + [m]
            ybar = ranks[p + b0:p + b1] + [n]
            tasks = plan_tasks(n, m, pA, xbar, ybar, pB)
            x, y = block_starts(n, pA), block_starts(m, pB)
            # owners: A-side task q on A rank a0+q, B-side task q on B rank b0+q
            owned = [(a0 + q if k < pA else b0 + (k - pA), t) for k, (q, *t) in enumerate(tasks)]
            plans.append((a0, b0, b1, n, m, x, y, owned))
            if a0 <= r < b1:
                mypair = plans[-1]
            for k, (owner, (ta0, ta1, tb0, tb1)) in enumerate(owned):
                for side, lo, hi, length, st, base in (("A", ta0, ta1, n, x, a0), ("B", tb0, tb1, m, y, b0)):
                    if hi <= lo:
                        continue
                    holder = base + block_of(lo, length, len(st) - 1)
                    if holder == owner:
                        continue
                    if peer_access:                      # read in place from the holder's block
                        if owner == r:
                            s0, s1 = lo - st[holder - base], hi - st[holder - base]
                            pk, pv = peers[holder]
                            recv[(a0, k, side)] = (pk[s0:s1], None if pv is None else pv[s0:s1])
                        continue
                    if owner == r:
                        kt_ = torch.empty((hi - lo,) + tuple(keys.shape[1:]), dtype=keys.dtype, device=dev)
                        ops_list.append(dist.P2POp(dist.irecv, kt_, holder, group=group))
                        vt_ = None
                        if vals is not None:
                            vt_ = torch.empty(hi - lo, dtype=vals.dtype, device=dev)
                            ops_list.append(dist.P2POp(dist.irecv, vt_, holder, group=group))
                        recv[(a0, k, side)] = (kt_, vt_)
                    elif holder == r:
                        s0, s1 = lo - st[r - base], hi - st[r - base]
                        ops_list.append(dist.P2POp(dist.isend, keys[s0:s1].contiguous(), owner, group=group))
                        if vals is not None:
                            ops_list.append(dist.P2POp(dist.isend, vals[s0:s1].contiguous(), owner, group=group))
        if ops_list:
            for w in dist.batch_isend_irecv(ops_list):
                w.wait()
        # local merges of this rank's tasks -> pieces (offset in the merged run)
        pieces = []
        if mypair is not None:
            a0, b0, b1, n, m, x, y, owned = mypair
            for k, (owner, (ta0, ta1, tb0, tb1)) in enumerate(owned):
                if owner != r or ta1 - ta0 + tb1 - tb0 == 0:
                    continue

                def local(side, lo, hi, st, base):
                    if (a0, k, side) in recv:
                        return recv[(a0, k, side)]
                    if hi <= lo:
                        return keys[:0], (None if vals is None else vals[:0])
                    s0, s1 = lo - st[r - base], hi - st[r - base]
                    return keys[s0:s1], (None if vals is None else vals[s0:s1])

                ak, av = local("A", ta0, ta1, x, a0)
                bk, bv = local("B", tb0, tb1, y, b0)
                ck, cv = ops.merge(ak.contiguous(), None if av is None else av.contiguous(), bk.contiguous(),
                                   None if bv is None else bv.contiguous())
                pieces.append((ta0 + tb0, ck, cv))
        if peer_access:
            recv.clear()
            peers.clear()                                # inputs read: release the mappings
            keys, vals = _reblock_peer(plans, pieces, mypair, keys, vals, r, p, group)
            h *= 2
            continue
        # re-block every merged run over its ranks (one round of sends)
        ops_list, incoming = [], []
        for (a0, b0, b1, n, m, x, y, owned) in plans:
            z = block_starts(n + m, b1 - a0)
            for k, (owner, (ta0, ta1, tb0, tb1)) in enumerate(owned):
                off, L = ta0 + tb0, ta1 - ta0 + tb1 - tb0
                for blk in range(b1 - a0):
                    lo, hi = max(off, z[blk]), min(off + L, z[blk + 1])
                    if hi <= lo:
                        continue
                    dest = a0 + blk
                    if owner == r:
                        ck, cv = next((pk, pv) for (po, pk, pv) in pieces if po == off)
                        seg_k, seg_v = ck[lo - off:hi - off], None if cv is None else cv[lo - off:hi - off]
                        if dest == r:
                            incoming.append((lo, seg_k, seg_v))
                        else:
                            ops_list.append(dist.P2POp(dist.isend, seg_k.contiguous(), dest, group=group))
                            if vals is not None:
                                ops_list.append(dist.P2POp(dist.isend, seg_v.contiguous(), dest, group=group))
                    elif dest == r:
                        kt_ = torch.empty((hi - lo,) + tuple(keys.shape[1:]), dtype=keys.dtype, device=dev)
                        ops_list.append(dist.P2POp(dist.irecv, kt_, owner, group=group))
                        vt_ = None
                        if vals is not None:
                            vt_ = torch.empty(hi - lo, dtype=vals.dtype, device=dev)
                            ops_list.append(dist.P2POp(dist.irecv, vt_, owner, group=group))
                        incoming.append((lo, kt_, vt_))
        if ops_list:
            for w in dist.batch_isend_irecv(ops_list):
                w.wait()
        if mypair is not None:
            incoming.sort(key=lambda t: t[0])
            keys = _cat([t[1] for t in incoming], keys)
            vals = None if vals is None else _cat([t[2] for t in incoming], vals)
        # the merged runs' ranks now hold blocks of runs of 2h ranks
        h *= 2
    return keys, vals
