"""Reading R20 checked on the CPU, independently of the CUDA
path: the paper's partition (Steps 1-2, the cross ranks of
the block starts) generalised from two sorted arrays to four.

A small numpy model written from the reading alone: every block start
e = R_j[qS] is ranked in each other run j' -- rank_high (elements <= e) when
j' < j, rank_low (elements < e) when j' > j (L304-309 with the tie rule of
reading R2: the earlier run first) -- its place in the merged group is
f(e) = qS + the three ranks, and consecutive block starts in f order delimit
the subproblems.  Checked against brute force: the f values are the block
starts' true positions in the stable four-way merge, every subproblem takes
one contiguous range of at most S elements from every run (the task bound of
L388-393 for four arrays), the subproblems are disjoint and cover the group,
their output offset is the sum of their lower boundaries, and merging each
one stably (key, then run, then position) and concatenating gives the stable
merge of the four runs -- which is what two rounds of the paper's two-way
merges (R0 with R1, R2 with R3, then the results) produce."""
import numpy as np
import pytest


def stable_merge4(runs):
    """Brute force: all elements sorted by (key, run index, position)."""
    keys = np.concatenate(runs)
    run = np.concatenate([np.full(len(r), j) for j, r in enumerate(runs)])
    pos = np.concatenate([np.arange(len(r)) for r in runs])
    order = np.lexsort((pos, run, keys))
    return keys[order], run[order], pos[order]


def partition4(runs, S):
    """Boundaries (one rank per run) of the subproblems, in output order."""
    bnd = []
    for j, r in enumerate(runs):
        for q in range(0, len(r), S):
            e = r[q]
            rk = []
            for jj, o in enumerate(runs):
                if jj == j:
                    rk.append(q)
                else:
                    rk.append(int(np.searchsorted(o, e, side="right" if jj < j else "left")))
            bnd.append((sum(rk), tuple(rk)))
    bnd.sort()
    fs = [f for f, _ in bnd]
    return fs, [(0, 0, 0, 0)] + [b for _, b in bnd] + [tuple(len(r) for r in runs)]


CASES = [((50, 50, 50, 50), 7, 1000), ((64, 64, 64, 17), 16, 3), ((100, 0, 37, 5), 8, 2), ((33, 33, 0, 0), 5, 10),
         ((1, 1, 1, 1), 4, 1), ((200, 150, 100, 50), 32, 50), ((40, 40, 40, 40), 64, 5), ((97, 89, 83, 79), 1, 4)]


@pytest.mark.parametrize("lens,S,span", CASES)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_four_run_partition(lens, S, span, seed):
    rng = np.random.default_rng(seed * 1000 + S)
    runs = [np.sort(rng.integers(0, span, size=n)) for n in lens]
    mk, mrun, mpos = stable_merge4(runs)
    fs, bnd = partition4(runs, S)
    # f(e) is the block start's position in the stable merge: distinct, and exact
    assert len(set(fs)) == len(fs)
    where = {(int(j), int(p)): i for i, (j, p) in enumerate(zip(mrun, mpos))}
    k = 0
    for j, r in enumerate(runs):
        for q in range(0, len(r), S):
            k += 1
    got = sorted(where[(j, q)] for j, r in enumerate(runs) for q in range(0, len(r), S))
    assert got == fs and len(fs) == k
    # subproblems: contiguous, <= S per run, disjoint cover, offsets, and their merges
    out = []
    for lo, hi in zip(bnd[:-1], bnd[1:]):
        parts = []
        for j in range(4):
            assert 0 <= hi[j] - lo[j] <= S, (lo, hi, S)
            parts.append(runs[j][lo[j]:hi[j]])
        assert len(out) == sum(lo)                       # output offset = the sum of the lower boundaries
        sk, _, _ = stable_merge4(parts)
        out.extend(sk.tolist())
    assert out == mk.tolist()
    # the two rounds of two-way merges give the same sequence (ties: the earlier run first)
    def merge2(a, b):
        keys = np.concatenate([a, b])
        side = np.concatenate([np.zeros(len(a), int), np.ones(len(b), int)])
        pos = np.concatenate([np.arange(len(a)), np.arange(len(b))])
        return keys[np.lexsort((pos, side, keys))]
    assert merge2(merge2(runs[0], runs[1]), merge2(runs[2], runs[3])).tolist() == mk.tolist()


def test_four_run_partition_all_equal():
    """All keys equal: every rank is decided by the tie rule alone."""
    runs = [np.zeros(n, int) for n in (20, 20, 20, 9)]
    fs, bnd = partition4(runs, 6)
    assert fs == sorted(set(fs))
    for lo, hi in zip(bnd[:-1], bnd[1:]):
        assert all(0 <= h - l <= 6 for l, h in zip(lo, hi))
    assert bnd[-1] == (20, 20, 20, 9)
