"""O3 -- the paper's Steps 1-4 on the CPU, in the paper's order and notation.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Shares nothing with the
CUDA path.  Plain Python over lists or numpy arrays; slow by design.

Citations are PAPER.md line numbers (§2):
  block_starts   x_i = i*ceil(n/p) for i < r = n mod p, else i*floor(n/p) + r;
                 x_p = n                                          L168-182, L293
  block_of       index k belongs to block i if k < r*ceil(n/p) and
                 floor(k/ceil(n/p)) = i, or k >= r*ceil(n/p) and
                 floor((k - r*ceil(n/p))/floor(n/p)) + r = i      L294-300
                 reading R3/R5: block_of(len) = p (virtual block)
  rank_low       unique i with X[i-1] < x <= X[i]                 L119-123
  rank_high      unique j with X[j-1] <= x < X[j]                 L124-128
  Step 1         xbar_i = rank_low(A[x_i], B), xbar_p = m         L304-306
  Step 2         ybar_j = rank_high(B[y_j], A), ybar_p = n        L307-309
                 reading R4: an empty block's start (x_i = n) has xbar_i = m
  Step 3 (a)-(e) A-side classification                            L310-336
                 reading R1: case (d) A range ends at x_{i+1} (text: x_{j+1})
  Step 4         B-side "in the same fashion"                     L337-340
                 reading R2: ties inside B-side merges still go to A
  Output offset  C[x_i + xbar_i, ...] (A side), C[y_j + ybar_j, ...] (B side)

Reading R7: A and B may use different block counts p_A and
p_B; A-side tasks run over A's p_A blocks, B-side over B's p_B blocks.  The
paper's single p is the case p_A = p_B.
"""
from __future__ import annotations

from typing import List, NamedTuple, Sequence

import numpy as np


class Task(NamedTuple):
    side: str      # "A" (Step 3, PE at x_i) or "B" (Step 4, PE at y_j)
    case: str      # "a".."e"
    a0: int        # A range [a0, a1)
    a1: int
    b0: int        # B range [b0, b1)
    b1: int

    @property
    def off(self) -> int:
        """Output offset: x_i + xbar_i (A side) or y_j + ybar_j (B side)."""
        return self.a0 + self.b0

    @property
    def size(self) -> int:
        return (self.a1 - self.a0) + (self.b1 - self.b0)


def _ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def block_starts(length: int, p: int) -> List[int]:
    """x_0..x_p (L168-182; x_p = n at L293)."""
    if p < 1:
        raise ValueError("p must be >= 1")
    r = length % p
    ceil, floor = _ceil_div(length, p), length // p
    return [i * ceil if i < r else i * floor + r for i in range(p)] + [length]


def block_of(k: int, length: int, p: int) -> int:
    """Block containing index k (L294-300); k = length -> p (reading R3)."""
    if not 0 <= k <= length:
        raise ValueError("index out of range")
    if k == length:
        return p
    r = length % p
    ceil, floor = _ceil_div(length, p), length // p
    if k < r * ceil:
        return k // ceil
    return (k - r * ceil) // floor + r


def rank_low(x, X: Sequence) -> int:
    """Unique i with X[i-1] < x <= X[i], sentinels X[-1]=-inf, X[len]=+inf."""
    lo, hi = 0, len(X)
    while lo < hi:                  # invariant: X[lo-1] < x, x <= X[hi]
        mid = (lo + hi) // 2
        if X[mid] < x:
            lo = mid + 1
        else:
            hi = mid
    return lo


def rank_high(x, X: Sequence) -> int:
    """Unique j with X[j-1] <= x < X[j], same sentinels."""
    lo, hi = 0, len(X)
    while lo < hi:                  # invariant: X[lo-1] <= x, x < X[hi]
        mid = (lo + hi) // 2
        if X[mid] <= x:
            lo = mid + 1
        else:
            hi = mid
    return lo


def cross_ranks(A: Sequence, B: Sequence, pA: int, pB: int, vectorised: bool = False):
    """Steps 1 and 2: xbar[0..pA], ybar[0..pB].

    `vectorised=True` computes the same ranks with numpy.searchsorted
    (side='left' is rank_low, side='right' is rank_high) for large inputs;
    tests pin it against the plain binary search above."""
    n, m = len(A), len(B)
    x, y = block_starts(n, pA), block_starts(m, pB)
    if vectorised:
        A, B = np.asarray(A), np.asarray(B)
        xs = np.asarray(x[:-1], dtype=np.int64)
        ys = np.asarray(y[:-1], dtype=np.int64)
        xbar = np.full(pA + 1, m, dtype=np.int64)
        ybar = np.full(pB + 1, n, dtype=np.int64)
        ok = xs < n
        xbar[:-1][ok] = np.searchsorted(B, A[xs[ok]], side="left")
        ok = ys < m
        ybar[:-1][ok] = np.searchsorted(A, B[ys[ok]], side="right")
        return x, y, [int(v) for v in xbar], [int(v) for v in ybar]
    xbar = [rank_low(A[x[i]], B) if x[i] < n else m for i in range(pA)] + [m]
    ybar = [rank_high(B[y[j]], A) if y[j] < m else n for j in range(pB)] + [n]
    return x, y, xbar, ybar


def classify_a(i: int, x, y, xbar, ybar, n: int, m: int, pB: int) -> Task:
    """Step 3, the PE assigned to x_i (L310-336), cases tested (a),(e),(b),(d),(c)."""
    if xbar[i] == xbar[i + 1]:                                   # (a) L315-317
        return Task("A", "a", x[i], x[i + 1], xbar[i], xbar[i])
    j = block_of(xbar[i], m, pB)
    if xbar[i] == y[j]:                                          # (e) L332-335
        return Task("A", "e", x[i], ybar[j], xbar[i], xbar[i])
    if block_of(xbar[i + 1], m, pB) == j:                        # (b) L318-321
        return Task("A", "b", x[i], x[i + 1], xbar[i], xbar[i + 1])
    if xbar[i + 1] == y[j + 1]:                                  # (d) L327-331, R1
        return Task("A", "d", x[i], x[i + 1], xbar[i], y[j + 1])
    return Task("A", "c", x[i], ybar[j + 1], xbar[i], y[j + 1])  # (c) L322-326


def classify_b(j: int, x, y, xbar, ybar, n: int, m: int, pA: int) -> Task:
    """Step 4, the PE assigned to y_j: Step 3 with the roles of A and B swapped."""
    if ybar[j] == ybar[j + 1]:                                   # (a)
        return Task("B", "a", ybar[j], ybar[j], y[j], y[j + 1])
    i = block_of(ybar[j], n, pA)
    if ybar[j] == x[i]:                                          # (e)
        return Task("B", "e", ybar[j], ybar[j], y[j], xbar[i])
    if block_of(ybar[j + 1], n, pA) == i:                        # (b)
        return Task("B", "b", ybar[j], ybar[j + 1], y[j], y[j + 1])
    if ybar[j + 1] == x[i + 1]:                                  # (d)
        return Task("B", "d", ybar[j], x[i + 1], y[j], y[j + 1])
    return Task("B", "c", ybar[j], x[i + 1], y[j], xbar[i + 1])  # (c)


def build_plan(A: Sequence, B: Sequence, pA: int, pB: int = None, vectorised: bool = False):
    """Steps 1-4.  Returns (x, y, xbar, ybar, tasks) with tasks = the pA A-side
    tasks followed by the pB B-side tasks."""
    if pB is None:
        pB = pA
    n, m = len(A), len(B)
    x, y, xbar, ybar = cross_ranks(A, B, pA, pB, vectorised)
    tasks = [classify_a(i, x, y, xbar, ybar, n, m, pB) for i in range(pA)]
    tasks += [classify_b(j, x, y, xbar, ybar, n, m, pA) for j in range(pB)]
    return x, y, xbar, ybar, tasks


def stable_merge_afirst(a: Sequence, b: Sequence) -> list:
    """Sequential stable merge, ties to A (the subroutine of L354-357).
    Elements are compared by their first component when they are tuples."""
    key = (lambda e: e[0]) if (len(a) and isinstance(a[0], tuple)) or (len(b) and isinstance(b[0], tuple)) \
        else (lambda e: e)
    out, i, j = [], 0, 0
    while i < len(a) and j < len(b):
        if key(a[i]) <= key(b[j]):
            out.append(a[i]); i += 1
        else:
            out.append(b[j]); j += 1
    return out + list(a[i:]) + list(b[j:])


def execute_plan(tasks, A: Sequence, B: Sequence) -> list:
    """Run every task into its output interval (after the single sync)."""
    C = [None] * (len(A) + len(B))
    for t in tasks:
        C[t.off:t.off + t.size] = stable_merge_afirst(A[t.a0:t.a1], B[t.b0:t.b1])
    return C


def task_table(tasks) -> np.ndarray:
    """(len(tasks), 6) int64: side(0=A,1=B), case(0..4 for a..e), a0, a1, b0, b1."""
    t = np.zeros((len(tasks), 6), dtype=np.int64)
    for k, tk in enumerate(tasks):
        t[k] = (0 if tk.side == "A" else 1, "abcde".index(tk.case), tk.a0, tk.a1, tk.b0, tk.b1)
    return t
