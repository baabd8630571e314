"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no ranks, no partition, no
merge): it only draws pseudo-random keys, sorts them with a library sort where
the workload says "each array sorted", and attaches the source-index payloads
that make stability observable.  Both `oracle/` (through the tests) and the
CUDA path (through the tests, `smoke()` and `bench.py`) take their inputs from
here, so the two sides see the same bits.

Generator: SplitMix64 used as a counter-based generator (DESIGN.md "Input
recipe"):

    s       = mix64((seed << 8) | stream)
    r_i     = mix64(s + (i + 1) * 0x9E3779B97F4A7C15)      (mod 2^64)
    K(r, k) = ((r >> 32) * k) >> 32                        (Lemire, 0 <= K < k)

All arithmetic is done in torch int64 with wrap-around (two's complement) and
explicit masks after right shifts, so it is device-agnostic: the same tensor
comes out on the CPU and on `cuda:0`.  Unsigned keys (u32/u64) are carried in
int32/int64 tensors with the same bit pattern.

Workloads follow BASELINE.json `configs` (C1..C5) with the readings R13/R14 of
SURVEY.md §8(c):
  C1  n=m=2^20  u32 key = K(r, 2^16), payload A: i, B: 0x80000000|j
  C2  n=m=2^26  i32 key = top 32 bits of r (full signed range), keys only
  C3  n=2^28 m=2^16  i64 key = K(r, 1000), payloads as C1
  C4  n=2^27 m=2^25  u64 key = 2^63 with probability 0.9 (K(r4,10) < 9) else r
  C5  N=2^28  u32 key = K(r, 2^20) unsorted, payload = original index
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import torch

BASE_SEED = 0x12026575
STREAM_A, STREAM_B, STREAM_SORT, STREAM_BERN = 1, 2, 3, 4

_GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK64 = (1 << 64) - 1


def _s64(u: int) -> int:
    """Unsigned 64-bit constant -> the int64 with the same bits."""
    u &= _MASK64
    return u - (1 << 64) if u >= (1 << 63) else u


def _lsr(x: torch.Tensor, k: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return (x >> k) & ((1 << (64 - k)) - 1)


def _mix64(z: torch.Tensor) -> torch.Tensor:
    z = (z ^ _lsr(z, 30)) * _s64(_M1)
    z = (z ^ _lsr(z, 27)) * _s64(_M2)
    return z ^ _lsr(z, 31)


def _mix64_int(z: int) -> int:
    z &= _MASK64
    z = ((z ^ (z >> 30)) * _M1) & _MASK64
    z = ((z ^ (z >> 27)) * _M2) & _MASK64
    return z ^ (z >> 31)


def splitmix_stream(seed: int, stream: int, count: int, device="cpu", start: int = 0) -> torch.Tensor:
    """r_i for i in [start, start+count) as int64 bit patterns (uint64 values)."""
    s = _mix64_int(((seed << 8) | stream) & _MASK64)
    i = torch.arange(start + 1, start + count + 1, dtype=torch.int64, device=device)
    return _mix64(i * _s64(_GOLDEN) + _s64(s))


def bounded(r: torch.Tensor, k: int) -> torch.Tensor:
    """Lemire multiply-shift: uniform-ish integer in [0, k), k <= 2^32."""
    assert 0 < k <= (1 << 32)
    return _lsr(_lsr(r, 32) * k, 32)


def _order_key(x: torch.Tensor, order: str) -> torch.Tensor:
    """An integer with the key order, for a library sort: identity for signed,
    sign bit flipped for unsigned, and for IEEE 754 totalOrder the magnitude
    bits of negative values inverted (an involution)."""
    if order == "s":
        return x
    if order == "u":
        return x ^ torch.iinfo(x.dtype).min
    return torch.where(x < 0, x ^ torch.iinfo(x.dtype).max, x)


def sort_bits(x: torch.Tensor, order: str) -> torch.Tensor:
    """Library sort of keys carried as int32/int64 bit patterns, ascending in
    the key type's order ("s" signed, "u" unsigned, "f" IEEE totalOrder)."""
    return _order_key(torch.sort(_order_key(x, order), stable=True).values, order)


KEY_TYPES = {
    # name: (torch carrier dtype, order: s signed / u unsigned / f IEEE totalOrder, key bytes)
    "u32": (torch.int32, "u", 4),
    "i32": (torch.int32, "s", 4),
    "i64": (torch.int64, "s", 8),
    "u64": (torch.int64, "u", 8),
    "f32": (torch.int32, "f", 4),
    "f64": (torch.int64, "f", 8),
    # unsigned 128-bit: int64 carrier of shape (N, 2) = (lo, hi) words
    "u128": (torch.int64, "u128", 16),
}

# float bit patterns of the "special" distribution: +-0, +-inf, +-NaN (quiet,
# with payloads), the smallest subnormals, +-1, +-max
_SPECIAL = {
    "f32": [0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00000, 0x7FC00001, 0x00000001,
            0x80000001, 0x3F800000, 0xBF800000, 0x7F7FFFFF, 0xFF7FFFFF],
    "f64": [0x0, 0x8000000000000000, 0x7FF0000000000000, 0xFFF0000000000000, 0x7FF8000000000000,
            0xFFF8000000000000, 0x7FF8000000000001, 0x1, 0x8000000000000001, 0x3FF0000000000000,
            0xBFF0000000000000, 0x7FEFFFFFFFFFFFFF, 0xFFEFFFFFFFFFFFFF],
}


@dataclasses.dataclass
class MergeInput:
    key_type: str
    a_keys: torch.Tensor
    b_keys: torch.Tensor
    a_vals: Optional[torch.Tensor]
    b_vals: Optional[torch.Tensor]

    @property
    def n(self) -> int:
        return self.a_keys.shape[0]

    @property
    def m(self) -> int:
        return self.b_keys.shape[0]

    def to(self, device) -> "MergeInput":
        f = lambda t: None if t is None else t.to(device)
        return MergeInput(self.key_type, f(self.a_keys), f(self.b_keys), f(self.a_vals), f(self.b_vals))


@dataclasses.dataclass
class SortInput:
    key_type: str
    keys: torch.Tensor
    vals: Optional[torch.Tensor]

    @property
    def N(self) -> int:
        return self.keys.shape[0]


def source_payloads(n: int, m: int, device="cpu"):
    """R13: A[i] -> i, B[j] -> 0x80000000 | j (uint32 bits in int32)."""
    assert n < (1 << 31) and m < (1 << 31)
    a = torch.arange(n, dtype=torch.int32, device=device)
    b = torch.arange(m, dtype=torch.int64, device=device) | (1 << 31)
    b = b.to(torch.int32) if m == 0 else (b - (1 << 32)).to(torch.int32)
    return a, b


def _keys(dist: str, key_type: str, seed: int, stream: int, count: int, device) -> torch.Tensor:
    dtype, order, _ = KEY_TYPES[key_type]
    r = splitmix_stream(seed, stream, count, device)
    if order == "f":
        ftype = torch.float32 if dtype == torch.int32 else torch.float64
        if dist.startswith("bounded:"):             # small integers, negatives too, many ties
            k = int(dist.split(":", 1)[1])
            return (bounded(r, k) - k // 2).to(ftype).view(dtype)
        if dist == "full":                          # every bit pattern: NaNs, infinities, subnormals
            return r.to(dtype)
        if dist == "special":
            table = torch.tensor([_s64(v) if dtype == torch.int64 else (v - (1 << 32) if v >= (1 << 31) else v)
                                  for v in _SPECIAL[key_type]], dtype=dtype, device=device)
            return table[bounded(r, table.numel())]
        if dist == "equal":
            return torch.zeros(count, dtype=dtype, device=device)
        raise ValueError(dist)
    if dist.startswith("bounded:"):
        k = int(dist.split(":", 1)[1])
        v = bounded(r, k)
    elif dist == "full":
        v = _lsr(r, 32) if dtype == torch.int32 else r
        if dtype == torch.int32:
            v = torch.where(v >= (1 << 31), v - (1 << 32), v)
    elif dist.startswith("mostly:"):
        # "mostly:<V>:<num>/<den>": key = V with probability num/den, else r.
        _, vs, frac = dist.split(":")
        num, den = (int(t) for t in frac.split("/"))
        V = _s64(int(vs, 0))
        bern = bounded(splitmix_stream(seed, STREAM_BERN * 16 + stream, count, device), den) < num
        v = torch.where(bern, torch.full_like(r, V), r)
    elif dist == "equal":
        v = torch.zeros(count, dtype=torch.int64, device=device)
    else:
        raise ValueError(dist)
    return v.to(dtype)


def u128_keys(dist: str, seed: int, stream: int, count: int, device="cpu") -> torch.Tensor:
    """(count, 2) int64 = (lo, hi) words of unsigned 128-bit keys:
    "full" both words uniform; "tuple:K" hi uniform in [0, K) and lo in
    [0, 4) -- (key, tie) pairs with many equal keys and equal ties;
    "equal" all zero."""
    if dist == "equal":
        return torch.zeros(count, 2, dtype=torch.int64, device=device)
    r_lo = splitmix_stream(seed, stream, count, device)
    r_hi = splitmix_stream(seed, 16 * STREAM_BERN + 12 + stream, count, device)
    if dist == "full":
        lo, hi = r_lo, r_hi
    elif dist.startswith("tuple:"):
        lo, hi = bounded(r_lo, 4), bounded(r_hi, int(dist.split(":", 1)[1]))
    else:
        raise ValueError(dist)
    return torch.stack([lo, hi], 1).contiguous()


def u128_order(keys: torch.Tensor, descending: bool = False, seg: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Permutation sorting (segment, hi, lo) unsigned, stably (library sorts)."""
    idx = torch.sort(_order_key(keys[:, 0], "u"), stable=True, descending=descending).indices
    idx = idx[torch.sort(_order_key(keys[idx, 1], "u"), stable=True, descending=descending).indices]
    if seg is not None:
        idx = idx[torch.sort(seg[idx], stable=True).indices]
    return idx


def merge_input(n: int, m: int, key_type: str, dist: str, seed: int, payload: bool = True,
                device="cpu", descending: bool = False) -> MergeInput:
    """Two independently sorted arrays A (n) and B (m) of `dist` keys
    (non-increasing when `descending`)."""
    if key_type == "u128":
        a = u128_keys(dist, seed, STREAM_A, n, device)
        b = u128_keys(dist, seed, STREAM_B, m, device)
        a, b = a[u128_order(a, descending)], b[u128_order(b, descending)]
        av = bv = None
        if payload:
            av, bv = source_payloads(n, m, device)
        return MergeInput(key_type, a, b, av, bv)
    _, order, _ = KEY_TYPES[key_type]
    a = sort_bits(_keys(dist, key_type, seed, STREAM_A, n, device), order)
    b = sort_bits(_keys(dist, key_type, seed, STREAM_B, m, device), order)
    if descending:
        a, b = a.flip(0), b.flip(0)
    av = bv = None
    if payload:
        av, bv = source_payloads(n, m, device)
    return MergeInput(key_type, a, b, av, bv)


def sharded_merge_blocks(n_per: int, world: int, rank: int, seed: int, device="cpu"):
    """Rank `rank`'s blocks of a C2-class sharded merge (bench.py at N > 1):
    A and B of n_per * world int32 keys each, uniform over the full int32
    range, sorted, split into the paper's blocks of n_per (p = world).  The
    blocks are drawn stratified -- block r holds n_per keys uniform in the
    r-th 1/world of the key range, sorted -- so every rank makes its own
    blocks and their concatenation is the sorted array.  Returns (A_r, B_r)."""
    W = (1 << 32) // world
    lo = -(1 << 31) + rank * W
    width = W if rank < world - 1 else (1 << 32) - rank * W
    out = []
    for stream in (STREAM_A, STREAM_B):
        r = splitmix_stream(seed, 64 * stream + rank, n_per, device)
        k = (bounded(r, width) + lo).to(torch.int32)
        out.append(torch.sort(k).values)
    return out[0], out[1]


def sort_input(N: int, key_type: str, dist: str, seed: int, payload: bool = True, device="cpu") -> SortInput:
    keys = u128_keys(dist, seed, STREAM_SORT, N, device) if key_type == "u128" else \
        _keys(dist, key_type, seed, STREAM_SORT, N, device)
    vals = torch.arange(N, dtype=torch.int32, device=device) if payload else None
    return SortInput(key_type, keys, vals)


@dataclasses.dataclass
class BatchInput:
    key_type: str
    a_keys: torch.Tensor
    b_keys: torch.Tensor
    a_vals: Optional[torch.Tensor]
    b_vals: Optional[torch.Tensor]
    a_offsets: torch.Tensor      # int64 [S+1]
    b_offsets: torch.Tensor

    @property
    def S(self) -> int:
        return self.a_offsets.numel() - 1

    @property
    def n(self) -> int:
        return self.a_keys.shape[0]

    @property
    def m(self) -> int:
        return self.b_keys.shape[0]

    def to(self, device) -> "BatchInput":
        f = lambda t: None if t is None else t.to(device)
        return BatchInput(self.key_type, f(self.a_keys), f(self.b_keys), f(self.a_vals), f(self.b_vals),
                          f(self.a_offsets), f(self.b_offsets))


def _segmented(S: int, mean: int, key_type: str, dist: str, seed: int, stream: int, device,
               descending: bool = False):
    """S segments of lengths uniform in [0, 2*mean), each sorted (library
    sort on (segment, key)); returns (keys, offsets)."""
    _, order, _ = KEY_TYPES[key_type]
    lens = bounded(splitmix_stream(seed, 16 * STREAM_BERN + 8 + stream, S, device), 2 * mean)
    off = torch.zeros(S + 1, dtype=torch.int64, device=device)
    off[1:] = torch.cumsum(lens, 0)
    total = int(off[-1].item())
    seg = torch.repeat_interleave(torch.arange(S, device=device), lens)
    if key_type == "u128":
        keys = u128_keys(dist, seed, stream, total, device)
        return keys[u128_order(keys, descending, seg)], off
    keys = _keys(dist, key_type, seed, stream, total, device)
    # order by (segment, key): a stable sort by key, then a stable sort by segment
    idx = torch.sort(_order_key(keys, order), stable=True, descending=descending).indices
    idx = idx[torch.sort(seg[idx], stable=True).indices]
    return keys[idx], off


def batch_input(S: int, mean: int, key_type: str, dist: str, seed: int, payload: bool = True,
                device="cpu", descending: bool = False) -> BatchInput:
    """S independent merge pairs, segment lengths
    uniform in [0, 2*mean) on each side, keys of `dist` sorted per segment;
    payloads as R13 over the concatenated arrays."""
    a, aoff = _segmented(S, mean, key_type, dist, seed, STREAM_A, device, descending)
    b, boff = _segmented(S, mean, key_type, dist, seed, STREAM_B, device, descending)
    av = bv = None
    if payload:                                     # one payload per key (u128 keys are (N, 2) rows)
        av, bv = source_payloads(a.shape[0], b.shape[0], device)
    return BatchInput(key_type, a, b, av, bv, aoff, boff)


# BASELINE.json configs (index 1..5 as in SURVEY.md §8).  `scale` divides the
# sizes (power of two) for small parity cases of the same distribution.
CONFIGS = {
    1: dict(kind="merge", n=1 << 20, m=1 << 20, key_type="u32", dist="bounded:65536", payload=True),
    2: dict(kind="merge", n=1 << 26, m=1 << 26, key_type="i32", dist="full", payload=False),
    3: dict(kind="merge", n=1 << 28, m=1 << 16, key_type="i64", dist="bounded:1000", payload=True),
    4: dict(kind="merge", n=1 << 27, m=1 << 25, key_type="u64", dist="mostly:0x8000000000000000:9/10",
            payload=True),
    5: dict(kind="sort", N=1 << 28, key_type="u32", dist="bounded:1048576", payload=True),
    # not a BASELINE.json config: the batched-merge NEXT row,
    # 2^16 pairs of mean 2^10 + 2^10 elements (~1.3e8 elements), C1's key mix
    6: dict(kind="batch", S=1 << 16, mean=1 << 10, key_type="u32", dist="bounded:65536", payload=True),
}


def config_input(cfg: int, scale: int = 1, device="cpu"):
    c = CONFIGS[cfg]
    seed = BASE_SEED + cfg
    if c["kind"] == "merge":
        return merge_input(max(c["n"] // scale, 1), max(c["m"] // scale, 1), c["key_type"], c["dist"], seed,
                           c["payload"], device)
    if c["kind"] == "batch":
        return batch_input(max(c["S"] // scale, 1), c["mean"], c["key_type"], c["dist"], seed, c["payload"], device)
    return sort_input(max(c["N"] // scale, 1), c["key_type"], c["dist"], seed, c["payload"], device)


def elem_bytes(key_type: str, payload: bool) -> int:
    return KEY_TYPES[key_type][2] + (4 if payload else 0)
