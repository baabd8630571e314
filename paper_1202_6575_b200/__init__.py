"""B200-native stable parallel merge and stable merge sort (arXiv 1202.6575).

Thin Python binding over the C ABI in include/stablemerge.h
(paper_1202_6575_b200/lib/libstablemerge.so): argument marshalling only.
Every step of the path (cross ranks, classification, copy/merge, block sort,
merge rounds) runs in the library's CUDA kernels.  There is no CPU fallback:
importing this package fails loudly if the library is missing.

    merge_stable(a_keys, a_vals, b_keys, b_vals, out_keys=None, out_vals=None)
    merge_stable_batched(a_keys, a_vals, a_offsets, b_keys, b_vals, b_offsets)
    mergesort_stable(keys, vals=None)
    merge_plan(a_keys, b_keys, p_A, p_B)          # Steps 1-4 only (tests)

Tensors may live on a CUDA device (asynchronous on the current stream) or on
the host (the library stages them; the binding then synchronises the stream
so host results are ready on return).  Unsigned keys: pass torch.uint32 /
torch.uint64 tensors, or int32/int64 carriers with key_type="u32"/"u64".
Floating-point keys (float32 / float64, or int32/int64 bit carriers with
key_type="f32"/"f64") are ordered by IEEE 754 totalOrder.  128-bit keys
(key_type="u128", always explicit): int64 tensors of shape (N, 2) holding
(lo, hi) words of the unsigned value hi * 2^64 + lo, i.e. (hi, lo) tuples
in lexicographic order -- "(key, tie)" pairs.  descending=True
uses the reversed key order (inputs and outputs non-increasing; ties still
keep A first / input order).
Payloads: 1-D 32-bit tensors (int32 / uint32) take the fused path; any
other payload (64-bit, or rows of any dtype and trailing shape, e.g. a
(n, 3) float64 tensor or a structured record as uint8 (n, 24)) takes the
wide-payload path (CUDA tensors only): the same method with an index payload
and one row gather.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# SM_LIB_PATH: an alternative build of the same library (tuning experiments:
# scripts/build_variants.py); the default is the in-tree build.
LIB_PATH = os.environ.get("SM_LIB_PATH") or os.path.join(_PKG, "lib", "libstablemerge.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python build_native.py` "
                      "(there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

KEY_TYPES = ("u32", "i32", "i64", "u64", "f32", "f64", "u128")
_BYTES = {"u32": 4, "i32": 4, "i64": 8, "u64": 8, "f32": 4, "f64": 8, "u128": 16}
_DTYPE_KT = {torch.int32: "i32", torch.int64: "i64", torch.uint32: "u32", torch.uint64: "u64",
             torch.float32: "f32", torch.float64: "f64"}
_CARRIER = {"u32": (torch.int32, torch.uint32), "i32": (torch.int32,), "i64": (torch.int64,),
            "u64": (torch.int64, torch.uint64), "f32": (torch.float32, torch.int32),
            "f64": (torch.float64, torch.int64), "u128": (torch.int64,)}

SM_OK, SM_EINVAL, SM_EALIAS, SM_ENOMEM, SM_ECUDA = range(5)
SM_FLAG_NO_PDL = 1
SM_FLAG_MERGE_PATH = 2


class SmOptions(ctypes.Structure):
    _fields_ = [("p_A", ctypes.c_int64), ("p_B", ctypes.c_int64), ("block", ctypes.c_int64),
                ("sort_run", ctypes.c_int64), ("flags", ctypes.c_int64)]


_P, _I = ctypes.c_void_p, ctypes.c_int64
for _kt in KEY_TYPES + tuple(f"desc_{k}" for k in KEY_TYPES):
    for _name, _args in ((f"merge_stable_{_kt}", [_P, _P, _I, _P, _P, _I, _P, _P, _P]),
                         (f"merge_stable_ex_{_kt}", [_P, _P, _I, _P, _P, _I, _P, _P, _P, ctypes.POINTER(SmOptions)]),
                         (f"merge_plan_ex_{_kt}", [_P, _I, _P, _I, _I, _I, _P, _P, _P, _P]),
                         (f"merge_stable_batched_{_kt}", [_P, _P, _I, _P, _P, _P, _I, _P, _I, _P, _P, _P]),
                         (f"ranks_stable_{_kt}", [_P, _I, _P, _I, ctypes.c_int32, _P, _P]),
                         (f"mergesort_stable_{_kt}", [_P, _P, _I, _P]),
                         (f"mergesort_stable_ex_{_kt}", [_P, _P, _I, _P, ctypes.POINTER(SmOptions)]),
                         (f"merge_stable_wide_{_kt}", [_P, _P, _I, _P, _P, _I, _P, _P, _I, _P]),
                         (f"merge_stable_batched_wide_{_kt}", [_P, _P, _I, _P, _P, _P, _I, _P, _I, _P, _P, _I, _P]),
                         (f"mergesort_stable_wide_{_kt}", [_P, _P, _I, _I, _P])):
        _f = getattr(_lib, _name)
        _f.argtypes = _args
        _f.restype = ctypes.c_int
_lib.sm_tile_capacity.argtypes = [ctypes.c_int32, ctypes.c_int32]
_lib.sm_tile_capacity.restype = ctypes.c_int64
_lib.sm_sort_run.argtypes = [ctypes.c_int32, ctypes.c_int32]
_lib.sm_sort_run.restype = ctypes.c_int64
_lib.sm_debug_cover.argtypes = [ctypes.c_void_p, ctypes.c_int64]
_lib.sm_debug_cover.restype = ctypes.c_int
_lib.sm_is_debug_build.argtypes = []
_lib.sm_is_debug_build.restype = ctypes.c_int32
_lib.sm_set_k1_variant.argtypes = [ctypes.c_int32]
_lib.sm_set_k1_variant.restype = None
_lib.sm_set_small_fuse.argtypes = [ctypes.c_int32]
_lib.sm_set_small_fuse.restype = None
_lib.sm_set_sort_ways.argtypes = [ctypes.c_int32]
_lib.sm_set_sort_ways.restype = None
_lib.sm_sort_merge_passes.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64]
_lib.sm_sort_merge_passes.restype = ctypes.c_int32
_lib.sm_plan_from_ranks.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p]
_lib.sm_plan_from_ranks.restype = ctypes.c_int
_lib.sm_plan_tasks.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                               ctypes.c_void_p, ctypes.c_void_p]
_lib.sm_plan_tasks.restype = ctypes.c_int
_lib.sm_sort_run_n.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64]
_lib.sm_sort_run_n.restype = ctypes.c_int64
_lib.sm_status_string.argtypes = [ctypes.c_int]
_lib.sm_status_string.restype = ctypes.c_char_p
_lib.sm_last_error.argtypes = []
_lib.sm_last_error.restype = ctypes.c_char_p
_lib.sm_last_launch_count.argtypes = []
_lib.sm_last_launch_count.restype = ctypes.c_int64
_lib.sm_profile_enable.argtypes = [ctypes.c_int]
_lib.sm_profile_enable.restype = None
_lib.sm_profile_read.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
_lib.sm_profile_read.restype = ctypes.c_int

PROF_K1, PROF_K2, PROF_K3 = 0, 1, 2


class StableMergeError(RuntimeError):
    def __init__(self, status: int, fn: str):
        self.status = status
        msg = _lib.sm_status_string(status).decode()
        detail = _lib.sm_last_error().decode()
        super().__init__(f"{fn}: {msg}" + (f" ({detail})" if detail else ""))


def _check(status: int, fn: str):
    if status != SM_OK:
        raise StableMergeError(status, fn)


def _key_type(t: torch.Tensor, key_type: Optional[str]) -> str:
    if key_type is None:
        if t.dtype not in _DTYPE_KT:
            raise TypeError(f"unsupported key dtype {t.dtype}")
        if t.dim() != 1:
            raise ValueError("multi-dimensional key tensor: pass key_type='u128' for 128-bit keys")
        return _DTYPE_KT[t.dtype]
    if key_type not in KEY_TYPES:
        raise ValueError(f"key_type must be one of {KEY_TYPES}")
    if t.dtype not in _CARRIER[key_type]:
        raise TypeError(f"key_type {key_type} cannot be carried in {t.dtype}")
    return key_type


def _count(t: torch.Tensor, kt: str) -> int:
    """Number of keys in a key tensor (u128: rows of an (N, 2) int64 tensor)."""
    if kt == "u128":
        if t.dim() != 2 or t.shape[1] != 2:
            raise ValueError("u128 keys are int64 tensors of shape (N, 2) = (lo, hi) words")
        return t.shape[0]
    return t.numel()


def _empty_keys(count: int, like: torch.Tensor, kt: str) -> torch.Tensor:
    shape = (count, 2) if kt == "u128" else (count,)
    return torch.empty(shape, dtype=like.dtype, device=like.device)


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_contiguous():
        raise ValueError("tensors must be contiguous")
    return t.data_ptr() or None


def _vals_ok(t: Optional[torch.Tensor]):
    if t is not None and t.dtype not in (torch.int32, torch.uint32):
        raise TypeError("payloads must be 32-bit (int32 / uint32)")


def _is_wide(*vals) -> bool:
    """Payload rows other than one 32-bit word: the wide-payload path."""
    return any(v is not None and (v.dim() != 1 or v.element_size() != 4) for v in vals)


def _row_bytes(v: torch.Tensor) -> int:
    b = v.element_size()
    for d in v.shape[1:]:
        b *= d
    return b


def _wide_args(a_vals, b_vals):
    if a_vals is None or b_vals is None:
        raise ValueError("payloads must be given for both inputs or neither")
    if a_vals.dtype != b_vals.dtype or a_vals.shape[1:] != b_vals.shape[1:]:
        raise ValueError("A and B payload rows must have the same dtype and shape")
    if not (a_vals.is_cuda and b_vals.is_cuda):
        raise ValueError("wide payloads take CUDA tensors")
    vb = _row_bytes(a_vals)
    if vb < 1 or vb > 4096:
        raise ValueError("payload rows must be 1..4096 bytes")
    return vb


def _sym(op: str, kt: str, descending: bool) -> str:
    return f"{op}_desc_{kt}" if descending else f"{op}_{kt}"


_FN = {}


def _fn(op: str, kt: str, descending: bool):
    """(ctypes function, its name), cached per (op, key type, order)."""
    k = (op, kt, descending)
    f = _FN.get(k)
    if f is None:
        name = _sym(op, kt, descending)
        f = _FN[k] = (getattr(_lib, name), name)
    return f


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream_for(t: torch.Tensor, stream):
    if stream is not None:
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    if t.is_cuda:   # torch's current stream of the tensor's device (the raw handle: no Stream object)
        return _raw_stream(t.device.index) if _raw_stream else torch.cuda.current_stream(t.device).cuda_stream
    return 0


def _sync_if_host(t: torch.Tensor, stream_handle):
    if not t.is_cuda:
        torch.cuda.synchronize() if stream_handle == 0 else \
            torch.cuda.ExternalStream(stream_handle).synchronize()


def tile_capacity(key_type: str = "u32", has_vals: bool = True) -> int:
    return int(_lib.sm_tile_capacity(_BYTES[key_type], int(has_vals)))


def is_debug_build() -> bool:
    return bool(_lib.sm_is_debug_build())


def debug_cover(cover: Optional[torch.Tensor]) -> None:
    """SM_DEBUG builds: K2 counts every output element it stores in `cover`
    (a zeroed int32 CUDA tensor at least as long as the output); None stops."""
    if cover is None:
        _check(_lib.sm_debug_cover(None, 0), "sm_debug_cover")
    else:
        _check(_lib.sm_debug_cover(_ptr(cover), cover.numel()), "sm_debug_cover")


def set_k1_variant(variant: int) -> None:
    """Test hook: 0 automatic, 1 warp per search, 2 sample kernel, 3 thread per search."""
    _lib.sm_set_k1_variant(int(variant))


def set_small_fuse(on: bool) -> None:
    """Small plain merges in one launch (each K2 CTA ranks its own tasks) or
    K1 then K2 (the default)."""
    _lib.sm_set_small_fuse(int(bool(on)))


def set_sort_ways(ways: int) -> None:
    """Merge sort phase 2: 0 (default) automatic, 4 -- two merge rounds per
    HBM pass, 2 -- one round per pass.  Same output."""
    _lib.sm_set_sort_ways(int(ways))


def sort_merge_passes(key_type: str, has_vals: bool, n: int) -> int:
    """Phase-2 HBM passes of a sort of n elements under the current setting."""
    return int(_lib.sm_sort_merge_passes(_BYTES[key_type], int(has_vals), int(n)))


def plan_from_ranks(n: int, m: int, p: int, xbar, ybar) -> list:
    """Test hook: the host's coarse Steps 3-4 on given cross ranks; the 2p
    tasks (a0, a1, b0, b1) ordered by output offset."""
    xb = (ctypes.c_int64 * (p + 1))(*xbar)
    yb = (ctypes.c_int64 * (p + 1))(*ybar)
    out = (ctypes.c_int64 * (8 * p))()
    _check(_lib.sm_plan_from_ranks(n, m, p, xb, yb, out), "sm_plan_from_ranks")
    return [tuple(out[4 * k:4 * k + 4]) for k in range(2 * p)]


def plan_tasks(n: int, m: int, pA: int, pB: int, xbar, ybar) -> list:
    """Steps 3-4 on the host for given cross ranks x̄[0..pA], ȳ[0..pB]: the
    pA + pB tasks (a0, a1, b0, b1) in task order (A-side task i, then B-side
    task j), by the library's classification (sm_plan_tasks)."""
    xb = (ctypes.c_int64 * (pA + 1))(*[int(v) for v in xbar])
    yb = (ctypes.c_int64 * (pB + 1))(*[int(v) for v in ybar])
    out = (ctypes.c_int64 * (4 * (pA + pB)))()
    _check(_lib.sm_plan_tasks(n, m, pA, pB, xb, yb, out), "sm_plan_tasks")
    return [tuple(out[4 * k:4 * k + 4]) for k in range(pA + pB)]


def sort_run(key_type: str = "u32", has_vals: bool = True, n: Optional[int] = None) -> int:
    """Initial run length of the merge sort: the shared-memory block-sort tile
    (n None), or the run length a sort of n elements uses on the current
    device (phase 1 with one block per SM when n is large)."""
    if n is None:
        return int(_lib.sm_sort_run(_BYTES[key_type], int(has_vals)))
    return int(_lib.sm_sort_run_n(_BYTES[key_type], int(has_vals), int(n)))


def last_launch_count() -> int:
    """Kernel launches issued by the last library call on this thread."""
    return int(_lib.sm_last_launch_count())


def profile_enable(on: bool = True):
    """Bracket every library kernel launch with CUDA events on its stream."""
    _lib.sm_profile_enable(int(on))


def profile_read(kind: int):
    """(total ms, launches) of one kernel kind since profile_enable()."""
    t = ctypes.c_double(0.0)
    c = ctypes.c_int64(0)
    _check(_lib.sm_profile_read(kind, ctypes.byref(t), ctypes.byref(c)), "sm_profile_read")
    return t.value, c.value


def _options(p_A, p_B, block, flags, sort_run_=None):
    if p_A is None and p_B is None and block is None and not flags and sort_run_ is None:
        return None
    return SmOptions(p_A or 0, p_B or 0, block or 0, sort_run_ or 0, flags or 0)


def _check_args(pairs, tensors):
    """Every (tensor, expected rows, what) holds exactly that many rows, and
    every tensor lives on one device: the C ABI trusts the sizes it is given
    (a short buffer would be read or written past its end on the GPU)."""
    for t, want, what in pairs:
        if t is not None and int(t.shape[0] if t.dim() else 1) != want:
            raise ValueError(f"{what} must hold {want} rows, has {int(t.shape[0]) if t.dim() else 1}")
    devs = {t.device for t in tensors if t is not None}
    if len(devs) > 1:
        raise ValueError(f"all tensors must be on one device, got {sorted(map(str, devs))}")


def merge_stable(a_keys: torch.Tensor, a_vals: Optional[torch.Tensor], b_keys: torch.Tensor,
                 b_vals: Optional[torch.Tensor], out_keys: Optional[torch.Tensor] = None,
                 out_vals: Optional[torch.Tensor] = None, *, key_type: Optional[str] = None, stream=None,
                 p_A: Optional[int] = None, p_B: Optional[int] = None, block: Optional[int] = None,
                 pdl: bool = True, merge_path: bool = False, descending: bool = False):
    """Stable merge of sorted A and B (ties: A first).  Returns (keys, vals).
    merge_path=True runs the equal-output merge-path COMPARISON instead of the
    paper's method (same result; CUDA tensors only)."""
    kt = _key_type(a_keys, key_type)
    _key_type(b_keys, kt)
    if (a_vals is None) != (b_vals is None):
        raise ValueError("payloads must be given for both inputs or neither")
    n, m = _count(a_keys, kt), _count(b_keys, kt)
    if _is_wide(a_vals, b_vals):
        vb = _wide_args(a_vals, b_vals)
        if out_keys is None:
            out_keys = _empty_keys(n + m, a_keys, kt)
        if out_vals is None:
            out_vals = torch.empty((n + m,) + tuple(a_vals.shape[1:]), dtype=a_vals.dtype, device=a_keys.device)
        _check_args([(a_vals, n, "a_vals"), (b_vals, m, "b_vals"), (out_vals, n + m, "out_vals")],
                    [a_keys, b_keys, a_vals, b_vals, out_keys, out_vals])
        if _count(out_keys, kt) != n + m or (n + m and out_vals.element_size() * out_vals[0:1].numel() != vb):
            raise ValueError("outputs must hold n + m keys and rows of the payloads' width")
        s = _stream_for(a_keys, stream)
        fn = _sym("merge_stable_wide", kt, descending)
        _check(getattr(_lib, fn)(_ptr(a_keys), _ptr(a_vals), n, _ptr(b_keys), _ptr(b_vals), m, _ptr(out_keys),
                                 _ptr(out_vals), vb, s), fn)
        return out_keys, out_vals
    _vals_ok(a_vals); _vals_ok(b_vals)
    if out_keys is None:
        out_keys = _empty_keys(n + m, a_keys, kt)
    if a_vals is not None and out_vals is None:
        out_vals = torch.empty(n + m, dtype=a_vals.dtype, device=a_keys.device)
    if _count(out_keys, kt) != n + m or (out_vals is not None and out_vals.numel() != n + m):
        raise ValueError("output length must be n + m")
    _check_args([(a_vals, n, "a_vals"), (b_vals, m, "b_vals")], [a_keys, b_keys, a_vals, b_vals, out_keys, out_vals])
    s = _stream_for(a_keys, stream)
    opt = _options(p_A, p_B, block, (0 if pdl else SM_FLAG_NO_PDL) | (SM_FLAG_MERGE_PATH if merge_path else 0))
    args = (_ptr(a_keys), _ptr(a_vals), n, _ptr(b_keys), _ptr(b_vals), m, _ptr(out_keys), _ptr(out_vals), s)
    if opt is None:
        f, name = _fn("merge_stable", kt, descending)
        st = f(*args)
    else:
        f, name = _fn("merge_stable_ex", kt, descending)
        st = f(*args, ctypes.byref(opt))
    if st:
        _check(st, name)
    if not out_keys.is_cuda:
        _sync_if_host(out_keys, s)
    return out_keys, out_vals


def merge_stable_batched(a_keys: torch.Tensor, a_vals: Optional[torch.Tensor], a_offsets: torch.Tensor,
                         b_keys: torch.Tensor, b_vals: Optional[torch.Tensor], b_offsets: torch.Tensor,
                         out_keys: Optional[torch.Tensor] = None, out_vals: Optional[torch.Tensor] = None, *,
                         key_type: Optional[str] = None, stream=None, descending: bool = False):
    """S = len(a_offsets) - 1 independent stable merges (ties: A first):
    segment s of A (a_keys[a_offsets[s]:a_offsets[s+1]]) with segment s of B
    into out[a_offsets[s] + b_offsets[s] : ...].  CUDA tensors only; offsets
    int64.  Returns (keys, vals)."""
    kt = _key_type(a_keys, key_type)
    _key_type(b_keys, kt)
    if (a_vals is None) != (b_vals is None):
        raise ValueError("payloads must be given for both inputs or neither")
    wide = _is_wide(a_vals, b_vals)
    if not wide:
        _vals_ok(a_vals); _vals_ok(b_vals)
    if a_offsets.dtype != torch.int64 or b_offsets.dtype != torch.int64:
        raise TypeError("offsets must be int64")
    if a_offsets.numel() != b_offsets.numel() or a_offsets.numel() < 1:
        raise ValueError("a_offsets and b_offsets must both hold S + 1 entries")
    S = a_offsets.numel() - 1
    n, m = _count(a_keys, kt), _count(b_keys, kt)
    if out_keys is None:
        out_keys = _empty_keys(n + m, a_keys, kt)
    if _count(out_keys, kt) != n + m:
        raise ValueError("out_keys must hold n + m keys")
    _check_args([(a_vals, n, "a_vals"), (b_vals, m, "b_vals"), (out_vals, n + m, "out_vals")],
                [a_keys, b_keys, a_vals, b_vals, a_offsets, b_offsets, out_keys, out_vals])
    s = _stream_for(a_keys, stream)
    if wide:
        vb = _wide_args(a_vals, b_vals)
        if out_vals is None:
            out_vals = torch.empty((n + m,) + tuple(a_vals.shape[1:]), dtype=a_vals.dtype, device=a_keys.device)
        fn = _sym("merge_stable_batched_wide", kt, descending)
        _check(getattr(_lib, fn)(_ptr(a_keys), _ptr(a_vals), n, _ptr(a_offsets), _ptr(b_keys), _ptr(b_vals), m,
                                 _ptr(b_offsets), S, _ptr(out_keys), _ptr(out_vals), vb, s), fn)
        return out_keys, out_vals
    if a_vals is not None and out_vals is None:
        out_vals = torch.empty(n + m, dtype=a_vals.dtype, device=a_keys.device)
    fn = _sym("merge_stable_batched", kt, descending)
    _check(getattr(_lib, fn)(_ptr(a_keys), _ptr(a_vals), n, _ptr(a_offsets), _ptr(b_keys), _ptr(b_vals), m,
                             _ptr(b_offsets), S, _ptr(out_keys), _ptr(out_vals), s), fn)
    return out_keys, out_vals


def ranks_stable(X: torch.Tensor, keys: torch.Tensor, high: bool = False, *, key_type: Optional[str] = None,
                 stream=None, descending: bool = False) -> torch.Tensor:
    """rank_low (high=False) or rank_high (high=True) of every key in sorted
    X.  CUDA tensors; returns int64 ranks."""
    kt = _key_type(X, key_type)
    _key_type(keys, kt)
    nk = _count(keys, kt)
    out = torch.empty(nk, dtype=torch.int64, device=keys.device)
    s = _stream_for(X, stream)
    fn = _sym("ranks_stable", kt, descending)
    _check(getattr(_lib, fn)(_ptr(X), _count(X, kt), _ptr(keys), nk, int(bool(high)), _ptr(out), s), fn)
    return out


def mergesort_stable(keys: torch.Tensor, vals: Optional[torch.Tensor] = None, *, key_type: Optional[str] = None,
                     stream=None, pdl: bool = True, descending: bool = False, run: Optional[int] = None):
    """Stable merge sort in place (equal keys keep input order).  Returns (keys, vals).
    run: the initial run length (tests; sm_options.sort_run)."""
    kt = _key_type(keys, key_type)
    N = _count(keys, kt)
    s = _stream_for(keys, stream)
    if _is_wide(vals):
        if vals.shape[0] != N:
            raise ValueError("vals must have one row per key")
        vb = _wide_args(vals, vals)
        fn = _sym("mergesort_stable_wide", kt, descending)
        _check(getattr(_lib, fn)(_ptr(keys), _ptr(vals), N, vb, s), fn)
        return keys, vals
    _vals_ok(vals)
    if vals is not None and vals.numel() != N:
        raise ValueError("vals must have the same length as keys")
    _check_args([], [keys, vals])
    args = (_ptr(keys), _ptr(vals), N, s)
    if pdl and not run:
        fn = _sym("mergesort_stable", kt, descending)
        _check(getattr(_lib, fn)(*args), fn)
    else:
        opt = SmOptions(0, 0, 0, int(run or 0), 0 if pdl else SM_FLAG_NO_PDL)
        fn = _sym("mergesort_stable_ex", kt, descending)
        _check(getattr(_lib, fn)(*args, ctypes.byref(opt)), fn)
    _sync_if_host(keys, s)
    return keys, vals


def merge_plan(a_keys: torch.Tensor, b_keys: torch.Tensor, p_A: int, p_B: Optional[int] = None, *,
               key_type: Optional[str] = None, stream=None, descending: bool = False):
    """Steps 1-4 on the device: (xbar[p_A+1], ybar[p_B+1], tasks[p_A+p_B, 6]) int64 tensors."""
    kt = _key_type(a_keys, key_type)
    _key_type(b_keys, kt)
    if p_B is None:
        p_B = p_A
    dev = a_keys.device
    if not a_keys.is_cuda:
        raise ValueError("merge_plan takes CUDA tensors")
    xbar = torch.empty(p_A + 1, dtype=torch.int64, device=dev)
    ybar = torch.empty(p_B + 1, dtype=torch.int64, device=dev)
    tasks = torch.empty((p_A + p_B, 6), dtype=torch.int64, device=dev)
    s = _stream_for(a_keys, stream)
    fn = _sym("merge_plan_ex", kt, descending)
    _check(getattr(_lib, fn)(_ptr(a_keys), _count(a_keys, kt), _ptr(b_keys), _count(b_keys, kt), p_A, p_B, _ptr(xbar),
                             _ptr(ybar), _ptr(tasks), s), fn)
    return xbar, ybar, tasks


__all__ = ["merge_stable", "merge_stable_batched", "mergesort_stable", "ranks_stable", "merge_plan", "plan_tasks", "tile_capacity", "sort_run", "last_launch_count",
           "StableMergeError", "KEY_TYPES", "LIB_PATH", "profile_enable", "profile_read", "PROF_K1", "PROF_K2",
           "PROF_K3"]
