"""CPU oracle for arXiv 1202.6575 (stable two-way merge and stable merge sort).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this
package.  The product path (`paper_1202_6575_b200`) never imports it, and this
package imports nothing from the product path: the two share no code.

Contents
  oracle.c   O1 merge, O2 sort, rank_low/rank_high, O4 closed-form positions
             (plain C, single thread, built by `build()` with gcc)
  plan.py    O3: the paper's Steps 1-4 (block partition, cross ranks,
             classification into cases (a)-(e)), in plain Python, used to pin
             the worked example of Fig. 1 and to compare the device plan.

Pins (tests/test_oracle.py, `-m "not gpu"`): Fig. 1 golden values
(tests/golden/fig1.json), brute-force stable sort of the tagged concatenation,
Python's stable `sorted`, the closed-form positions, exhaustive small
instances and the output invariants.  No function here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# u128: unsigned 128-bit keys as (lo, hi) little-endian uint64 pairs (the
# bytes of a C unsigned __int128); torch carrier: int64 tensors of shape (N, 2)
U128 = np.dtype([("lo", "<u8"), ("hi", "<u8")])
NP_DTYPES = {"u32": np.uint32, "i32": np.int32, "i64": np.int64, "u64": np.uint64, "f32": np.float32,
             "f64": np.float64, "u128": U128}
_C_KEY = {"u32": ctypes.c_uint32, "i32": ctypes.c_int32, "i64": ctypes.c_int64, "u64": ctypes.c_uint64,
          "f32": ctypes.c_float, "f64": ctypes.c_double}

_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c into liboracle.so (gcc, -O2, no vectorisation tricks)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", _LIB, _SRC])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        I = ctypes.c_int64
        for kt in list(NP_DTYPES) + [f"desc_{k}" for k in NP_DTYPES]:
            getattr(_lib, f"oracle_merge_{kt}").argtypes = [P, P, I, P, P, I, P, P]
            getattr(_lib, f"oracle_merge_{kt}").restype = None
            getattr(_lib, f"oracle_sort_{kt}").argtypes = [P, P, I]
            getattr(_lib, f"oracle_sort_{kt}").restype = ctypes.c_int
            if not kt.endswith("u128"):
                getattr(_lib, f"oracle_rank_low_{kt}").argtypes = [_C_KEY[kt.replace("desc_", "")], P, I]
                getattr(_lib, f"oracle_rank_low_{kt}").restype = I
                getattr(_lib, f"oracle_rank_high_{kt}").argtypes = [_C_KEY[kt.replace("desc_", "")], P, I]
                getattr(_lib, f"oracle_rank_high_{kt}").restype = I
            else:
                for f in ("low", "high"):
                    getattr(_lib, f"oracle_rank_{f}_ptr_{kt}").argtypes = [P, P, I]
                    getattr(_lib, f"oracle_rank_{f}_ptr_{kt}").restype = I
            getattr(_lib, f"oracle_merge_wide_{kt}").argtypes = [P, P, I, P, P, I, P, P, I]
            getattr(_lib, f"oracle_merge_wide_{kt}").restype = None
            getattr(_lib, f"oracle_sort_wide_{kt}").argtypes = [P, P, I, I]
            getattr(_lib, f"oracle_sort_wide_{kt}").restype = ctypes.c_int
            getattr(_lib, f"oracle_positions_{kt}").argtypes = [P, I, P, I, P, P]
            getattr(_lib, f"oracle_positions_{kt}").restype = None
            getattr(_lib, f"oracle_positions_sample_{kt}").argtypes = [P, I, P, I, P, I, P, P, I, P]
            getattr(_lib, f"oracle_positions_sample_{kt}").restype = None
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def as_np(x, key_type: str = None):
    """torch CPU tensor / array -> contiguous numpy array.  With `key_type`
    the bits are viewed in that key type (u32/u64 carried in int32/int64)."""
    if x is None:
        return None
    if hasattr(x, "detach"):
        x = x.detach().cpu().contiguous().numpy()
    x = np.ascontiguousarray(x)
    if key_type == "u128":
        if x.dtype == U128:
            return x
        return np.ascontiguousarray(x).view(np.uint64).reshape(-1, 2).view(U128).reshape(-1)
    if key_type is not None:
        x = x.view(NP_DTYPES[key_type])
    return x


def u128_ints(x):
    """u128 keys -> Python ints (high << 64 | low)."""
    a = as_np(x, "u128")
    return [(int(h) << 64) | int(lo) for lo, h in zip(a["lo"], a["hi"])]


def vals_np(x):
    """Payload array -> numpy uint32 view."""
    if x is None:
        return None
    return as_np(x).view(np.uint32)


def _fn(name: str, key_type: str, descending: bool):
    return getattr(lib(), f"oracle_{name}_{'desc_' if descending else ''}{key_type}")


def merge(a_keys, a_vals, b_keys, b_vals, key_type: str, descending: bool = False):
    """O1: the stable merge of A and B, ties to A.  Returns (c_keys, c_vals)
    as numpy arrays (c_vals None when the inputs carry no payload).
    descending=True: the same under the reversed key order."""
    a, b = as_np(a_keys, key_type), as_np(b_keys, key_type)
    va, vb = vals_np(a_vals), vals_np(b_vals)
    assert (va is None) == (vb is None)
    n, m = a.size, b.size
    c = np.empty(n + m, dtype=NP_DTYPES[key_type])
    vc = None if va is None else np.empty(n + m, dtype=np.uint32)
    _fn("merge", key_type, descending)(_ptr(a), _ptr(va), n, _ptr(b), _ptr(vb), m, _ptr(c), _ptr(vc))
    return c, vc


def sort(keys, vals, key_type: str, descending: bool = False):
    """O2: stable bottom-up merge sort.  Returns sorted copies."""
    k = as_np(keys, key_type).copy()
    v = None if vals is None else vals_np(vals).copy()
    rc = _fn("sort", key_type, descending)(_ptr(k), _ptr(v), k.size)
    if rc != 0:
        raise MemoryError("oracle_sort: allocation failed")
    return k, v


def _rows(v, count: int):
    """Payload tensor/array with `count` rows -> contiguous numpy bytes (count, w)."""
    v = np.ascontiguousarray(as_np(v))
    assert v.shape[0] == count
    w = v.dtype.itemsize * int(np.prod(v.shape[1:], dtype=np.int64))
    return np.frombuffer(v.tobytes(), dtype=np.uint8).reshape(count, w), v


def merge_wide(a_keys, a_vals, b_keys, b_vals, key_type: str, descending: bool = False):
    """O1 with payloads of any width: row i of a_vals (any dtype and trailing
    shape) travels with A[i].  Returns (c_keys, c_vals) with c_vals shaped
    and typed like the inputs' rows."""
    a, b = as_np(a_keys, key_type), as_np(b_keys, key_type)
    ra, va = _rows(a_vals, a.size)
    rb, vb = _rows(b_vals, b.size)
    w = ra.shape[1]
    assert rb.shape[1] == w
    c = np.empty(a.size + b.size, dtype=NP_DTYPES[key_type])
    rc = np.empty((a.size + b.size, w), dtype=np.uint8)
    _fn("merge_wide", key_type, descending)(_ptr(a), _ptr(ra), a.size, _ptr(b), _ptr(rb), b.size, _ptr(c),
                                             _ptr(rc), w)
    return c, rc.view(va.dtype).reshape((a.size + b.size,) + va.shape[1:])


def sort_wide(keys, vals, key_type: str, descending: bool = False):
    """O2 with payloads of any width (rows of `vals`).  Returns sorted copies."""
    k = as_np(keys, key_type).copy()
    rv, v = _rows(vals, k.size)
    rv = rv.copy()
    rc = _fn("sort_wide", key_type, descending)(_ptr(k), _ptr(rv), k.size, rv.shape[1])
    if rc != 0:
        raise MemoryError("oracle_sort_wide: allocation failed")
    return k, rv.view(v.dtype).reshape(v.shape)


def _rank_u128(which, x, X, descending):
    X = as_np(X, "u128")
    xa = np.array([(int(x) & ((1 << 64) - 1), int(x) >> 64)], dtype=U128)
    return int(getattr(lib(), f"oracle_rank_{which}_ptr_{'desc_' if descending else ''}u128")(_ptr(xa), _ptr(X),
                                                                                              X.size))


def rank_low(x, X, key_type: str, descending: bool = False) -> int:
    """rank_low(x, X); u128 keys x as a Python int."""
    if key_type == "u128":
        return _rank_u128("low", x, X, descending)
    X = as_np(X, key_type)
    return int(_fn("rank_low", key_type, descending)(NP_DTYPES[key_type](x).item(), _ptr(X), X.size))


def rank_high(x, X, key_type: str, descending: bool = False) -> int:
    if key_type == "u128":
        return _rank_u128("high", x, X, descending)
    X = as_np(X, key_type)
    return int(_fn("rank_high", key_type, descending)(NP_DTYPES[key_type](x).item(), _ptr(X), X.size))


def positions(a_keys, b_keys, key_type: str, descending: bool = False):
    """O4: closed-form output positions."""
    a, b = as_np(a_keys, key_type), as_np(b_keys, key_type)
    pa = np.empty(a.size, dtype=np.int64)
    pb = np.empty(b.size, dtype=np.int64)
    _fn("positions", key_type, descending)(_ptr(a), a.size, _ptr(b), b.size, _ptr(pa), _ptr(pb))
    return pa, pb


def positions_sample(a_keys, b_keys, key_type: str, ia, jb, descending: bool = False):
    """O4 for sampled indices ia (into A) and jb (into B)."""
    a, b = as_np(a_keys, key_type), as_np(b_keys, key_type)
    ia = np.ascontiguousarray(ia, dtype=np.int64)
    jb = np.ascontiguousarray(jb, dtype=np.int64)
    pa = np.empty(ia.size, dtype=np.int64)
    pb = np.empty(jb.size, dtype=np.int64)
    _fn("positions_sample", key_type, descending)(_ptr(a), a.size, _ptr(b), b.size, _ptr(ia), ia.size,
                                                  _ptr(pa), _ptr(jb), jb.size, _ptr(pb))
    return pa, pb
