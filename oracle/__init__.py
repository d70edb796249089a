"""ctypes wrapper for the CPU oracle (oracle/ahs_oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  The product
path (paper_2506_20677_b200) never imports it, and it never imports the
product.  See the header of ahs_oracle.c for the paper passages each function
follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ahs_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

I32, U32, I64, U64 = 0, 1, 2, 3
INSERTION, COUNTING, RADIX, QUICK = 0, 1, 2, 3
STRATEGY4_NAMES = {INSERTION: "insertion", COUNTING: "counting", RADIX: "radix", QUICK: "quick"}
RULE_NAMES = {0: "EMPTY", 1: "CONSTANT", 2: "SMALL_N", 3: "SMALL_RANGE", 4: "LOW_ENTROPY", 5: "DEFAULT"}
FLAG_EMPTY, FLAG_CONSTANT, FLAG_BUCKETED, FLAG_SORTED, FLAG_STRICT_DESC, FLAG_SIGNED = 1, 2, 4, 8, 16, 32
FLAG_K_SATURATED = 64  # k = 2^64 (64-bit keys spanning the whole range): reported as 2^64 - 1

# Table II / reading A3-A5 defaults
DEFAULT_THRESHOLDS = dict(n_insertion=20, k_counting=1024, k_radix=1_000_000,
                          entropy_coeff=0.7, norm=0, entropy_bits=16)


class Features(C.Structure):
    _fields_ = [("n", C.c_uint64), ("min", C.c_int64), ("max", C.c_int64), ("k", C.c_uint64),
                ("bits", C.c_uint32), ("shift", C.c_uint32), ("nb", C.c_uint32), ("dtype", C.c_uint32),
                ("entropy", C.c_double), ("descents", C.c_uint64), ("flags", C.c_uint32),
                ("pad", C.c_uint32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "pad"}

    def key_min(self):
        """min as a Python int in the key's own type (uint64: min holds the bit pattern)."""
        return self.min & 0xFFFFFFFFFFFFFFFF if self.dtype == U64 else self.min

    def key_max(self):
        return self.max & 0xFFFFFFFFFFFFFFFF if self.dtype == U64 else self.max


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain -O2, one thread)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        vp, u64, i32, u32, dbl = C.c_void_p, C.c_uint64, C.c_int, C.c_uint32, C.c_double
        L.oracle_features.argtypes = [vp, u64, i32, u32, C.POINTER(Features), vp]
        L.oracle_h_exact.argtypes = [vp, u64, i32]
        L.oracle_h_exact.restype = dbl
        L.oracle_select.argtypes = [C.POINTER(Features), u64, u64, u64, dbl, i32,
                                    C.POINTER(C.c_int), C.POINTER(C.c_int)]
        for name in ("oracle_counting", "oracle_radix", "oracle_quicksort"):
            getattr(L, name).argtypes = [vp, vp, u64, i32, vp, vp]
        L.oracle_insertion.argtypes = [vp, vp, u64, i32]
        L.oracle_insertion.restype = None
        L.oracle_sort.argtypes = [vp, vp, u64, i32, i32, vp, vp]
        L.oracle_ahs.argtypes = [vp, vp, u64, i32, u64, u64, u64, dbl, i32, u32, vp, vp,
                                 C.POINTER(Features), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        _lib = L
    return _lib


_DTYPES = {np.dtype(np.int32): I32, np.dtype(np.uint32): U32, np.dtype(np.int64): I64, np.dtype(np.uint64): U64}


def _dtype_code(keys: np.ndarray) -> int:
    try:
        return _DTYPES[keys.dtype]
    except KeyError:  # P:409 integers only; 64-bit per S:20 (NEXT-3)
        raise TypeError(f"oracle keys must be int32, uint32, int64 or uint64, got {keys.dtype}") from None


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def features(keys: np.ndarray, entropy_bits: int = 16, with_hist: bool = False):
    keys = np.ascontiguousarray(keys)
    f = Features()
    dt = _dtype_code(keys)
    hist = None
    if with_hist and keys.size:
        # nb <= 2^entropy_bits; allocate the upper bound then trim
        hist = np.zeros(1 << entropy_bits, dtype=np.uint64)
    rc = lib().oracle_features(_ptr(keys), keys.size, dt, entropy_bits, C.byref(f), _ptr(hist))
    if rc:
        raise RuntimeError(f"oracle_features failed rc={rc}")
    if with_hist:
        return f, (hist[: f.nb] if hist is not None else np.zeros(0, np.uint64))
    return f


def h_exact_sorted(sorted_keys: np.ndarray) -> float:
    sorted_keys = np.ascontiguousarray(sorted_keys)
    return lib().oracle_h_exact(_ptr(sorted_keys), sorted_keys.size, _dtype_code(sorted_keys))


def select(f: Features, n_insertion=20, k_counting=1024, k_radix=1_000_000,
           entropy_coeff=0.7, norm=0):
    s, r = C.c_int(), C.c_int()
    rc = lib().oracle_select(C.byref(f), n_insertion, k_counting, k_radix, entropy_coeff, norm,
                             C.byref(s), C.byref(r))
    if rc:
        raise ValueError("invalid thresholds")
    return s.value, r.value


def sort(keys: np.ndarray, vals: np.ndarray | None, strategy4: int):
    """Run one of the paper's four algorithms; returns (keys_out, vals_out|None)."""
    keys = np.ascontiguousarray(keys)
    dt = _dtype_code(keys)
    ok = np.empty_like(keys)
    ov = None
    if vals is not None:
        vals = np.ascontiguousarray(vals, dtype=np.uint32)
        assert vals.shape == keys.shape
        ov = np.empty_like(vals)
    rc = lib().oracle_sort(_ptr(keys), _ptr(vals), keys.size, dt, strategy4, _ptr(ok), _ptr(ov))
    if rc:
        raise RuntimeError(f"oracle_sort({STRATEGY4_NAMES.get(strategy4)}) failed rc={rc}")
    return ok, ov


def ahs(keys: np.ndarray, vals: np.ndarray | None = None, **th):
    """Full pipeline: features -> FSM -> sort.  Returns dict."""
    t = dict(DEFAULT_THRESHOLDS)
    t.update(th)
    keys = np.ascontiguousarray(keys)
    dt = _dtype_code(keys)
    ok = np.empty_like(keys)
    ov = None
    if vals is not None:
        vals = np.ascontiguousarray(vals, dtype=np.uint32)
        ov = np.empty_like(vals)
    f = Features()
    s, r = C.c_int(), C.c_int()
    rc = lib().oracle_ahs(_ptr(keys), _ptr(vals), keys.size, dt, t["n_insertion"], t["k_counting"],
                          t["k_radix"], t["entropy_coeff"], t["norm"], t["entropy_bits"],
                          _ptr(ok), _ptr(ov), C.byref(f), C.byref(s), C.byref(r))
    if rc:
        raise RuntimeError(f"oracle_ahs failed rc={rc}")
    return dict(features=f, strategy4=s.value, rule=r.value, keys=ok, vals=ov)


def gpu_strategy(strategy4: int) -> str:
    """Map the paper's 4 algorithms to the GPU's 3 strategies (INSERTION, QUICK -> GENERAL)."""
    return {INSERTION: "GENERAL", COUNTING: "COUNTING", RADIX: "RADIX", QUICK: "GENERAL"}[strategy4]
