"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no min/max, entropy, FSM or
sorting).  It only draws keys with a counter-based SplitMix64 so that every
host, every test and every process gets identical bytes for a (config, seed).

Recipe ("Synthetic inputs"):

    mix64(z): z += 0x9E3779B97F4A7C15
              z  = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9
              z  = (z ^ (z >> 27)) * 0x94D049BB133111EB
              return z ^ (z >> 31)
    x_i = mix64(mix64(seed) + i)            (all arithmetic mod 2^64)

    uniform in [0, m)   : ((x >> 32) * m) >> 32
    full 32-bit         : x >> 32
    fp64 uniform [0, 1) : (x >> 11) * 2^-53

The configs are BASELINE.json `configs[0..4]` (cfg1..cfg5).  They stand in for
the paper's workload families (§III.B; Table VII) whose
real corpora (NYC Taxi, IoT, genomic k-mers) are not available here.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    """SplitMix64 output function (Vigna), elementwise on uint64 arrays."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + GAMMA
        z = (z ^ (z >> np.uint64(30))) * M1
        z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def stream(seed: int, n: int, start: int = 0) -> np.ndarray:
    """x_i = mix64(mix64(seed) + i) for i in [start, start + n), uint64."""
    base = mix64(np.uint64(seed & 0xFFFFFFFFFFFFFFFF))
    idx = np.arange(start, start + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return mix64(idx + base)


def uniform_below(x: np.ndarray, m: int) -> np.ndarray:
    """((x >> 32) * m) >> 32  — exact in uint64 for m <= 2^32."""
    assert 0 < m <= (1 << 32)
    hi = x >> np.uint64(32)
    if m == (1 << 32):
        return hi
    with np.errstate(over="ignore"):
        return (hi * np.uint64(m)) >> np.uint64(32)


def unit_f64(x: np.ndarray) -> np.ndarray:
    return (x >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


# ----------------------------------------------------------------------------
# Config recipes (BASELINE.json configs[0..4])
# ----------------------------------------------------------------------------

def _chunked(seed: int, n: int, fn, out_dtype, chunk: int = 1 << 24):
    out = np.empty(n, dtype=out_dtype)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        out[s:e] = fn(stream(seed, e - s, start=s))
    return out


def cfg1(n: int = 1 << 20, seed: int = 1):
    """int32 i.i.d. uniform in [0, 1000)."""
    return _chunked(seed, n, lambda x: uniform_below(x, 1000).astype(np.int32), np.int32)


def cfg2(n: int = 1 << 24, seed: int = 2):
    """uint32 i.i.d. uniform over the full 32-bit range."""
    return _chunked(seed, n, lambda x: (x >> np.uint64(32)).astype(np.uint32), np.uint32)


ZIPF_S = 1.1
ZIPF_K = 4096
CFG3_BASE = 1_000_000
CFG3_STEP = 262_144


def zipf_cdf(k: int = ZIPF_K, s: float = ZIPF_S) -> np.ndarray:
    w = (np.arange(1, k + 1, dtype=np.float64)) ** (-s)
    c = np.cumsum(w)  # sequential fp64 accumulation
    cdf = c / c[-1]
    cdf[-1] = 1.0
    return cdf


def cfg3(n: int = 1 << 26, seed: int = 3):
    """int32, 4096 distinct values 1e6 + 262144*j, j ~ Zipf(1.1) by inverse CDF."""
    cdf = zipf_cdf()

    def f(x):
        j = np.searchsorted(cdf, unit_f64(x), side="right")
        return (CFG3_BASE + CFG3_STEP * j).astype(np.int32)

    return _chunked(seed, n, f, np.int32)


def cfg4a(n: int = 1 << 26, seed: int = 4):
    """int32 ascending 0..n-1 with floor(n/200) transpositions applied in order."""
    a = np.arange(n, dtype=np.int32)
    m = n // 200
    if m == 0:
        return a
    x = stream(seed, 2 * m)
    ij = uniform_below(x, n).astype(np.int64)
    ii = ij[0::2].tolist()
    jj = ij[1::2].tolist()
    for i, j in zip(ii, jj):
        a[i], a[j] = a[j], a[i]
    return a


def cfg4b(n: int = 1 << 26, seed: int = 4):
    """int32 strictly descending n-1 .. 0."""
    return np.arange(n - 1, -1, -1, dtype=np.int32)


def cfg4c(n: int = 1 << 26, seed: int = 4):
    """int32 all keys equal to 42."""
    return np.full(n, 42, dtype=np.int32)


def cfg4d(n: int = 1 << 26, seed: int = 4):
    """int32 uniform in [-8, 8)."""
    return _chunked(seed, n, lambda x: (uniform_below(x, 16).astype(np.int64) - 8).astype(np.int32), np.int32)


CFG5_R = (8, 16, 20, 24, 28, 32)


def cfg5(r: int, n: int = 1 << 28, seed: int | None = None):
    """(uint32 key uniform in [0, 2^r), uint32 value = index), seed 5 + r."""
    if seed is None:
        seed = 5 + r
    sh = np.uint64(32 - r)
    keys = _chunked(seed, n, lambda x: ((x >> np.uint64(32)) >> sh).astype(np.uint32), np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    return keys, vals


# Registry: name -> (dtype, default n, builder(n) -> (keys, vals|None), kv)
def _kv_index(keys):
    return keys, np.arange(keys.shape[0], dtype=np.uint32)


CONFIGS = {
    "cfg1": ("i32", 1 << 20, lambda n: (cfg1(n), None)),
    "cfg2": ("u32", 1 << 24, lambda n: (cfg2(n), None)),
    "cfg2kv": ("u32", 1 << 24, lambda n: _kv_index(cfg2(n))),
    "cfg3": ("i32", 1 << 26, lambda n: (cfg3(n), None)),
    "cfg4a": ("i32", 1 << 26, lambda n: (cfg4a(n), None)),
    "cfg4b": ("i32", 1 << 26, lambda n: (cfg4b(n), None)),
    "cfg4c": ("i32", 1 << 26, lambda n: (cfg4c(n), None)),
    "cfg4d": ("i32", 1 << 26, lambda n: (cfg4d(n), None)),
}
for _r in CFG5_R:
    CONFIGS[f"cfg5_r{_r}"] = ("u32", 1 << 28, (lambda r: (lambda n: cfg5(r, n)))(_r))


def cfg7(n: int = 1 << 28, seed: int = 7):
    """Key-value COUNTING beyond 8-bit digits (not a BASELINE config): (uint32 key
    uniform in [0, 1000), uint32 value = index), 2^28 pairs: k = 1000 <= k_counting (Table II), so
    the FSM picks COUNTING, and the stable scatter needs a 10-bit digit."""
    keys = _chunked(seed, n, lambda x: uniform_below(x, 1000).astype(np.uint32), np.uint32)
    return keys, np.arange(n, dtype=np.uint32)


CONFIGS["cfg7kv"] = ("u32", 1 << 28, lambda n: cfg7(n))


def _cfg6(n: int, kv: bool):
    keys = kmers(6, n)  # NEXT-3: genomic-like 30-mers, k = 4^30, uint64
    return keys, (np.arange(n, dtype=np.uint32) if kv else None)


CONFIGS["cfg6"] = ("u64", 1 << 26, lambda n: _cfg6(n, False))
CONFIGS["cfg6kv"] = ("u64", 1 << 26, lambda n: _cfg6(n, True))


def make(name: str, n: int | None = None):
    """Return (keys ndarray, vals ndarray or None, dtype 'i32'|'u32'|'u64') for a config."""
    dtype, n0, fn = CONFIGS[name]
    keys, vals = fn(n0 if n is None else n)
    return keys, vals, dtype


# ----------------------------------------------------------------------------
# Extra families for edge-case tests (§III.B: uniform-value,
# ascending/descending, sawtooth, alternating).
# ----------------------------------------------------------------------------

def sawtooth(n: int, period: int = 97, dtype=np.int32):
    i = np.arange(n, dtype=np.int64)
    up = (i // period) % 2 == 0
    v = np.where(up, i % period, period - 1 - (i % period))
    return v.astype(dtype)


def alternating(n: int, a: int, b: int, dtype=np.int32):
    v = np.where(np.arange(n) % 2 == 0, a, b)
    return v.astype(dtype)


def uniform_range(seed: int, n: int, lo: int, hi: int, dtype=np.int32):
    """Uniform integers in [lo, hi] (inclusive), hi - lo + 1 <= 2^32."""
    m = hi - lo + 1
    x = stream(seed, n)
    v = uniform_below(x, m).astype(np.int64) + lo
    return v.astype(dtype)


# ---------------------------------------------------------- 64-bit keys (NEXT-3)
def wide_u64(seed: int, n: int) -> np.ndarray:
    """Full-range uint64 keys: the SplitMix64 words themselves."""
    return stream(seed, n)


def wide_i64(seed: int, n: int) -> np.ndarray:
    """Full-range int64 keys (the same words reinterpreted)."""
    return stream(seed, n).view(np.int64)


def kmers(seed: int, n: int, k: int = 30) -> np.ndarray:
    """Genomic-like 2-bit-packed k-mer codes, uniform over [0, 4^k), uint64."""
    assert 1 <= k <= 32
    return stream(seed, n) >> np.uint64(64 - 2 * k)


def uniform_range64(seed: int, n: int, lo: int, hi: int, dtype=np.int64) -> np.ndarray:
    """Uniform integers in [lo, hi] for spans up to 2^32 (uniform_below), as int64 / uint64."""
    m = hi - lo + 1
    x = stream(seed, n)
    v = uniform_below(x, m)
    if dtype == np.uint64:
        with np.errstate(over="ignore"):
            return v + np.uint64(lo)
    return (v.astype(np.int64) + np.int64(lo)).astype(dtype)
