"""NEXT-3 pins: the CPU oracle on 64-bit keys (SPEC's SortKey is i64; k in
128-bit arithmetic), checked against things other than itself:

- brute force: every permutation of 64-bit multisets with the extreme values,
  all four algorithms, against Python's sorted() on (key, index);
- features against Python big-int arithmetic: min, max, descents,
  k = max - min + 1 (saturated at 2^64 - 1 when it is 2^64), bits, shift, nb,
  and H16 re-derived with collections.Counter over the buckets;
- entropy closed forms at the ends of the 64-bit range;
- numpy.argsort(kind='stable') on larger random inputs (genomic-like
  k = 4^30, full-range uint64, int64 across zero).
"""
import collections
import itertools
import math

import numpy as np
import pytest

import oracle

ALGOS = (oracle.INSERTION, oracle.COUNTING, oracle.RADIX, oracle.QUICK)
I64_MIN, I64_MAX, U64_MAX = -(2 ** 63), 2 ** 63 - 1, 2 ** 64 - 1
NP = {"i64": np.int64, "u64": np.uint64}


def stable_ref(keys):
    order = sorted(range(len(keys)), key=lambda i: (int(keys[i]), i))
    return [int(keys[i]) for i in order], order


def _check_all_algos(keys_list, dt):
    keys = np.array(keys_list, dtype=NP[dt])
    vals = np.arange(len(keys_list), dtype=np.uint32)
    ref_k, ref_v = stable_ref(keys_list)
    k = (max(keys_list) - min(keys_list) + 1) if keys_list else 1
    for algo in ALGOS:
        if algo == oracle.COUNTING and k > (1 << 28):
            if keys_list:
                with pytest.raises(RuntimeError):
                    oracle.sort(keys, vals, algo)
            continue
        ok, ov = oracle.sort(keys, vals, algo)
        assert [int(x) for x in ok.tolist()] == ref_k, (keys_list, algo)
        assert ov.tolist() == ref_v, (keys_list, algo)


MULTISETS = {
    "i64_extremes": ("i64", [I64_MIN, -1, -1, 0, 7, I64_MAX, 3]),
    "i64_near": ("i64", [-3, -2, -2, 5, 0, -3, 1]),
    "u64_extremes": ("u64", [0, 1, U64_MAX, 2 ** 63, 2 ** 63 - 1, 2 ** 63, 2 ** 32]),
    "u64_high": ("u64", [2 ** 63 + 5, 2 ** 63 + 5, 2 ** 63 + 1, 2 ** 63 + 9, 2 ** 63, 2 ** 63 + 2]),
}


@pytest.mark.parametrize("name", list(MULTISETS))
def test_exhaustive_permutations_64(name):
    dt, ms = MULTISETS[name]
    for n in range(0, len(ms) + 1):
        for perm in set(itertools.permutations(ms[:n])):
            _check_all_algos(list(perm), dt)


def py_features(keys_list, bits16=16):
    """Features by Python big-int arithmetic (no oracle code)."""
    n = len(keys_list)
    mn, mx = min(keys_list), max(keys_list)
    k = mx - mn + 1
    bits = (k - 1).bit_length()
    shift = max(0, bits - bits16)
    nb = ((k - 1) >> shift) + 1
    desc = sum(1 for i in range(n - 1) if keys_list[i] > keys_list[i + 1])
    c = collections.Counter((x - mn) >> shift for x in keys_list)
    H = -sum((v / n) * math.log2(v / n) for v in c.values())
    H = min(max(H, 0.0), math.log2(nb))
    return dict(min=mn, max=mx, k=k, bits=bits, shift=shift, nb=nb, descents=desc, H=H)


FEATURE_CASES = {
    "full_i64": ("i64", [I64_MIN, I64_MAX, 0, -1, 5]),
    "full_u64": ("u64", [0, U64_MAX, 2 ** 63, 17]),
    "almost_full_u64": ("u64", [1, U64_MAX, 2 ** 40, 3]),
    "genomic_4pow30": ("u64", [0, 4 ** 30 - 1, 12345, 4 ** 29, 4 ** 29]),
    "i64_small_range": ("i64", [-5, -1, -3, -5, 2]),
    "u64_high_const": ("u64", [2 ** 63 + 7] * 4),
}


@pytest.mark.parametrize("name", list(FEATURE_CASES))
def test_features_vs_bigint(name):
    dt, ks = FEATURE_CASES[name]
    f = oracle.features(np.array(ks, dtype=NP[dt]))
    want = py_features(ks)
    assert f.key_min() == (want["min"] & U64_MAX if dt == "u64" else want["min"])
    assert f.key_max() == (want["max"] & U64_MAX if dt == "u64" else want["max"])
    assert f.descents == want["descents"]
    assert f.bits == want["bits"] and f.shift == want["shift"] and f.nb == want["nb"]
    if want["k"] == 2 ** 64:  # k = 2^64 is reported saturated
        assert f.k == U64_MAX and f.flags & oracle.FLAG_K_SATURATED
    else:
        assert f.k == want["k"] and not f.flags & oracle.FLAG_K_SATURATED
    assert abs(f.entropy - want["H"]) <= 1e-12
    assert bool(f.flags & oracle.FLAG_SIGNED) == (dt == "i64")
    assert bool(f.flags & oracle.FLAG_CONSTANT) == (want["k"] == 1)


def test_entropy_closed_forms_64():
    # two equiprobable values at the ends of the range: buckets 0 and 65535, H = 1
    for dt, lo, hi in (("i64", I64_MIN, I64_MAX), ("u64", 0, U64_MAX)):
        ks = np.array([lo, hi] * 50, dtype=NP[dt])
        f = oracle.features(ks)
        assert f.nb == 65536 and f.shift == 48 and abs(f.entropy - 1.0) <= 1e-12
    # 2^16 equiprobable values spread over 2^60 (one per bucket): H = 16
    ks = (np.arange(65536, dtype=np.uint64) << np.uint64(44))
    f = oracle.features(ks)
    assert f.bits == 60 and f.shift == 44 and f.nb == 65536 and abs(f.entropy - 16.0) <= 1e-9


def test_fsm_on_saturated_k():
    ks = np.array([I64_MIN, I64_MAX] * 20 + [0] * 5, dtype=np.int64)
    f = oracle.features(ks)
    assert f.k == U64_MAX
    s, r = oracle.select(f)  # k > 10^6 and H < 0.7 log2 nb (nb = 65536) -> RADIX
    assert s == oracle.RADIX and oracle.RULE_NAMES[r] == "LOW_ENTROPY"
    s, r = oracle.select(f, norm=1)  # RANGE: 0.7 log2(2^64 - 1) ~ 44.8
    assert s == oracle.RADIX


def _rng_keys(kind, n, seed):
    rng = np.random.default_rng(seed)
    if kind == "genomic":  # k = 4^30 (P:120 k-mers)
        return rng.integers(0, 4 ** 30, n, dtype=np.uint64)
    if kind == "full_u64":
        return rng.integers(0, 2 ** 64 - 1, n, dtype=np.uint64, endpoint=True)
    if kind == "i64_cross":
        return rng.integers(-(2 ** 40), 2 ** 40, n, dtype=np.int64)
    if kind == "u64_dups":
        return (rng.integers(0, 50, n, dtype=np.uint64) << np.uint64(57))
    if kind == "i64_small":
        return rng.integers(-300, 300, n, dtype=np.int64)
    raise ValueError(kind)


@pytest.mark.parametrize("kind", ["genomic", "full_u64", "i64_cross", "u64_dups", "i64_small"])
def test_algorithms_vs_numpy_stable_64(kind):
    for n in (1, 2, 21, 1000, 20000):
        ks = _rng_keys(kind, n, 1234 + n)
        vals = np.arange(n, dtype=np.uint32)
        order = np.argsort(ks, kind="stable")
        for algo in ALGOS:
            if algo == oracle.INSERTION and n > 2000:
                continue
            span = int(ks.max()) - int(ks.min()) + 1
            if algo == oracle.COUNTING and span > (1 << 28):
                continue
            ok, ov = oracle.sort(ks, vals, algo)
            assert np.array_equal(ok, ks[order]), (kind, n, algo)
            assert np.array_equal(ov, vals[order]), (kind, n, algo)


def test_radix_digit_count_boundaries():
    # Eq. 4: d = ceil(log_256 k); ranges 2^56 (d = 7) and 2^56 + 1 (d = 8) must both sort
    for span in (2 ** 56, 2 ** 56 + 1, 2 ** 64):
        lo = 3
        hi = lo + span - 1
        if hi > U64_MAX:
            lo, hi = 0, U64_MAX
        ks = np.array([hi, lo, hi - 1, lo + 1, (lo + hi) // 2, lo, hi], dtype=np.uint64)
        ok, _ = oracle.sort(ks, None, oracle.RADIX)
        assert [int(x) for x in ok] == sorted(int(x) for x in ks)
