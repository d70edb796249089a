"""CPU-side checks of the C ABI (no GPU compute): the library loads, exports
every symbol include/ahs.h declares, the host FSM agrees with the oracle's,
and the no-device / bad-argument paths fail loudly."""
import ctypes as C
import itertools
import math
import os
import re

import numpy as np
import pytest

import oracle
import paper_2506_20677_b200 as ahs
from paper_2506_20677_b200 import build as ahs_build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    ahs_build.build()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "ahs.h")).read()
    return sorted(set(re.findall(r"AHS_API[^;(]*?\b(ahs_\w+)\s*\(", src)))


def test_header_declares_the_three_calls():
    syms = header_symbols()
    for s in ("ahs_features", "ahs_select", "ahs_sort"):
        assert s in syms
    assert len(syms) >= 15


def test_library_exports_every_header_symbol():
    L = C.CDLL(ahs.lib_path())
    for s in header_symbols():
        assert hasattr(L, s), s
    # nothing but the API is exported (static cudart hidden)
    out = os.popen(f"nm -D --defined-only {ahs.lib_path()}").read()
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    assert exported == set(header_symbols()), exported ^ set(header_symbols())


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {ahs.lib_path()}").read()
    assert "sm_100a" in out


def test_defaults_table_ii():
    th = ahs.ahs_thresholds_default()
    assert (th.n_insertion, th.k_counting, th.k_radix) == (20, 1024, 1_000_000)
    assert th.entropy_coeff == 0.7 and th.entropy_norm == 0


def test_sizes():
    assert ahs.ahs_workspace_bytes(1) >= (65536 * 2 + 1) * 4
    a, b = ahs.ahs_sort_tmp_bytes(1 << 20, False), ahs.ahs_sort_tmp_bytes(1 << 20, True)
    assert a >= 4 << 20 and b >= a + (4 << 20)
    assert ahs.ahs_host_scratch_bytes(1000, True) > ahs.ahs_host_scratch_bytes(1000, False)


def _pair(n, k, H, nb, norm=0, **th):
    f = ahs.Features()
    f.n, f.k, f.entropy, f.nbins = n, k, H, nb
    s, r = ahs.ahs_select(f, ahs.ahs_thresholds_default(entropy_norm=norm, **th))
    of = oracle.Features()
    of.n, of.k, of.entropy, of.nb = n, k, H, nb
    s4, r4 = oracle.select(of, norm=norm, **th)
    return (ahs.STRATEGY_NAMES[s], ahs.RULE_NAMES[r]), (oracle.gpu_strategy(s4), oracle.RULE_NAMES[r4])


def test_host_fsm_matches_oracle_fsm_grid():
    ns = [0, 1, 2, 19, 20, 21, 1000, 10 ** 6]
    ks = [1, 2, 999, 1000, 1023, 1024, 1025, 10 ** 6 - 1, 10 ** 6, 10 ** 6 + 1, 2 ** 24 + 1, 2 ** 32]
    for n, k in itertools.product(ns, ks):
        bits = (k - 1).bit_length()
        nb = ((k - 1) >> max(0, bits - 16)) + 1
        for norm in (0, 1):
            thr = 0.7 * math.log2(nb if norm == 0 else k)
            for H in (0.0, 1.0, thr - 1e-9, thr, thr + 1e-9, 16.0, 32.0):
                a, b = _pair(n, k, H, nb, norm)
                assert a == b, (n, k, H, nb, norm, a, b)


def test_host_fsm_spec_examples():
    assert _pair(10, 10 ** 9, 20.0, 61036)[0] == ("GENERAL", "SMALL_N")
    assert _pair(10 ** 4, 500, 5.0, 500)[0] == ("COUNTING", "SMALL_RANGE")
    assert _pair(10 ** 4, 10 ** 7, 3.0, 39063)[0] == ("RADIX", "LOW_ENTROPY")
    assert _pair(10 ** 4, 10 ** 5, 10.0, 10 ** 5 >> 1)[0] == ("GENERAL", "DEFAULT")


def test_host_fsm_custom_thresholds():
    a, b = _pair(5000, 1000, 5.0, 1000, k_counting=500)
    assert a == b == ("GENERAL", "DEFAULT")
    a, b = _pair(15, 100, 5.0, 100, n_insertion=10)
    assert a == b == ("COUNTING", "SMALL_RANGE")


def test_host_fsm_rejects_bad_thresholds():
    f = ahs.Features()
    f.n, f.k, f.nbins = 100, 100, 100
    for bad in (dict(n_insertion=0), dict(k_counting=2_000_000), dict(entropy_coeff=0.0),
                dict(entropy_coeff=1.01), dict(entropy_norm=7), dict(reserved=1)):
        with pytest.raises(ahs.AhsError):
            ahs.ahs_select(f, ahs.ahs_thresholds_default(**bad))


def test_sort_passes_eq4():
    f = ahs.Features()
    f.n = 100
    for k, p in ((10 ** 6, 3), (10 ** 8, 4), (256, 1), (257, 2), (2 ** 32, 4), (2 ** 24, 3), (2 ** 24 + 1, 4)):
        f.k = k
        f.bits = (k - 1).bit_length()
        f.shift = max(0, f.bits - 16)
        assert ahs.ahs_sort_passes(f, ahs.AHS_RADIX, False) == p
        assert ahs.ahs_sort_passes(f, ahs.AHS_GENERAL, True) == 4


def test_empty_features_without_device():
    L = ahs.lib()
    f = ahs.Features()
    rc = L.ahs_features(None, 0, ahs.AHS_I32, None, 0, C.byref(f), None)
    assert rc == 0 and f.n == 0 and f.flags & 1
    s, r = ahs.ahs_select(f)
    assert (ahs.STRATEGY_NAMES[s], ahs.RULE_NAMES[r]) == ("COUNTING", "EMPTY")


def test_bad_arguments_fail_loudly():
    L = ahs.lib()
    f = ahs.Features()
    assert L.ahs_features(None, 0, 7, None, 0, C.byref(f), None) == -1          # bad dtype
    assert L.ahs_features(None, 10, 0, None, 0, C.byref(f), None) == -1         # NULL keys
    assert L.ahs_features(C.c_void_p(4096), 1 << 31, 0, C.c_void_p(4096), 1 << 30, C.byref(f), None) == -3
    assert L.ahs_features(C.c_void_p(4098), 10, 0, C.c_void_p(4096), 1 << 30, C.byref(f), None) == -1  # misaligned
    assert L.ahs_features(C.c_void_p(4096), 10, 0, C.c_void_p(4096), 16, C.byref(f), None) == -2      # ws small
    f.n = 5
    assert L.ahs_sort(C.c_void_p(4096), None, C.c_void_p(8192), None, 6, 2, C.byref(f), None, 0,
                      None, 0, None) == -4                                                  # feat mismatch
    assert L.ahs_sort(C.c_void_p(4096), None, C.c_void_p(8192), None, 5, 9, C.byref(f), None, 0,
                      None, 0, None) == -1                                                  # bad strategy


def test_entropy_sorted_arguments():
    L = ahs.lib()
    h = C.c_double(-1.0)
    assert L.ahs_entropy_sorted(None, 0, None, 0, C.byref(h), None) == 0 and h.value == 0.0  # empty
    assert L.ahs_entropy_sorted(None, 10, None, 0, C.byref(h), None) == -1                    # NULL keys
    assert L.ahs_entropy_sorted(C.c_void_p(4098), 10, C.c_void_p(4096), 1 << 30, C.byref(h), None) == -1
    assert L.ahs_entropy_sorted(C.c_void_p(4096), 10, C.c_void_p(4096), 16, C.byref(h), None) == -2
    assert L.ahs_entropy_sorted(C.c_void_p(4096), 10, C.c_void_p(4096), 1 << 30, None, None) == -1


def test_new_entry_points_check_arguments():
    """NEXT-3 / NEXT-4 entry points reject bad arguments before touching a device."""
    L = ahs.lib()
    f = ahs.Features()
    f.n, f.dtype = 5, ahs.AHS_U32
    # ahs_sort_ex: values of 3 bytes, misaligned 8-byte values
    assert L.ahs_sort_ex(C.c_void_p(4096), C.c_void_p(8192), C.c_void_p(12288), C.c_void_p(16384), 5, 3, 2,
                         C.byref(f), None, 0, None, 0, None) == -1
    assert L.ahs_sort_ex(C.c_void_p(4096), C.c_void_p(8196), C.c_void_p(12288), C.c_void_p(16384), 5, 8, 2,
                         C.byref(f), None, 0, None, 0, None) == -1
    assert L.ahs_sort_tmp_bytes_ex(100, 3, 0) == 0 and L.ahs_sort_tmp_bytes_ex(100, 8, 9) == 0
    assert L.ahs_sort_tmp_bytes_ex(1 << 20, 8, 3) > L.ahs_sort_tmp_bytes_ex(1 << 20, 4, 3) > \
        L.ahs_sort_tmp_bytes_ex(1 << 20, 0, 3) > L.ahs_sort_tmp_bytes_ex(1 << 20, 0, 1)
    # 64-bit keys must be 8-byte aligned
    assert L.ahs_features(C.c_void_p(4100), 10, ahs.AHS_U64, C.c_void_p(4096), 1 << 30, C.byref(f), None) == -1
    # segment sort: above the 8192-key limit, bad dtype, missing counter
    bad = C.c_void_p(4096)
    assert L.ahs_sort_segments(C.c_void_p(4096), None, C.c_void_p(8192), None, 10, C.c_void_p(12288), 2, 8193,
                               0, bad, None) == -3
    assert L.ahs_sort_segments(C.c_void_p(4096), None, C.c_void_p(8192), None, 10, C.c_void_p(12288), 2, 32,
                               7, bad, None) == -1
    assert L.ahs_sort_segments(C.c_void_p(4096), None, C.c_void_p(8192), None, 10, C.c_void_p(12288), 2, 32,
                               0, None, None) == -1
    # classifier: NULL inputs
    h = C.c_void_p()
    assert L.ahs_model_load(None, 0, C.byref(h), None, 0) == -1
    a = C.c_int32()
    assert L.ahs_model_predict(None, 1.0, 1.0, 1.0, C.byref(a), None) == -1


@pytest.mark.skipif(os.path.exists("/dev/nvidia0"), reason="checks the no-GPU path")
def test_no_device_is_an_error_not_a_fallback():
    L = ahs.lib()
    f = ahs.Features()
    rc = L.ahs_features(C.c_void_p(4096), 10, 0, C.c_void_p(4096), 1 << 30, C.byref(f), None)
    assert rc == -6   # AHS_ENODEV
    h = C.c_double()
    assert L.ahs_entropy_sorted(C.c_void_p(4096), 10, C.c_void_p(4096), 1 << 30, C.byref(h), None) == -6


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2506_20677_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).replace("oracle/", ""), fn
