"""Randomised structured inputs through the whole pipeline (features -> FSM -> sort) against the CPU
oracle: sizes log-uniform up to 2^22, int32 / uint32 keys, with and without values, drawn from
families that exercise the data-dependent paths -- value ranges of every width and offset (digit
placement, trivial-pass skipping, COUNTING / RADIX / GENERAL), keys sharing low bits (multiples
of 2^k: the digit placement at the lowest varying bit), few distinct values with skew (hot digits),
nearly sorted and reversed runs (the warp-uniform paths), and the bucket-local plan's bins (large n,
wide range).  Every case is seeded; the parameters are printed on failure.
"""
import numpy as np
import pytest

import oracle
import synth

from test_gpu_parity import check_pipeline

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2506_20677_b200 as ahs  # noqa: E402


def draw_case(seed: int, n_override=None):
    r = synth.stream(1000 + seed, 16)
    u = [int(x) for x in r]
    n = int(2 ** (1 + (u[0] % 2100) / 100.0))  # log-uniform in [2, 2^22]
    n = min(n, 1 << 22)
    if n_override is not None:  # tests/soak_fuzz.py: larger sizes
        n = int(n_override)
    fam = u[1] % 6
    dt = np.int32 if u[2] & 1 else np.uint32
    kv = bool(u[2] & 2)
    x = synth.stream(2000 + seed, n)
    lo_i = -(2 ** 31) if dt == np.int32 else 0
    if fam == 0:  # a random-width range at a random offset
        w = 1 + u[3] % 32
        span = (1 << w) - 1
        off = lo_i + (u[4] % ((1 << 32) - span)) if span < (1 << 32) - 1 else lo_i
        k = off + synth.uniform_below(x, span + 1).astype(np.int64)
    elif fam == 1:  # multiples of 2^s plus a constant (shared low bits)
        s = 1 + u[3] % 24
        w = 1 + u[4] % (32 - s)
        c = u[5] % (1 << s)
        k = lo_i + c + (synth.uniform_below(x, 1 << w).astype(np.int64) << s)
    elif fam == 2:  # few distinct values, skewed (zipf-like by squaring a uniform)
        m = 2 + u[3] % 3000
        base = lo_i + u[4] % (1 << 31)
        step = 1 + u[5] % 100_000
        j = (synth.unit_f64(x) ** 3 * m).astype(np.int64)
        k = base + j * step
        k = np.clip(k, lo_i, lo_i + (1 << 32) - 1)
    elif fam == 3:  # nearly sorted: ascending with a fraction of random swaps
        k = lo_i + np.arange(n, dtype=np.int64) * (1 + u[3] % 7)
        k = np.clip(k, lo_i, lo_i + (1 << 32) - 1)
        nsw = max(1, n * (u[4] % 50) // 1000)
        a = synth.uniform_below(synth.stream(3000 + seed, nsw), n).astype(np.int64)
        b = synth.uniform_below(synth.stream(4000 + seed, nsw), n).astype(np.int64)
        for i, j in zip(a, b):
            k[i], k[j] = k[j], k[i]
    elif fam == 4:  # descending runs of random length
        run = 1 + u[3] % 5000
        idx = np.arange(n, dtype=np.int64)
        k = lo_i + (idx // run) * run + (run - 1 - idx % run)
        k = np.clip(k, lo_i, lo_i + (1 << 32) - 1)
    else:  # full range (GENERAL; bucket-local plan candidates at large n)
        k = (x >> np.uint64(32)).astype(np.int64) + lo_i
    keys = (k - lo_i).astype(np.uint64).astype(np.uint32)
    if dt == np.int32:
        keys = (keys ^ np.uint32(0x80000000)).view(np.int32)
    vals = synth.stream(5000 + seed, n).astype(np.uint32) if kv else None
    return keys, vals, dict(seed=seed, n=n, family=fam, dtype=np.dtype(dt).name, kv=kv)


@pytest.mark.parametrize("seed", range(128))
def test_random_structured_inputs(seed):
    keys, vals, desc = draw_case(seed)
    try:
        check_pipeline(keys, vals)
    except AssertionError as e:
        raise AssertionError(f"{desc}: {e}") from e
