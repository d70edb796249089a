"""T4/T5: the CUDA path through the C ABI against the CPU oracle.

Bar: features n/min/max/k/bits/shift/nbins/descents bit-exact, |dH| <= 1e-9
(BASELINE.json north_star), strategy + rule identical, keys and values
bit-exact (the unique stable order).  Sizes span several tiles (onesweep
tiles: 8192 keys (10752 from n = 2^24 on; RADIX: 11264) / 6400 pairs with the ordered ranking,
7680 / 4608 with the masked ranking, which has its own parity test) with ragged
tails, and sizes
where every persistent CTA walks several tiles; full BASELINE.json configs at
the end.
"""
import math

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2506_20677_b200 as ahs  # noqa: E402

H_TOL = 1e-9


@pytest.fixture(scope="module", autouse=True)
def cuda_ready():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    ahs.lib()


def to_dev(a: np.ndarray, misalign: int = 0):
    """Upload; with misalign > 0 the tensor starts `misalign` elements into a buffer."""
    t = torch.from_numpy(a.view(np.int32) if a.dtype == np.uint32 else a)
    if a.dtype == np.uint32:
        base = torch.empty(a.size + misalign, dtype=torch.int32, device="cuda")
        base[misalign:].copy_(t)
        return base.view(torch.uint32)[misalign:]
    base = torch.empty(a.size + misalign, dtype=torch.int32, device="cuda")
    base[misalign:].copy_(t)
    return base[misalign:]


def to_host(t) -> np.ndarray:
    if t.dtype == torch.uint32:
        return t.view(torch.int32).cpu().numpy().view(np.uint32)
    return t.cpu().numpy()


def check_features(f, of):
    assert f.n == of.n
    if of.n == 0:
        return
    assert (f.min, f.max, f.k, f.bits, f.shift, f.nbins, f.descents) == \
        (of.min, of.max, of.k, of.bits, of.shift, of.nb, of.descents)
    assert abs(f.entropy - of.entropy) <= H_TOL
    assert f.flags == of.flags


def run_gpu(keys, vals=None, strategy=None, misalign=0, inplace=False, th=None, stream=None, info=None):
    n = keys.size
    dk = to_dev(keys, misalign)
    dv = to_dev(vals, misalign) if vals is not None else None
    ws = ahs.Workspace(n, vals is not None)
    f = ahs.ahs_features(dk, ws, stream)
    s, r = ahs.ahs_select(f, th)
    if strategy is not None:
        s = strategy
    if inplace:
        ko, vo = dk, dv
    else:
        ko = to_dev(np.zeros_like(keys), misalign)
        vo = to_dev(np.zeros_like(vals), misalign) if vals is not None else None
    ahs.ahs_sort(dk, dv, ko, vo, s, f, ws, stream)
    torch.cuda.synchronize()
    if info is not None:
        info["executed"] = ahs.ahs_sort_executed_passes(ws, stream)
        info["nominal"] = ahs.ahs_sort_passes(f, s, vals is not None)
    return f, s, r, to_host(ko), (to_host(vo) if vo is not None else None)


def expected(keys, vals):
    order = np.argsort(keys, kind="stable")  # only used to cross-check the oracle below
    r = oracle.ahs(keys, vals)
    assert np.array_equal(r["keys"], keys[order])
    return r


def check_pipeline(keys, vals=None, **kw):
    f, s, r, ko, vo = run_gpu(keys, vals, **kw)
    ref = oracle.ahs(keys, vals)
    check_features(f, ref["features"])
    assert ahs.STRATEGY_NAMES[s] == oracle.gpu_strategy(ref["strategy4"])
    assert ahs.RULE_NAMES[r] == oracle.RULE_NAMES[ref["rule"]]
    assert np.array_equal(ko, ref["keys"])
    if vals is not None:
        assert np.array_equal(vo, ref["vals"])
    return f, s, r


def check_forced(keys, vals, strategy, **kw):
    f, s, r, ko, vo = run_gpu(keys, vals, strategy=strategy, **kw)
    ok, ov = oracle.sort(keys, vals, oracle.QUICK)   # the unique stable order
    assert np.array_equal(ko, ok), ahs.STRATEGY_NAMES[strategy]
    if vals is not None:
        assert np.array_equal(vo, ov), ahs.STRATEGY_NAMES[strategy]


# --------------------------------------------------------------- T4 small

SIZES = [1, 2, 3, 4, 5, 7, 8, 15, 16, 17, 21, 33, 1000, 4607, 4608, 4609, 7679, 7680, 7681,
         8191, 8192, 8193, 6399, 6400, 6401, 3 * 7680 + 77, 3 * 8192 + 77, 3 * 6400 + 77, 5 * 4608 + 13,
         65537, 250_001]

FAMILIES = {
    "u1000": lambda n, s: synth.uniform_range(s, n, 0, 999),
    "neg16": lambda n, s: synth.uniform_range(s, n, -8, 7),
    "full32": lambda n, s: synth.uniform_range(s, n, -(2 ** 31), 2 ** 31 - 1),
    "range3M": lambda n, s: synth.uniform_range(s, n, -1_500_000, 1_500_000),
    "zipf_wide": lambda n, s: synth.cfg3(n, seed=s),
    "sawtooth": lambda n, s: synth.sawtooth(n, period=97),
    "desc": lambda n, s: synth.cfg4b(n),
    "alt_extremes": lambda n, s: synth.alternating(n, -(2 ** 31), 2 ** 31 - 1),
    "const": lambda n, s: synth.cfg4c(n),
}


@pytest.mark.parametrize("family", list(FAMILIES))
def test_pipeline_small_sizes(family):
    for i, n in enumerate(SIZES):
        keys = FAMILIES[family](n, 100 + i)
        check_pipeline(keys)
        check_pipeline(keys, np.arange(n, dtype=np.uint32))


@pytest.mark.parametrize("family", ["full32", "zipf_wide", "neg16"])
def test_pipeline_many_tiles_per_cta(family):
    # > 296 resident CTAs x 7680: every persistent CTA takes several tickets,
    # with TMA prefetch across tiles and a ragged last tile
    n = 3_000_017
    keys = FAMILIES[family](n, 7)
    check_pipeline(keys)
    check_pipeline(keys, np.arange(n, dtype=np.uint32))


@pytest.mark.parametrize("n", [2 ** 24 - 1, 2 ** 24, 1561 * 10752, 1561 * 10752 + 1, 3121 * 10752, 3641 * 9216, 2 ** 25 + 77])
def test_large_keys_tile_boundaries(n):
    # keys-only ordered passes over n >= 2^24 run the 512 x 21 shape (tile 10752): the switch-over size
    # and the one below it, exact multiples of the tile, one key past, a multiple of the former 9216
    # tile, and a ragged tail
    keys = FAMILIES["full32"](n, 11)
    check_pipeline(keys)


@pytest.mark.parametrize("n", [11264, 11265, 3 * 11264 - 1, 300 * 11264, 300 * 11264 + 1, 2_000_003])
def test_radix_v2_tile_boundaries(n):
    # RADIX passes over 32-bit keys run K6 v2 at 512 x 22 (tile 11264): one tile, one key past it,
    # a tile short by one, a multiple with every persistent CTA busy, and ragged tails
    keys = synth.cfg3(n, seed=5)
    f, s, r = check_pipeline(keys)
    check_forced(keys, None, ahs.AHS_RADIX)
    check_forced(keys, np.arange(n, dtype=np.uint32), ahs.AHS_RADIX)


@pytest.mark.parametrize("bits,kind", [(25, "uniform"), (26, "uniform"), (28, "uniform"), (26, "nearly_sorted"),
                                       (29, "uniform")])
def test_narrow_top_digit_last_pass(bits, kind):
    # large keys-only sorts whose last pass has a top digit of 1-5 bits (few distinct digits per warp:
    # the returning rank atomic serves same-word lanes in turn), ragged last tile
    n = 2 ** 25 + 77
    if kind == "uniform":
        keys = synth.uniform_range(21 + bits, n, 0, 2 ** bits - 1).astype(np.int32)
    else:
        keys = np.arange(n, dtype=np.int64) % (2 ** bits)
        rng = np.random.default_rng(bits)
        i = rng.integers(0, n, n // 100)
        j = rng.integers(0, n, n // 100)
        keys[i], keys[j] = keys[j], keys[i]
        keys = keys.astype(np.int32)
    check_pipeline(keys)


@pytest.fixture
def masked_rank():
    """Run a test with the masked (order-agnostic) onesweep ranking, then restore."""
    prev = ahs.ahs_rank_mode()
    ahs.ahs_rank_mode(ahs.RANK_MASKED)
    yield
    ahs.ahs_rank_mode(prev)


def test_lane_order_selftest_selects_ordered_ranking():
    # B200 serves same-address lanes of one shared atomic in lane order
    # (tools/atomorder.cu); the library then uses the one-atomic ranking
    assert ahs.ahs_lane_order_ok()
    assert ahs.ahs_rank_mode() == ahs.RANK_ORDERED


@pytest.mark.parametrize("family", ["full32", "zipf_wide", "neg16", "alt_extremes", "const"])
def test_masked_ranking_parity(family, masked_rank):
    assert ahs.ahs_rank_mode() == ahs.RANK_MASKED
    for n in (1, 33, 7679, 7681, 4609, 3 * 7680 + 77, 250_001, 3_000_017):
        keys = FAMILIES[family](n, 11)
        check_pipeline(keys)
        check_pipeline(keys, np.arange(n, dtype=np.uint32))


@pytest.fixture
def skip_off():
    prev = ahs.ahs_set_skip_trivial(-1)
    ahs.ahs_set_skip_trivial(0)
    yield
    ahs.ahs_set_skip_trivial(prev)


# NEXT-1: (keys, strategy, expected executed passes with skipping)
TRIVIAL_CASES = {
    # key - min = j * 2^18: digits 0 and 1 constant (cfg3's structure) -> RADIX, 2 of 4 passes
    "cfg3_like": (lambda n: synth.cfg3(n, seed=5), None, 2),
    # k = 2^16 under GENERAL (4 passes): digits 2 and 3 of key - min are 0
    "general_16bit": (lambda n: synth.uniform_range(6, n, 1000, 1000 + 65535), 2, 2),
    # k = 2^20: only digit 3 constant
    "general_20bit": (lambda n: synth.uniform_range(7, n, -(2 ** 19), 2 ** 19 - 1), 2, 3),
    # full 32-bit: nothing to skip
    "general_32bit": (lambda n: synth.uniform_range(8, n, -(2 ** 31), 2 ** 31 - 1), 2, 4),
    # digit placement (K5): key - min = j * 2^12, j < 2^16, feature shift 12: every key shares its
    # low 12 bits, so the digits sit at bits 12 and 20 (bit 28 on: constant) -> 2 passes, where
    # byte-aligned digits would need 3 (bits 8-15, 16-23, 24-27)
    "general_shift12": (lambda n: (synth.uniform_range(9, n, 0, 65535).astype(np.int64) * 4096 - 777)
                        .astype(np.int32), 2, 2),
    # RADIX over j * 2^20 + c, j < 1024 (10 varying bits at 20..29): digits at 20 and 28
    "radix_shift20": (lambda n: (synth.uniform_range(10, n, 0, 1023).astype(np.int64) * (1 << 20) - (1 << 29) + 5)
                      .astype(np.int32), None, 2),
}


@pytest.mark.parametrize("case", list(TRIVIAL_CASES))
def test_trivial_pass_skipping(case):
    gen, strategy, want = TRIVIAL_CASES[case]
    for n in (33, 7681, 250_001):
        keys = gen(n)
        if strategy is None:
            ok, ov = oracle.sort(keys, np.arange(n, dtype=np.uint32), oracle.QUICK)
        for vals in (None, np.arange(n, dtype=np.uint32)):
            info = {}
            f, s, r, ko, vo = run_gpu(keys, vals, strategy=strategy, info=info)
            ok, ov = oracle.sort(keys, vals, oracle.QUICK)
            assert np.array_equal(ko, ok)
            if vals is not None:
                assert np.array_equal(vo, ov)
            if n > 1000:  # tiny inputs may have more constant digits by chance
                assert info["executed"] == want, (case, n, info)
            # in place: the parity must be known on the host, no skipping
            info2 = {}
            f, s, r, ko, vo = run_gpu(keys, vals, strategy=strategy, inplace=True, info=info2)
            assert np.array_equal(ko, ok)
            assert info2["executed"] == info2["nominal"]


def test_trivial_pass_skipping_off(skip_off):
    keys = synth.cfg3(250_001, seed=5)
    for vals in (None, np.arange(keys.size, dtype=np.uint32)):
        info = {}
        f, s, r, ko, vo = run_gpu(keys, vals, info=info)
        ok, ov = oracle.sort(keys, vals, oracle.QUICK)
        assert np.array_equal(ko, ok)
        assert info["executed"] == info["nominal"] == 4


def test_pipeline_empty():
    for vals in (None, np.zeros(0, np.uint32)):
        f, s, r, ko, vo = run_gpu(np.zeros(0, np.int32), vals)
        assert f.n == 0 and ahs.RULE_NAMES[r] == "EMPTY" and ko.size == 0


@pytest.mark.parametrize("dtype", ["i32", "u32"])
@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_forced_strategies(dtype, strategy):
    rng = np.random.default_rng(strategy)
    for i, n in enumerate([1, 2, 17, 4097, 8193, 40_000]):
        for lo, hi in ((0, 999), (-5, 5), (-(2 ** 31), 2 ** 31 - 1), (3, 70_000), (0, 2 ** 24)):
            if dtype == "u32":
                lo, hi = lo + 2 ** 31, hi + 2 ** 31
            keys = synth.uniform_range(i * 7 + strategy, n, lo, hi, dtype=np.int64)
            keys = keys.astype(np.int32 if dtype == "i32" else np.uint32)
            vals = rng.integers(0, 2 ** 32, n, dtype=np.uint64).astype(np.uint32)
            check_forced(keys, None, strategy)
            check_forced(keys, vals, strategy)


@pytest.mark.parametrize("misalign", [1, 2, 3])
def test_misaligned_pointers(misalign):
    for n in (5, 4099, 20_003):
        for fam in ("u1000", "full32", "range3M"):
            keys = FAMILIES[fam](n, misalign)
            check_pipeline(keys, misalign=misalign)
            check_pipeline(keys, np.arange(n, dtype=np.uint32), misalign=misalign)


@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_in_place(strategy):
    # RADIX on k ~ 2^17 has 3 passes (odd): exercises the extra copy
    for lo, hi in ((0, 999), (0, 130_000), (-(2 ** 31), 2 ** 31 - 1), (0, 200)):
        keys = synth.uniform_range(5, 30_011, lo, hi)
        vals = np.arange(keys.size, dtype=np.uint32)
        check_forced(keys, None, strategy, inplace=True)
        check_forced(keys, vals, strategy, inplace=True)


def test_unsigned_full_range_and_extremes():
    keys = np.array([0, 2 ** 32 - 1, 2 ** 31, 2 ** 31 - 1, 1, 2 ** 32 - 1, 0] * 3001, dtype=np.uint32)
    check_pipeline(keys)
    check_pipeline(keys, np.arange(keys.size, dtype=np.uint32))


def test_side_stream():
    s = torch.cuda.Stream()
    keys = synth.cfg2(100_003)
    with torch.cuda.stream(s):
        f, st, r, ko, vo = run_gpu(keys, None, stream=s)
    assert np.array_equal(ko, np.sort(keys))


def test_thresholds_custom():
    keys = synth.uniform_range(3, 50_000, 0, 4999)
    th = ahs.ahs_thresholds_default(k_counting=8192)
    f, s, r, ko, vo = run_gpu(keys, np.arange(keys.size, dtype=np.uint32), th=th)
    assert ahs.STRATEGY_NAMES[s] == "COUNTING"  # 13 bits: counting via 2 radix passes on key - min
    ok, ov = oracle.sort(keys, np.arange(keys.size, dtype=np.uint32), oracle.COUNTING)
    assert np.array_equal(ko, ok) and np.array_equal(vo, ov)
    th = ahs.ahs_thresholds_default(k_counting=1 << 20, k_radix=1 << 24)
    keys = synth.uniform_range(4, 50_000, 0, 200_000)  # shift > 0: histogram bucketed
    f, s, r, ko, vo = run_gpu(keys, None, th=th)
    assert ahs.STRATEGY_NAMES[s] == "COUNTING" and f.shift > 0
    assert np.array_equal(ko, np.sort(keys))


def test_host_entry_point():
    keys = synth.cfg1(1 << 18)
    vals = np.arange(keys.size, dtype=np.uint32)
    ko, vo = np.empty_like(keys), np.empty_like(vals)
    scratch = torch.empty(ahs.ahs_host_scratch_bytes(keys.size, True), dtype=torch.uint8, device="cuda")
    f, s, r = ahs.ahs_sort_host(keys, vals, ko, vo, scratch)
    ref = oracle.ahs(keys, vals)
    check_features(f, ref["features"])
    assert np.array_equal(ko, ref["keys"]) and np.array_equal(vo, ref["vals"])


def test_host_entry_point_async_two_streams():
    """ahs_sort_host_async on alternating streams / scratch buffers (pinned host memory), as the
    bench's e2e leg runs it: every output equals the oracle's."""
    inputs = [synth.cfg2(300_007), synth.uniform_range(71, 300_007, -50, 50), synth.cfg3(300_007, seed=72),
              synth.cfg2(123_457)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    nmax = max(k.size for k in inputs)
    scratch = [torch.empty(ahs.ahs_host_scratch_bytes(nmax, True), dtype=torch.uint8, device="cuda")
               for _ in range(2)]
    outs = []
    for i, keys in enumerate(inputs):
        hk = torch.from_numpy(keys.view(np.int32)).pin_memory()
        hv = torch.arange(keys.size, dtype=torch.int32).pin_memory().view(torch.uint32)
        ko, vo = torch.empty_like(hk).pin_memory(), torch.empty_like(hv).pin_memory()
        if keys.dtype == np.uint32:
            hk, ko = hk.view(torch.uint32), ko.view(torch.uint32)
        if i >= 2:
            streams[i % 2].synchronize()
        ahs.ahs_sort_host(hk, hv, ko, vo, scratch[i % 2], stream=streams[i % 2], sync=False)
        outs.append((keys, hk, hv, ko, vo))
    torch.cuda.synchronize()
    for keys, hk, hv, ko, vo in outs:
        ref = oracle.ahs(keys, np.arange(keys.size, dtype=np.uint32))
        assert np.array_equal(ko.view(torch.int32).numpy().view(keys.dtype), ref["keys"])
        assert np.array_equal(vo.view(torch.int32).numpy().view(np.uint32), ref["vals"])


def test_launch_count_and_profile():
    keys = synth.cfg2(1 << 16)
    c0 = ahs.ahs_launch_count()
    ahs.ahs_profile_begin()
    run_gpu(keys, None)
    ahs.ahs_profile_end()
    prof = ahs.ahs_profile_read()
    assert ahs.ahs_launch_count() - c0 == 3 + 1 + 4
    assert prof["onesweep"]["launches"] == 4 and prof["onesweep"]["ms"] > 0


def test_repeat_deterministic():
    keys = synth.cfg3(300_000)
    a = run_gpu(keys, None)
    b = run_gpu(keys, None)
    assert a[0].entropy == b[0].entropy and np.array_equal(a[3], b[3])


def test_hist_overflow_guard_bits():
    # > 32768 copies of a few values in a 2^16-bucket histogram within one CTA: exercises the
    # 15-bit counters' overflow path (mode B)
    n = 3_000_000
    keys = np.full(n, 5, np.int32)
    keys[::2] = 2 ** 30
    keys[1::1000] = -(2 ** 31)
    keys[7::777] = 123456789
    check_pipeline(keys)


# ------------------------------------------------------ T5 full configs

FULL = ["cfg1", "cfg2", "cfg2kv", "cfg3", "cfg4a", "cfg4b", "cfg4c", "cfg4d"]


@pytest.mark.parametrize("cfg", FULL)
def test_config_full_size(cfg):
    keys, vals, _ = synth.make(cfg)
    f, s, r = check_pipeline(keys, vals)
    expect = {"cfg1": "COUNTING", "cfg2": "GENERAL", "cfg2kv": "GENERAL", "cfg3": "RADIX",
              "cfg4a": "GENERAL", "cfg4b": "GENERAL", "cfg4c": "COUNTING", "cfg4d": "COUNTING"}[cfg]
    assert ahs.STRATEGY_NAMES[s] == expect


@pytest.mark.parametrize("r", synth.CFG5_R)
def test_cfg5_full_size(r):
    """2^28 pairs: features vs the oracle; the sort by the properties that
    define the unique stable order (sorted, payload permutation consistent
    with the keys, ties in index order) plus oracle-computed samples."""
    keys, vals = synth.cfg5(r)
    n = keys.size
    f, s, rule, ko, vo = run_gpu(keys, vals)
    of, hist = oracle.features(keys, with_hist=True)
    check_features(f, of)
    s4, r4 = oracle.select(of)
    assert ahs.STRATEGY_NAMES[s] == oracle.gpu_strategy(s4)
    assert ahs.RULE_NAMES[rule] == oracle.RULE_NAMES[r4]
    assert np.all(ko[1:] >= ko[:-1])
    seen = np.zeros(n, dtype=bool)
    seen[vo] = True
    assert seen.all()
    assert np.array_equal(ko, keys[vo])
    tie = ko[1:] == ko[:-1]
    assert np.all(vo[1:][tie] > vo[:-1][tie])
    if of.shift == 0:
        # sampled slots: out[i] = min + the bin holding rank i (oracle histogram)
        cum = np.cumsum(hist.astype(np.int64))
        idx = synth.uniform_below(synth.stream(99, 4096), n).astype(np.int64)
        b = np.searchsorted(cum, idx, side="right")
        assert np.array_equal(ko[idx].astype(np.int64), b + of.min)


# ------------------------------------------------------ NEXT-2: H over distinct values

ENT_CASES = {
    "u1000": lambda n: synth.uniform_range(31, n, 0, 999),
    "full32": lambda n: synth.uniform_range(32, n, -(2 ** 31), 2 ** 31 - 1),
    "zipf_wide": lambda n: synth.cfg3(n, seed=33),
    "two_values": lambda n: synth.uniform_range(34, n, 5, 6),
    "const": lambda n: synth.cfg4c(n),
    # one long run in the middle: spans many chunks of the cooperative grid
    "long_run": lambda n: np.concatenate([np.arange(n // 4, dtype=np.int32),
                                          np.full(n - n // 2, 7 * n, np.int32),
                                          np.arange(n // 2 - n // 4, dtype=np.int32) + 8 * n]),
}


@pytest.mark.parametrize("case", list(ENT_CASES))
def test_entropy_sorted_matches_oracle(case):
    """ahs_entropy_sorted vs the oracle's H_exact (run lengths of the sorted keys, Kahan), 1e-9."""
    for n in (1, 2, 17, 4095, 4097, 65537, 1_000_003, 5_000_011):
        keys = ENT_CASES[case](n)
        ok = np.sort(keys, kind="stable")  # any order with equal keys contiguous
        want = oracle.h_exact_sorted(ok)
        ws = ahs.Workspace(n, False)
        got = ahs.ahs_entropy_sorted(to_dev(ok), ws)
        assert abs(got - want) <= H_TOL, (case, n, got, want)
        # misaligned start (scalar load path)
        got2 = ahs.ahs_entropy_sorted(to_dev(ok, misalign=1), ws)
        assert abs(got2 - want) <= H_TOL, (case, n, got2, want)


def test_entropy_sorted_on_pipeline_output_and_paper_branch():
    """NEXT-2 on ahs_sort's output: H_exact; the paper-literal FSM (RANGE norm with H_exact)
    picks the same branch as reading B here."""
    for cfg in ("cfg1", "cfg2"):
        keys, vals, _ = synth.make(cfg)
        dk = to_dev(keys)
        ws = ahs.Workspace(keys.size, False)
        f = ahs.ahs_features(dk, ws)
        s, r = ahs.ahs_select(f)
        ko = torch.empty_like(dk)
        ahs.ahs_sort(dk, None, ko, None, s, f, ws)
        hx = ahs.ahs_entropy_sorted(ko, ws)
        assert abs(hx - oracle.h_exact_sorted(np.sort(keys))) <= H_TOL
        fp = ahs.Features.from_buffer_copy(f)
        fp.entropy = hx
        sp, _ = ahs.ahs_select(fp, ahs.ahs_thresholds_default(entropy_norm=1))
        assert sp == s, cfg


def test_entropy_sorted_empty():
    ws = ahs.Workspace(1, False)
    assert ahs.ahs_entropy_sorted(torch.empty(0, dtype=torch.int32, device="cuda"), ws) == 0.0


def test_maximum_n():
    """n = AHS_MAX_N = 2^30 - 1 (the 30-bit look-back counts), GENERAL pairs with values = input index:
    the oracle cannot sort 2^30 keys in test time, so properties that hold at any size: the output is
    non-decreasing; it is a permutation of the input (the values are a permutation of the indices and
    gather the output; sums of keys and squares agree); equal keys keep their input order; sampled
    positions hold the order statistic (counted on the host)."""
    n = (1 << 30) - 1
    g = torch.Generator(device="cuda").manual_seed(2506)
    dk = torch.randint(-(2 ** 31), 2 ** 31, (n,), dtype=torch.int64, device="cuda", generator=g).to(torch.int32)
    ws = ahs.Workspace(n, True)
    f = ahs.ahs_features(dk, ws)
    s, r = ahs.ahs_select(f)
    assert ahs.STRATEGY_NAMES[s] == "GENERAL"
    dv = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32)
    ko, vo = torch.empty_like(dk), torch.empty_like(dv)
    ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
    torch.cuda.synchronize()
    k64, o64 = dk.to(torch.int64), ko.to(torch.int64)
    assert bool((ko[1:] >= ko[:-1]).all())
    assert int(k64.sum()) == int(o64.sum()) and int((k64 * k64).sum()) == int((o64 * o64).sum())
    # values: the original index of each output key; every index exactly once, and gathering the
    # input by them reproduces the output (so the output is a permutation of the input)
    vi64 = vo.view(torch.int32).to(torch.int64)
    assert bool((torch.bincount(vi64, minlength=n) == 1).all())
    assert bool((dk[vi64] == ko).all())
    # stability: equal neighbours keep their input order
    same = ko[1:] == ko[:-1]
    vi = vo.view(torch.int32)
    assert bool((vi[1:][same] > vi[:-1][same]).all())
    hk = dk.cpu().numpy()
    for pos in (0, n // 3, n - 1):
        x = int(ko[pos])
        below, upto = int((hk < x).sum()), int((hk <= x).sum())
        assert below <= pos < upto
    assert f.n == n and f.min == int(dk.min()) and f.max == int(dk.max())


def test_concurrent_host_threads():
    """Three host threads, each with its own stream and workspace, sort different inputs at once
    (the library's per-thread state: the mapped features buffer; K6 grids of concurrent sorts share
    SMs): every result equals the oracle's."""
    import threading

    cases = [synth.cfg2(400_009), synth.uniform_range(91, 400_009, -600, 600), synth.cfg3(400_009, seed=92),
             synth.cfg4d(300_007), synth.cfg2(123_457), synth.uniform_range(93, 250_001, 0, 2 ** 20)]
    results, errors = {}, []

    def worker(t):
        try:
            stream = torch.cuda.Stream()
            for i in range(t, len(cases), 3):
                keys = cases[i]
                vals = np.arange(keys.size, dtype=np.uint32)
                with torch.cuda.stream(stream):
                    dk, dv = to_dev(keys), to_dev(vals)
                    ws = ahs.Workspace(keys.size, True)
                    f = ahs.ahs_features(dk, ws, stream)
                    s, r = ahs.ahs_select(f)
                    ko, vo = torch.empty_like(dk), torch.empty_like(dv)
                    ahs.ahs_sort(dk, dv, ko, vo, s, f, ws, stream)
                stream.synchronize()
                results[i] = (to_host(ko), to_host(vo))
        except Exception as e:  # reported below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(3)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    for i, keys in enumerate(cases):
        ref = oracle.ahs(keys, np.arange(keys.size, dtype=np.uint32))
        assert np.array_equal(results[i][0], ref["keys"]) and np.array_equal(results[i][1], ref["vals"]), i


# ------------------------------------------- bucket-local GENERAL plan (opt-in)

@pytest.fixture
def bucket_local():
    prev = ahs.ahs_set_bucket_local(-1)
    ahs.ahs_set_bucket_local(1)
    yield
    ahs.ahs_set_bucket_local(prev)


@pytest.mark.parametrize("family", ["full32", "range3M", "desc", "alt_extremes"])
def test_bucket_local_plan_parity(family, bucket_local):
    """Two passes over the feature-bin digits + the in-shared-memory bucket pass (K10): keys and
    values against the oracle, and the plan it reports (bucket-local exactly when the bins are
    coarser than single values and the largest bin fits the K10 capacity)."""
    for i, n in enumerate((5000, 65537, 250_001, 3_000_017)):
        keys = FAMILIES[family](n, 900 + i)
        vals = np.arange(n, dtype=np.uint32)
        for v in (None, vals):
            f, s, r = check_pipeline(keys, v)
            if ahs.STRATEGY_NAMES[s] != "GENERAL":
                continue
            dk = to_dev(keys)
            ws = ahs.Workspace(n, v is not None)
            f2 = ahs.ahs_features(dk, ws)
            ko = torch.empty_like(dk)
            dv = to_dev(v) if v is not None else None
            vo = torch.empty_like(dv) if dv is not None else None
            ahs.ahs_sort(dk, dv, ko, vo, s, f2, ws)
            passes, bl = ahs.ahs_sort_plan(ws)
            if f2.shift == 0:
                assert bl == 0
            if bl:
                assert 1 <= passes <= 2  # the two bin digits (a constant one is skipped)
                assert ahs.ahs_sort_executed_passes(ws) == passes + 1


@pytest.mark.parametrize("kv", [False, True])
def test_bucket_local_plan_large(kv, bucket_local):
    """2^27 keys over the full 32-bit range: bins of ~2048 keys, so the plan is bucket-local (two
    bin-digit passes + K10 with 4096-key capacity).  Checked by the properties that define the
    unique stable order plus oracle-computed samples, against the classic plan's output too."""
    n = 1 << 27
    keys = (synth.stream(71, n) >> np.uint64(32)).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32) if kv else None
    dk = to_dev(keys)
    dv = to_dev(vals) if kv else None
    ws = ahs.Workspace(n, kv)
    f = ahs.ahs_features(dk, ws)
    s, r = ahs.ahs_select(f)
    assert ahs.STRATEGY_NAMES[s] == "GENERAL" and f.shift == 16
    ko, vo = torch.empty_like(dk), (torch.empty_like(dv) if kv else None)
    ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
    assert ahs.ahs_sort_plan(ws) == (2, 1)
    k1 = to_host(ko)
    assert np.all(k1[1:] >= k1[:-1])
    assert np.array_equal(np.bincount(k1 >> np.uint32(16), minlength=65536),
                          np.bincount(keys >> np.uint32(16), minlength=65536))
    idx = synth.uniform_below(synth.stream(72, 4096), n).astype(np.int64)
    assert np.array_equal(k1[idx], np.sort(keys)[idx])
    if kv:
        v1 = to_host(vo)
        assert np.array_equal(k1, keys[v1])
        tie = k1[1:] == k1[:-1]
        assert np.all(v1[1:][tie] > v1[:-1][tie])
    # the classic plan gives the same bytes
    prev = ahs.ahs_set_bucket_local(0)
    try:
        ko2, vo2 = torch.empty_like(dk), (torch.empty_like(dv) if kv else None)
        ahs.ahs_sort(dk, dv, ko2, vo2, s, f, ws)
        assert ahs.ahs_sort_plan(ws)[1] == 0
        assert torch.equal(ko, ko2) and (not kv or torch.equal(vo, vo2))
    finally:
        ahs.ahs_set_bucket_local(prev)


def test_bucket_local_plan_falls_back_on_a_large_bin(bucket_local):
    """A bin far above the bucket pass's capacity (a tenth of 2^27 keys share one value): K5 picks
    the classic plan on the device, and the bucket pass launched after it returns at once."""
    n = 1 << 27
    x = synth.stream(73, n)
    keys = (x >> np.uint64(32)).astype(np.uint32)
    keys[(x & np.uint64(1023)) < np.uint64(102)] = np.uint32(0x9e3779b9)
    vals = np.arange(n, dtype=np.uint32)
    dk, dv = to_dev(keys), to_dev(vals)
    ws = ahs.Workspace(n, True)
    f = ahs.ahs_features(dk, ws)
    s, r = ahs.ahs_select(f)
    assert ahs.STRATEGY_NAMES[s] == "GENERAL" and f.shift == 16
    ko, vo = torch.empty_like(dk), torch.empty_like(dv)
    ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
    assert ahs.ahs_sort_plan(ws) == (4, 0)
    k1, v1 = to_host(ko), to_host(vo)
    assert np.all(k1[1:] >= k1[:-1])
    assert np.array_equal(k1, keys[v1])
    tie = k1[1:] == k1[:-1]
    assert np.all(v1[1:][tie] > v1[:-1][tie])
