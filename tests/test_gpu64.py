"""NEXT-3: 64-bit keys (int64 / uint64, k in 128-bit arithmetic S:69)
through the C ABI against the CPU oracle (tests/test_oracle64.py pins it).

Bar as for 32-bit keys: features bit-exact (min, max, k saturated at 2^64 - 1
with its flag, bits, shift, nbins, descents, flags), |dH| <= 1e-9, strategy +
rule identical, keys and values bit-exact (the unique stable order).  Sizes
span several 64-bit K6 tiles (6144 keys, 3840 pairs ordered; 4608 / 2560
masked) with ragged tails; families reach every digit source of K5 for 64-bit
keys (feature histogram, K1 / K2 rows, and K5b's key read for digits 2-5).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2506_20677_b200 as ahs  # noqa: E402

H_TOL = 1e-9
I64_MIN, I64_MAX, U64_MAX = -(2 ** 63), 2 ** 63 - 1, 2 ** 64 - 1


@pytest.fixture(scope="module", autouse=True)
def cuda_ready():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    ahs.lib()


def to_dev(a: np.ndarray, misalign: int = 0):
    """Upload int64 / uint64 / uint32 arrays; misalign > 0 offsets the start by that many elements."""
    if a.dtype in (np.int64, np.uint64):
        t = torch.from_numpy(a.view(np.int64))
        base = torch.empty(a.size + misalign, dtype=torch.int64, device="cuda")
        base[misalign:].copy_(t)
        out = base[misalign:]
        return out.view(torch.uint64) if a.dtype == np.uint64 else out
    t = torch.from_numpy(a.view(np.int32))
    base = torch.empty(a.size + misalign, dtype=torch.int32, device="cuda")
    base[misalign:].copy_(t)
    return base.view(torch.uint32)[misalign:] if a.dtype == np.uint32 else base[misalign:]


def to_host(t, dtype) -> np.ndarray:
    if t.element_size() == 8:
        return t.view(torch.int64).cpu().numpy().view(dtype)
    return t.view(torch.int32).cpu().numpy().view(dtype)


def check_features(f, of):
    assert f.n == of.n
    if of.n == 0:
        return
    assert (f.key_min(), f.key_max(), f.k, f.bits, f.shift, f.nbins, f.descents) == \
        (of.key_min(), of.key_max(), of.k, of.bits, of.shift, of.nb, of.descents)
    assert abs(f.entropy - of.entropy) <= H_TOL
    assert f.flags == of.flags


def run_gpu(keys, vals=None, strategy=None, misalign=0, inplace=False, info=None):
    n = keys.size
    dk = to_dev(keys, misalign)
    dv = to_dev(vals, misalign) if vals is not None else None
    ws = ahs.Workspace(n, vals is not None, key_dtype=keys.dtype)
    f = ahs.ahs_features(dk, ws)
    s, r = ahs.ahs_select(f)
    if strategy is not None:
        s = strategy
    if inplace:
        ko, vo = dk, dv
    else:
        ko = to_dev(np.zeros_like(keys), misalign)
        vo = to_dev(np.zeros_like(vals), misalign) if vals is not None else None
    ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
    torch.cuda.synchronize()
    if info is not None:
        info["executed"] = ahs.ahs_sort_executed_passes(ws)
        info["nominal"] = ahs.ahs_sort_passes(f, s, vals is not None)
    return f, s, r, to_host(ko, keys.dtype), (to_host(vo, np.uint32) if vo is not None else None)


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


FAMILIES = {
    "full_u64": lambda n: synth.wide_u64(41, n),
    "full_i64": lambda n: synth.wide_i64(42, n),
    "kmers30": lambda n: synth.kmers(43, n),
    "i64_small": lambda n: synth.uniform_range64(44, n, -300, 299),            # COUNTING
    "u64_high_small": lambda n: synth.uniform_range64(45, n, 2 ** 63 - 100, 2 ** 63 + 99, np.uint64),
    "i64_cross40": lambda n: synth.uniform_range64(46, n, -(2 ** 31), 2 ** 31 - 1, np.int64) * np.int64(512),
    "u64_top_bits": lambda n: (synth.uniform_range64(47, n, 0, 49, np.uint64) << np.uint64(57)),
    "i64_extremes": lambda n: np.where(synth.uniform_range64(48, n, 0, 2, np.int64) == 0, I64_MIN,
                                       np.where(synth.uniform_range64(49, n, 0, 1, np.int64) == 0, I64_MAX, -1)
                                       ).astype(np.int64),
}
SIZES = [1, 2, 3, 17, 21, 1000, 2559, 2560, 2561, 3071, 3072, 3073, 3839, 3840, 3841, 4607, 4608, 4609, 5376, 6143, 6144,
         6145, 9217, 12289, 100_003]


@pytest.mark.parametrize("family", list(FAMILIES))
def test_pipeline_64_keys(family):
    for n in SIZES:
        check_pipeline(FAMILIES[family](n))


@pytest.mark.parametrize("family", list(FAMILIES))
def test_pipeline_64_pairs(family):
    for n in SIZES:
        keys = FAMILIES[family](n)
        check_pipeline(keys, np.arange(n, dtype=np.uint32))


@pytest.mark.parametrize("family", ["full_u64", "kmers30", "i64_cross40", "u64_top_bits"])
def test_many_tiles_per_cta_64(family):
    n = 3_000_017
    keys = FAMILIES[family](n)
    check_pipeline(keys)
    check_pipeline(keys, np.arange(n, dtype=np.uint32))


def test_k_saturated_full_range():
    keys = np.array([I64_MIN, I64_MAX, 0, -5, 7] * 2000, dtype=np.int64)
    f, s, r = check_pipeline(keys)
    assert f.k == U64_MAX and f.flags & ahs.FLAG_K_SATURATED and f.bits == 64 and f.shift == 48


@pytest.mark.parametrize("strategy", [0, 1, 2])
@pytest.mark.parametrize("dt", ["i64", "u64"])
def test_forced_strategies_64(strategy, dt):
    """Every strategy on inputs the FSM would not pick for it gives the unique stable order."""
    n = 50_001
    keys = synth.uniform_range64(50, n, -200, 800) if dt == "i64" else synth.kmers(51, n, 10)
    vals = np.arange(n, dtype=np.uint32)
    for v in (None, vals):
        f, s, r, ko, vo = run_gpu(keys, v, strategy=strategy)
        ok, ov = oracle.sort(keys, v, oracle.QUICK)
        assert np.array_equal(ko, ok)
        if v is not None:
            assert np.array_equal(vo, ov)


@pytest.mark.parametrize("strategy", [0, 1, 2])
def test_in_place_64(strategy):
    n = 40_000
    keys = synth.kmers(52, n, 12)
    vals = np.arange(n, dtype=np.uint32)
    for v in (None, vals):
        f, s, r, ko, vo = run_gpu(keys, v, strategy=strategy, inplace=True)
        ok, ov = oracle.sort(keys, v, oracle.QUICK)
        assert np.array_equal(ko, ok)
        if v is not None:
            assert np.array_equal(vo, ov)


def test_misaligned_64():
    """An 8-byte-aligned start that is not 16-byte aligned: the scalar load paths."""
    for fam in ("full_u64", "i64_small", "kmers30"):
        keys = FAMILIES[fam](30_001)
        check_pipeline(keys, misalign=1)
        check_pipeline(keys, np.arange(keys.size, dtype=np.uint32), misalign=1)


def test_trivial_pass_skipping_64():
    """Constant digits are skipped (NEXT-1): top-bits keys have one varying digit."""
    n = 200_003
    keys = FAMILIES["u64_top_bits"](n)  # v << 57, v < 50: bits 57..62 vary
    info = {}
    f, s, r, ko, vo = run_gpu(keys, info=info)
    assert np.array_equal(ko, np.sort(keys, kind="stable"))
    assert info["nominal"] == 8 and info["executed"] == 1
    keys = synth.kmers(53, n)  # k = 4^30: 60 bits, all 8 digits vary
    info = {}
    f, s, r, ko, vo = run_gpu(keys, info=info)
    assert np.array_equal(ko, np.sort(keys, kind="stable"))
    assert info["executed"] == 8


def test_host_entry_point_64():
    n = 20_011
    keys = synth.wide_i64(54, n)
    vals = np.arange(n, dtype=np.uint32)
    ko, vo = np.empty_like(keys), np.empty_like(vals)
    scratch = torch.empty(ahs.ahs_host_scratch_bytes(n, True, keys.dtype), dtype=torch.uint8, device="cuda")
    f, s, r = ahs.ahs_sort_host(keys, vals, ko, vo, scratch)
    ok, ov = oracle.sort(keys, vals, oracle.QUICK)
    assert np.array_equal(ko, ok) and np.array_equal(vo, ov)


@pytest.mark.parametrize("dt", ["u32", "i64", "u64"])
def test_dirty_workspace(dt):
    """The library may not rely on zeroed scratch: ws and tmp start as 0xff bytes (stale look-back
    statuses, tickets, plans), repeated sorts reuse them."""
    n = 2_000_003
    keys = {"u32": lambda: synth.uniform_range(60, n, 0, 2 ** 32 - 1, np.uint32),
            "i64": lambda: synth.wide_i64(61, n), "u64": lambda: synth.kmers(62, n)}[dt]()
    vals = np.arange(n, dtype=np.uint32)
    want_k, want_v = oracle.sort(keys, vals, oracle.QUICK)
    for kv in (False, True):
        ws = ahs.Workspace(n, kv, key_dtype=None if dt == "u32" else keys.dtype)
        for rep in range(3):
            ws.ws.fill_(255)
            ws.tmp.fill_(255)
            dk = to_dev(keys)
            dv = to_dev(vals) if kv else None
            f = ahs.ahs_features(dk, ws)
            s, r = ahs.ahs_select(f)
            ko = to_dev(np.zeros_like(keys))
            vo = to_dev(np.zeros_like(vals)) if kv else None
            ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
            torch.cuda.synchronize()
            assert np.array_equal(to_host(ko, keys.dtype), want_k), (dt, kv, rep)
            if kv:
                assert np.array_equal(to_host(vo, np.uint32), want_v), (dt, kv, rep)


@pytest.mark.parametrize("family", ["full_u64", "i64_small", "u64_top_bits", "i64_extremes", "kmers30"])
def test_entropy_sorted_64(family):
    """NEXT-2 on 64-bit keys: K8 over the sorted output vs the oracle's H_exact (1e-9)."""
    for n in (1, 2, 17, 4097, 100_003, 1_000_003):
        keys = FAMILIES[family](n)
        ok = np.sort(keys, kind="stable")
        want = oracle.h_exact_sorted(ok)
        ws = ahs.Workspace(n, False, key_dtype=keys.dtype)
        got = ahs.ahs_entropy_sorted(to_dev(ok), ws)
        assert abs(got - want) <= H_TOL, (family, n, got, want)
        got = ahs.ahs_entropy_sorted(to_dev(ok, misalign=1), ws)
        assert abs(got - want) <= H_TOL, (family, n, got, want)


@pytest.mark.parametrize("kdt", ["u32", "i32", "u64", "i64"])
def test_64bit_payloads(kdt):
    """NEXT-3 payloads: 8-byte values travel bit-exactly with their keys (ahs_sort_ex), every strategy."""
    fams = {"u32": lambda n: synth.cfg2(n), "i32": lambda n: synth.uniform_range(81, n, -200, 200),
            "u64": lambda n: synth.kmers(82, n), "i64": lambda n: synth.uniform_range64(83, n, -3, 3)}
    for n in (1, 17, 3071, 3457, 100_003, 1_500_007):
        keys = fams[kdt](n)
        vals = synth.stream(84, n)  # full 64-bit payloads
        ref_k, order = oracle.sort(keys, np.arange(n, dtype=np.uint32), oracle.QUICK)
        for strategy in (None, 0, 1, 2):
            dk = to_dev(keys)
            dv = torch.from_numpy(vals.view(np.int64)).cuda()
            ws = ahs.Workspace(n, True, key_dtype=keys.dtype, val_bytes=8)
            f = ahs.ahs_features(dk, ws)
            s, r = ahs.ahs_select(f)
            s = s if strategy is None else strategy
            ko, vo = to_dev(np.zeros_like(keys)), torch.empty_like(dv)
            ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
            torch.cuda.synchronize()
            assert np.array_equal(to_host(ko, keys.dtype), ref_k), (kdt, n, strategy)
            assert np.array_equal(vo.cpu().numpy().view(np.uint64), vals[order]), (kdt, n, strategy)


def test_empty_and_constant_64():
    """n = 0 (no launch, flags EMPTY | SORTED) and a constant 64-bit input under every strategy."""
    for dt in (np.int64, np.uint64):
        keys = np.zeros(0, dtype=dt)
        ws = ahs.Workspace(1, False, key_dtype=dt)
        dk = torch.zeros(0, dtype=torch.int64, device="cuda")
        f = ahs.ahs_features(dk.view(torch.uint64) if dt == np.uint64 else dk, ws)
        assert f.n == 0 and f.flags & 1
        keys = np.full(5000, I64_MIN if dt == np.int64 else 2 ** 63 + 5, dtype=dt)
        vals = np.arange(5000, dtype=np.uint32)
        for strategy in (None, 0, 1, 2):
            f, s, r, ko, vo = run_gpu(keys, vals, strategy=strategy)
            assert f.k == 1 and np.array_equal(ko, keys) and np.array_equal(vo, vals)


@pytest.mark.parametrize("cfg", ["cfg6", "cfg6kv"])
def test_config_full_size_64(cfg):
    """NEXT-3 at BASELINE size: 2^26 uint64 30-mer codes (k = 4^30), keys and
    (cfg6kv) values = input index, in the bench's launch configuration: features, strategy, rule,
    keys and values bit-exact against the oracle."""
    keys, vals, _ = synth.make(cfg)
    check_pipeline(keys, vals)


@pytest.mark.parametrize("cfg", ["cfg3", "cfg4d", "cfg6"])
def test_entropy_sorted_full_size(cfg):
    """NEXT-2 (K8) at BASELINE sizes (2^26 keys: Zipf-like cfg3, 16 long runs in cfg4d, 64-bit cfg6)
    against the oracle's H_exact over the same sorted array (1e-9)."""
    keys, _, _ = synth.make(cfg)
    ok = np.sort(keys, kind="stable")  # K8's input: equal keys contiguous (any sort)
    want = oracle.h_exact_sorted(ok)
    ws = ahs.Workspace(keys.size, False, key_dtype=keys.dtype)
    got = ahs.ahs_entropy_sorted(to_dev(ok), ws)
    assert abs(got - want) <= H_TOL, (cfg, got, want)
