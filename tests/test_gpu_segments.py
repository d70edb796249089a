"""NEXT-4: batched segment sort (ahs_sort_segments) against the CPU oracle, per segment:
Listing 1's insertion sort (oracle.INSERTION) for segments up to 32
keys, the oracle's stable QuickSort for the CTA-per-segment path; keys and values bit-exact
(the unique stable order).  Covers all four key types, empty and one-key segments, offsets
that do not start at 0 or cover the array (keys outside every segment untouched), in-place
calls, and segments longer than the declared maximum (counted, left as they were).
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2506_20677_b200 as ahs  # noqa: E402

DT = {"i32": np.int32, "u32": np.uint32, "i64": np.int64, "u64": np.uint64}


def to_dev(a: np.ndarray):
    if a.dtype.itemsize == 8:
        t = torch.from_numpy(a.view(np.int64).copy()).cuda()
        return t.view(torch.uint64) if a.dtype == np.uint64 else t
    t = torch.from_numpy(a.view(np.int32).copy()).cuda()
    return t.view(torch.uint32) if a.dtype == np.uint32 else t


def to_host(t, dtype):
    w = torch.int64 if t.element_size() == 8 else torch.int32
    return t.view(w).cpu().numpy().view(dtype)


def make_keys(dt, n, seed, small_range=False):
    if small_range:  # many equal keys: stability matters
        v = synth.uniform_range64(seed, n, -4, 4) if dt in ("i32", "i64") else synth.uniform_range64(seed, n, 0, 7,
                                                                                                     np.uint64)
        return v.astype(DT[dt])
    x = synth.stream(seed, n)
    return {"i32": lambda: (x >> np.uint64(32)).astype(np.uint32).view(np.int32),
            "u32": lambda: (x >> np.uint64(32)).astype(np.uint32),
            "i64": lambda: x.view(np.int64), "u64": lambda: x}[dt]()


def make_offsets(n_segs, max_len, seed, start=0):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, max_len + 1, n_segs)
    off = np.zeros(n_segs + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    return (off + start).astype(np.uint32)


def expected(keys, vals, off, max_len):
    ok, ov = keys.copy(), (vals.copy() if vals is not None else None)
    algo = oracle.INSERTION if max_len <= 32 else oracle.QUICK
    for s in range(off.size - 1):
        a, b = int(off[s]), int(off[s + 1])
        if b - a < 1:
            continue
        k2, v2 = oracle.sort(keys[a:b], vals[a:b] if vals is not None else None, algo)
        ok[a:b] = k2
        if vals is not None:
            ov[a:b] = v2
    return ok, ov


def run(keys, vals, off, max_len, inplace=False):
    dk, doff = to_dev(keys), torch.from_numpy(off.view(np.int32).copy()).cuda()
    dv = to_dev(vals) if vals is not None else None
    if inplace:
        ko, vo = dk, dv
    else:
        ko = to_dev(np.zeros_like(keys))
        vo = to_dev(np.zeros_like(vals)) if vals is not None else None
        # keys outside every segment must be left alone: pre-fill the output with the input
        ko.copy_(dk)
        if vo is not None:
            vo.copy_(dv)
    bad = ahs.ahs_sort_segments(dk, dv, ko, vo, doff, max_len)
    torch.cuda.synchronize()
    return to_host(ko, keys.dtype), (to_host(vo, np.uint32) if vo is not None else None), int(bad.item())


@pytest.mark.parametrize("dt", list(DT))
@pytest.mark.parametrize("max_len", [1, 2, 20, 32])
def test_small_segments(dt, max_len):
    nseg = 3000
    off = make_offsets(nseg, max_len, 7 + max_len)
    n = int(off[-1])
    for small_range in (False, True):
        keys = make_keys(dt, n, 11 + max_len, small_range)
        vals = np.arange(n, dtype=np.uint32)
        for v in (None, vals):
            ko, vo, bad = run(keys, v, off, max_len)
            ek, ev = expected(keys, v, off, max_len)
            assert bad == 0
            assert np.array_equal(ko, ek), (dt, max_len, small_range)
            if v is not None:
                assert np.array_equal(vo, ev)


@pytest.fixture(params=["ordered", "masked"])
def rank(request):
    prev = ahs.ahs_rank_mode()
    if request.param == "masked":
        ahs.ahs_rank_mode(ahs.RANK_MASKED)
    yield request.param
    ahs.ahs_rank_mode(prev)


@pytest.mark.parametrize("dt", list(DT))
@pytest.mark.parametrize("max_len", [33, 100, 512, 1000, 1536, 2048, 4096, 8192])
def test_medium_segments(dt, max_len, rank):
    nseg = 300 if max_len <= 100 else 40
    off = make_offsets(nseg, max_len, 17 + max_len)
    n = int(off[-1])
    keys = make_keys(dt, n, 19 + max_len, small_range=max_len == 1000)
    vals = np.arange(n, dtype=np.uint32)
    for v in (None, vals):
        ko, vo, bad = run(keys, v, off, max_len)
        ek, ev = expected(keys, v, off, max_len)
        assert bad == 0
        assert np.array_equal(ko, ek), (dt, max_len)
        if v is not None:
            assert np.array_equal(vo, ev)


@pytest.mark.parametrize("pattern", ["byte2", "bytes0_7", "top_bit", "all_equal", "two_values"])
@pytest.mark.parametrize("max_len", [256, 1536, 2048, 8192])
def test_medium_digit_patterns(pattern, max_len, rank):
    """keys that differ only in some bytes: the radix path skips the shared digits"""
    nseg = 60
    off = make_offsets(nseg, max_len, 31 + max_len)
    n = int(off[-1])
    x = synth.stream(37, n)
    base = np.uint64(0x0123456789ABCDEF)
    k = {"byte2": base ^ ((x & np.uint64(0xff)) << np.uint64(16)),
         "bytes0_7": base ^ (x & np.uint64(0xff)) ^ ((x >> np.uint64(8)) << np.uint64(56)),
         "top_bit": base ^ ((x & np.uint64(1)) << np.uint64(63)),
         "all_equal": np.full(n, base, dtype=np.uint64),
         "two_values": base ^ ((x & np.uint64(1)) * np.uint64(0x0000010000000100))}[pattern]
    vals = np.arange(n, dtype=np.uint32)
    for dt in ("u64", "i64", "u32", "i32"):
        keys = k.view(np.int64).astype(DT[dt]) if dt == "i64" else (
            k.astype(DT[dt]) if dt == "u64" else (k & np.uint64(0xffffffff) if pattern != "bytes0_7" else
                                                   (k & np.uint64(0xff)) | ((k >> np.uint64(32)) & np.uint64(0xff000000))
                                                   ).astype(np.uint32).view(DT[dt]))
        ko, vo, bad = run(keys, vals, off, max_len)
        ek, ev = expected(keys, vals, off, max_len)
        assert bad == 0
        assert np.array_equal(ko, ek) and np.array_equal(vo, ev), (pattern, dt)


@pytest.mark.parametrize("max_len", [20, 500])
def test_partial_cover_and_in_place(max_len):
    """offsets start at 5 and stop short of n: the keys outside stay; in place works."""
    nseg = 700
    off = make_offsets(nseg, max_len, 23, start=5)
    n = int(off[-1]) + 9
    keys = make_keys("i32", n, 29)
    vals = np.arange(n, dtype=np.uint32)
    for inplace in (False, True):
        ko, vo, bad = run(keys, vals, off, max_len, inplace=inplace)
        ek, ev = expected(keys, vals, off, max_len)
        assert bad == 0 and np.array_equal(ko, ek) and np.array_equal(vo, ev)
        assert np.array_equal(ko[:5], keys[:5]) and np.array_equal(ko[-9:], keys[-9:])


def test_segments_longer_than_declared_are_refused():
    keys = make_keys("u32", 5000, 31)
    # medium path: one segment of 300 with max_segment 200 -> refused, the others sorted
    off = np.array([0, 100, 400, 500], dtype=np.uint32)
    ko, vo, bad = run(keys, None, off, 200)
    assert bad == 1
    assert np.array_equal(ko[100:400], keys[100:400])
    assert np.array_equal(ko[:100], np.sort(keys[:100])) and np.array_equal(ko[400:500], np.sort(keys[400:500]))
    # small path: a 40-key segment with max_segment 32 -> refused
    off = np.array([0, 10, 50, 60], dtype=np.uint32)
    ko, vo, bad = run(keys, None, off, 32)
    assert bad >= 1
    assert np.array_equal(ko[10:50], keys[10:50])
    # a segment reaching past n
    off = np.array([0, 10, 6000], dtype=np.uint32)
    ko, vo, bad = run(keys, None, off, 2048)
    assert bad == 1 and np.array_equal(ko[:10], np.sort(keys[:10]))


@pytest.mark.parametrize("inplace", [False, True])
def test_small_path_one_long_segment_spares_its_neighbours(inplace):
    """One over-long segment pushes a K9s CTA's range past its staging buffer: only that
    segment is reported (and left unsorted); the CTA's 255 other segments are still sorted."""
    lens = np.full(300, 20, dtype=np.int64)
    lens[100] = 10000
    lens[7] = 0
    off = np.zeros(lens.size + 1, dtype=np.uint32)
    off[1:] = np.cumsum(lens)
    n = int(off[-1])
    keys = make_keys("i32", n, 43)
    vals = np.arange(n, dtype=np.uint32)
    ko, vo, bad = run(keys, vals, off, 32, inplace=inplace)
    assert bad == 1
    ek, ev = expected(keys, vals, off, 32)
    a, b = int(off[100]), int(off[101])
    ek[a:b], ev[a:b] = keys[a:b], vals[a:b]  # the refused segment stays as it was
    assert np.array_equal(ko, ek) and np.array_equal(vo, ev)


def test_no_segments_and_errors():
    keys = to_dev(make_keys("i32", 10, 37))
    off = torch.zeros(1, dtype=torch.int32, device="cuda")
    bad = ahs.ahs_sort_segments(keys, None, keys, None, off, 32)
    torch.cuda.synchronize()
    assert int(bad.item()) == 0
    with pytest.raises(ahs.AhsError):
        ahs.ahs_sort_segments(keys, None, keys, None, off, 8193)  # ERANGE: above the 8192-key limit


@pytest.mark.parametrize("lo,hi,nseg", [(1, 20, 1 << 20), (1000, 2048, 1 << 13)])
def test_bench_size_properties(lo, hi, nseg, rank):
    """The bench's segment workloads at full size (2^20 segments of 1..20 keys: Listing 1's path;
    2^13 of 1000..2048: the radix path), values = input index.  The per-segment oracle is too slow
    here, so properties that hold at any size: every segment is non-decreasing, the values are a
    permutation of the indices inside each segment that gathers the output from the input, and
    equal keys keep their input order (stability)."""
    rng = np.random.default_rng(7)
    lens = rng.integers(lo, hi + 1, nseg)
    off = np.zeros(nseg + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    n = int(off[-1])
    keys = (synth.stream(5, n) >> np.uint64(40)).astype(np.uint32).view(np.int32)  # 24-bit: duplicates
    vals = np.arange(n, dtype=np.uint32)
    ko, vo, bad = run(keys, vals, off.astype(np.uint32), hi)
    assert bad == 0
    seg = np.repeat(np.arange(nseg), lens)
    inner = seg[1:] == seg[:-1]  # adjacent pairs inside one segment
    assert (ko[1:][inner] >= ko[:-1][inner]).all()
    vi = vo.astype(np.int64)
    assert (seg[vi] == seg).all()  # values stay in their segment
    assert np.array_equal(np.sort(vi), np.arange(n))
    assert np.array_equal(keys[vi], ko)  # the values gather the output
    eq = inner & (ko[1:] == ko[:-1])
    assert (vi[1:][eq] > vi[:-1][eq]).all()  # stable


@pytest.mark.parametrize("dt", ["i32", "u32"])
@pytest.mark.parametrize("max_len", [1536, 2048, 4096, 8192])
@pytest.mark.parametrize("spread", ["low16", "low16_dups", "crosses16"])
def test_narrow_segments(dt, max_len, spread):
    """K10's narrow path: 32-bit keys with values whose segment keys agree above bit 16 sort as
    (low 16 bits, local index) slots with the values gathered at the end; a segment whose keys
    cross a 2^16 boundary (bit 16 differs) takes the 64-bit slot path.  Keys and values against
    the oracle's stable order per segment."""
    nseg = 24
    off = make_offsets(nseg, max_len, 41 + max_len)
    n = int(off[-1])
    x = synth.stream(43 + max_len, n)
    seg = np.repeat(np.arange(nseg), np.diff(off.astype(np.int64)))
    base = (synth.stream(47, nseg) & np.uint64(0x7fff0000)).astype(np.int64)[seg]
    if spread == "low16":
        k = base + (x & np.uint64(0xffff)).astype(np.int64)
    elif spread == "low16_dups":  # few distinct low bits: long runs of equal keys
        k = base + (x & np.uint64(0x0f0f)).astype(np.int64)
    else:  # keys around a 2^16 boundary of the segment's base
        k = base + 0x8000 + (x & np.uint64(0xffff)).astype(np.int64)
    keys = (k - 0x40000000).astype(np.int32) if dt == "i32" else k.astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    ko, vo, bad = run(keys, vals, off, max_len)
    ek, ev = expected(keys, vals, off, max_len)
    assert bad == 0
    assert np.array_equal(ko, ek) and np.array_equal(vo, ev)
