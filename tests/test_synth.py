"""T0: the seeded generators (synth/) are deterministic and match known answers."""
import json
import os

import numpy as np

import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix_known_answers():
    g = json.load(open(os.path.join(GOLD, "splitmix.json")))
    assert int(synth.mix64(np.uint64(0))) == int(g["mix64_of_0"], 16)
    x = synth.stream(1, 2)
    assert int(x[0]) == int(g["seed1_x0"], 16)
    assert int(x[1]) == int(g["seed1_x1"], 16)
    assert int(synth.stream(2, 1)[0]) == int(g["seed2_x0"], 16)
    assert synth.cfg1(8).tolist() == g["cfg1_first8"]


def test_stream_is_counter_based():
    a = synth.stream(7, 1000)
    b = synth.stream(7, 500, start=500)
    assert np.array_equal(a[500:], b)
    # chunked generation equals one-shot generation
    k1 = synth._chunked(9, 3000, lambda x: (x >> np.uint64(32)).astype(np.uint32), np.uint32, chunk=1024)
    k2 = (synth.stream(9, 3000) >> np.uint64(32)).astype(np.uint32)
    assert np.array_equal(k1, k2)


def test_uniform_below_range():
    x = synth.stream(3, 100000)
    for m in (1, 2, 16, 1000, 65536, (1 << 32) - 5, 1 << 32):
        u = synth.uniform_below(x, m)
        assert int(u.max()) < m


def test_config_shapes_small():
    for name in synth.CONFIGS:
        keys, vals, dt = synth.make(name, n=4096)
        assert keys.shape == (4096,)
        assert keys.dtype == {"i32": np.int32, "u32": np.uint32, "i64": np.int64, "u64": np.uint64}[dt]
        if vals is not None:
            assert np.array_equal(vals, np.arange(4096, dtype=np.uint32))
    assert (synth.cfg4c(100) == 42).all()
    d = synth.cfg4d(100000)
    assert d.min() == -8 and d.max() == 7
    b = synth.cfg4b(10)
    assert b.tolist() == list(range(9, -1, -1))
    a = synth.cfg4a(20000)
    assert sorted(a.tolist()) == list(range(20000))
    c3 = synth.cfg3(50000)
    assert ((c3 - synth.CFG3_BASE) % synth.CFG3_STEP == 0).all()
    assert c3.max() < synth.CFG3_BASE + synth.CFG3_STEP * 4096
    for r in (8, 16, 32):
        k, v = synth.cfg5(r, n=10000)
        assert int(k.max()) < (1 << r)


def test_zipf_cdf():
    cdf = synth.zipf_cdf()
    assert cdf.shape == (4096,) and cdf[-1] == 1.0
    assert np.all(np.diff(cdf) > 0)


def test_kmers_cover_4pow30():
    """cfg6 (NEXT-3): 30-mer codes are the top 60 bits of the SplitMix64 words."""
    x = synth.stream(6, 1000)
    k = synth.kmers(6, 1000)
    assert k.dtype == np.uint64 and int(k.max()) < 4 ** 30
    assert np.array_equal(k, x >> np.uint64(4))
