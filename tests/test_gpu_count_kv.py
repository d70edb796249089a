"""Key-value COUNTING with 256 < k <= 1024 (§III.F Listing 2; k_counting =
1024, Table II) on a B200, in both modes of the library: two 8-bit radix passes over
key - min (the default) and one stable 10-bit scatter (ahs_set_count_kv_single(1)).
Bar: keys and values bit-exact against the oracle's Listing-2 counting sort (the unique stable
order), features and strategy as the oracle's; the single mode must report and run one pass."""
import numpy as np
import pytest

import oracle
import synth
from test_gpu_parity import check_pipeline, run_gpu, check_features

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
import paper_2506_20677_b200 as ahs  # noqa: E402


@pytest.fixture(params=[0, 1], ids=["two_passes", "single_pass"])
def kv_mode(request):
    prev = ahs.ahs_set_count_kv_single(-1)
    ahs.ahs_set_count_kv_single(request.param)
    yield request.param
    ahs.ahs_set_count_kv_single(prev)


# k = max - min + 1 in (256, 1024]: 9- and 10-bit digits, signed and unsigned, ragged sizes
# around the 4096-pair tile of the single pass and the 6400-pair tile of the radix passes
CASES = [(257, "i32"), (300, "u32"), (1000, "i32"), (1024, "u32"), (513, "i32")]
SIZES = [1, 2, 33, 4095, 4096, 4097, 6399, 6400, 6401, 3 * 4096 + 17, 250_001, 1_000_003]


@pytest.mark.parametrize("k,dt", CASES)
def test_count_kv_parity(k, dt, kv_mode):
    for i, n in enumerate(SIZES):
        lo = -(k // 2) if dt == "i32" else 7
        keys = synth.uniform_range(400 + i, n, lo, lo + k - 1)
        keys = keys.astype(np.int32) if dt == "i32" else keys.astype(np.uint32)
        vals = np.arange(n, dtype=np.uint32)
        f, s, r = check_pipeline(keys, vals)
        if n > 20 and f.k > 256:  # n <= 20: the FSM's Insertion rule (GENERAL)
            info = {}
            run_gpu(keys, vals, info=info)
            assert ahs.STRATEGY_NAMES[s] == "COUNTING"
            assert info["nominal"] == (1 if kv_mode else 2)


def test_count_kv_full_size_k1000(kv_mode):
    """2^28 pairs, keys uniform in [0, 1000) (synth cfg7kv): against the oracle's counting sort."""
    keys, vals = synth.cfg7()
    f, s, r, ko, vo = run_gpu(keys, vals)
    of = oracle.features(keys)
    check_features(f, of)
    assert ahs.STRATEGY_NAMES[s] == "COUNTING" and f.k == 1000
    ok, ov = oracle.sort(keys, vals, oracle.COUNTING)  # Listing 2: stable, values travel with keys
    assert np.array_equal(ko, ok)
    assert np.array_equal(vo, ov)
