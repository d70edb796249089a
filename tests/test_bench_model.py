"""bench.py's byte models (host logic, CPU): the roofline's algorithmic bytes and
BASELINE.json's contract bytes (the per-config table: 36n / 72n / 8n / 16n ...),
pinned to the table's values so a changed model fails here, not silently in a bench line."""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

N = 1 << 20
COUNTING, RADIX, GENERAL = 0, 1, 2


@pytest.mark.parametrize("strategy,passes,kv,kb,per_key", [
    (GENERAL, 4, False, 4, 36),  # cfg2 / cfg4a / cfg4b keys
    (RADIX, 4, False, 4, 36),    # cfg3 (nominal 4 passes, 2 executed)
    (GENERAL, 4, True, 4, 72),   # cfg2kv, cfg5 r >= 16
    (COUNTING, 0, False, 4, 8),  # cfg1, cfg4d: a read and a write of the keys
    (COUNTING, 1, True, 4, 16),  # cfg5 r = 8: one stable scatter pass of the pairs
    (GENERAL, 8, False, 8, 136),  # cfg6: 64-bit keys, (2 x 8 + 1) x 8
])
def test_contract_bytes_match_the_survey_table(strategy, passes, kv, kb, per_key):
    assert bench.contract_bytes(strategy, passes, N, kv, kb) == per_key * N


@pytest.mark.parametrize("strategy,passes,kv,kb,shift,per_key", [
    (GENERAL, 4, False, 4, 16, 32),   # 4 executed passes x read + write of 4-byte keys; K5 reads no keys
    (RADIX, 2, False, 4, 16, 16),     # cfg3: 2 of 4 passes executed (NEXT-1)
    (GENERAL, 4, True, 4, 16, 64),    # pairs: + read + write of 4-byte values per pass
    (COUNTING, 0, False, 4, 0, 4),    # keys-only COUNTING writes the fill (the features read the keys)
    (COUNTING, 1, True, 4, 0, 16),    # pairs COUNTING: one scatter pass
    (GENERAL, 8, False, 8, 32, 136),  # 64-bit keys, k-mers: K5b reads the keys once (8n) + 8 x 16n
    (GENERAL, 8, False, 8, 16, 128),  # 64-bit keys whose feature buckets are <= 16 bits: no K5b read
])
def test_sort_bytes_model(strategy, passes, kv, kb, shift, per_key):
    assert bench.sort_bytes(strategy, passes, N, kv, shift, kb) == per_key * N


def test_constant_input_moves_nothing():
    # cfg4c (all keys equal): CONSTANT shortcut, no pass executes and nothing is written
    assert bench.sort_bytes(RADIX, 0, N, False) == 0
