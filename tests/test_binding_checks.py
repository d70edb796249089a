"""The binding refuses output buffers the C ABI would overrun (host logic, CPU):
ahs_sort's keys_out / vals_out must match the inputs' numel and element width, and the host
entry point's arrays must be C-contiguous with 4-byte values."""
import numpy as np
import pytest
import torch

import paper_2506_20677_b200 as ahs
from paper_2506_20677_b200 import _lib


def t(n, dt=torch.int32):
    return torch.zeros(n, dtype=dt)


def test_outputs_accepted_when_they_match():
    _lib._check_outputs(t(8), None, t(8), None)
    _lib._check_outputs(t(8), t(8, torch.int64), t(8), t(8, torch.int64))
    _lib._check_outputs(t(8, torch.uint64), t(8), t(8, torch.uint64), t(8, torch.float32))


@pytest.mark.parametrize("ko,vi,vo", [
    (t(7), None, None),                          # short keys_out
    (t(8, torch.int64), None, None),             # wider keys_out
    (t(8, torch.uint32), None, None),            # other key dtype (same width)
    (t(8), t(8, torch.int64), t(8)),             # 8-byte values into a 4-byte vals_out
    (t(8), t(8), t(4)),                          # short vals_out
    (t(8), t(8), None),                          # vals_out missing
    (t(8), None, t(8)),                          # vals_out without vals_in
    (t(8), t(9), t(9)),                          # one value per key
])
def test_outputs_refused(ko, vi, vo):
    with pytest.raises(ValueError):
        _lib._check_outputs(t(8), vi, ko, vo)


def test_host_entry_refuses_bad_host_arrays():
    k = np.zeros(16, dtype=np.int32)
    scratch = torch.zeros(1, dtype=torch.uint8)
    with pytest.raises(ValueError):  # 8-byte host values
        ahs.ahs_sort_host(k, np.zeros(16, dtype=np.int64), np.zeros(16, np.int32), np.zeros(16, np.int64), scratch)
    with pytest.raises(ValueError):  # non-contiguous keys
        ahs.ahs_sort_host(np.zeros(32, np.int32)[::2], None, np.zeros(16, np.int32), None, scratch)
    with pytest.raises(ValueError):  # short output
        ahs.ahs_sort_host(k, None, np.zeros(15, np.int32), None, scratch)
