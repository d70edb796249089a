"""Bucket-local final pass probe (development tool): time ahs_sort_segments (K9) on arrays that are
already sorted by their top bits, as two LSD passes over the feature-bin digits would leave them.

    python tools/bucketbench.py
Cases: 2^26 int32 in 65536 buckets of 1024 (cfg4a-like: 10 low bits vary), 2^24 in 65536 of 256
(cfg2-like, 16 low bits vary), 2^28 pairs in 65536 buckets of ~4096 is above K9's 2048 cap.
"""
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20677_b200 as ahs  # noqa: E402
import synth  # noqa: E402


def case(name, n, low_bits, seg, kv=False, reps=10, cap=None):
    cap = cap or seg
    nseg = n // seg
    x = synth.stream(11, n)
    low = (x >> np.uint64(40)).astype(np.uint32) & np.uint32((1 << low_bits) - 1)
    bucket = (np.arange(n, dtype=np.uint64) // seg).astype(np.uint32)
    keys = ((bucket << np.uint32(low_bits)) | low).astype(np.uint32)
    dk = torch.from_numpy(keys.view(np.int32)).cuda().view(torch.uint32)
    dv = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32) if kv else None
    ko = torch.empty_like(dk)
    vo = torch.empty_like(dv) if kv else None
    off = torch.arange(0, n + 1, seg, dtype=torch.int32, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ahs.ahs_sort_segments(dk, dv, ko, vo, off, cap, bad)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ahs.ahs_sort_segments(dk, dv, ko, vo, off, cap, bad)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    h = ko.view(torch.int32).cpu().numpy().view(np.uint32)
    ok = bool(np.all(h[1:] >= h[:-1])) and int(bad.item()) == 0
    byts = n * (8 + (8 if kv else 0))
    print(f"{name}: n={n} segs={nseg}x{seg} cap={cap} low_bits={low_bits} kv={kv}: {ms * 1e3:.1f} us "
          f"{n / ms / 1e6:.1f} Gkeys/s {byts / ms / 1e6:.0f} GB/s sorted={ok}")


if __name__ == "__main__":
    case("r32-like pairs, 4096 cap 4608", 1 << 28, 16, 4096, kv=True, cap=4608)
    case("r32-like pairs, 4096 cap 5120", 1 << 28, 16, 4096, kv=True, cap=5120)
    case("r24-like pairs, 4096 cap 4608", 1 << 28, 8, 4096, kv=True, cap=4608)
    case("r32-like keys, 4096 cap 4608", 1 << 28, 16, 4096, kv=False, cap=4608)
