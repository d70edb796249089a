"""Throughput of ahs_sort_segments (NEXT-4) on a few segment-length mixes (development tool).

    python tools/segbench.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20677_b200 as ahs  # noqa: E402
import synth  # noqa: E402


def bench(name, nseg, lo, hi, max_len, kv, dtype=np.int32, reps=20):
    rng = np.random.default_rng(7)
    lens = rng.integers(lo, hi + 1, nseg)
    off = np.zeros(nseg + 1, dtype=np.int64)
    off[1:] = np.cumsum(lens)
    n = int(off[-1])
    x = synth.stream(5, n)
    keys = (x >> np.uint64(32)).astype(np.uint32).view(np.int32) if dtype == np.int32 else x
    dk = torch.from_numpy(keys.view(np.int64 if keys.itemsize == 8 else np.int32).copy()).cuda()
    if dtype == np.uint64:
        dk = dk.view(torch.uint64)
    dv = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32) if kv else None
    ko, vo = torch.empty_like(dk), (torch.empty_like(dv) if kv else None)
    doff = torch.from_numpy(off.astype(np.uint32).view(np.int32)).cuda()
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ahs.ahs_sort_segments(dk, dv, ko, vo, doff, max_len, bad)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        ahs.ahs_sort_segments(dk, dv, ko, vo, doff, max_len, bad)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = float(np.median(ts))
    kb = keys.itemsize
    byts = n * (2 * kb + (8 if kv else 0)) + 4 * (nseg + 1)
    out = {"case": name, "segments": nseg, "n": n, "kv": kv, "key_bytes": kb, "us": round(ms * 1e3, 1),
           "Gkeys_s": round(n / (ms * 1e-3) / 1e9, 2), "GBps": round(byts / (ms * 1e-3) / 1e9, 1),
           "frac_of_6548": round(byts / (ms * 1e-3) / 1e9 / 6548.5, 3), "bad": int(bad.item())}
    print(json.dumps(out), flush=True)


bench("insertion n<=20", 1 << 20, 1, 20, 20, False)
bench("insertion n<=20 kv", 1 << 20, 1, 20, 20, True)
bench("insertion n<=32 u64", 1 << 20, 1, 32, 32, False, np.uint64)
bench("radix 100-200", 1 << 16, 100, 200, 200, False)
bench("radix 1000-2048", 1 << 13, 1000, 2048, 2048, False)
bench("radix 1000-2048 kv", 1 << 13, 1000, 2048, 2048, True)
bench("radix 1000-2048 u64", 1 << 13, 1000, 2048, 2048, False, np.uint64)
bench("radix 33-256", 1 << 16, 33, 256, 256, False)
bench("radix 300-512", 1 << 15, 300, 512, 512, False)
bench("radix 600-1024 kv", 1 << 14, 600, 1024, 1024, True)
bench("radix 600-1024", 1 << 14, 600, 1024, 1024, False)
bench("radix 600-1024 u64", 1 << 14, 600, 1024, 1024, False, np.uint64)
bench("radix 300-512 kv", 1 << 15, 300, 512, 512, True)
