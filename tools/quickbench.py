"""Per-kernel device times for a few workloads (development tool, not the bench).

    python tools/quickbench.py [cfg ...]   (env AHS_RANK=match|ballot etc. pass through)
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20677_b200 as ahs  # noqa: E402
import synth  # noqa: E402


def run(cfg, reps=10):
    keys, vals, dt = synth.make(cfg)
    n = keys.size
    wide = keys.dtype.itemsize == 8
    dk = torch.from_numpy(keys.view(np.int64 if wide else np.int32)).cuda()
    if keys.dtype == np.uint32:
        dk = dk.view(torch.uint32)
    elif keys.dtype == np.uint64:
        dk = dk.view(torch.uint64)
    dv = torch.from_numpy(vals.view(np.int32)).cuda().view(torch.uint32) if vals is not None else None
    ko, vo = torch.empty_like(dk), (torch.empty_like(dv) if dv is not None else None)
    ws = ahs.Workspace(n, dv is not None, key_dtype=keys.dtype if wide else None)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        f = ahs.ahs_features(dk, ws)
        s, r = ahs.ahs_select(f)
        ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
    torch.cuda.synchronize()
    ahs.ahs_profile_begin()
    for _ in range(reps):
        flush.zero_()
        f = ahs.ahs_features(dk, ws)
        s, r = ahs.ahs_select(f)
        ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
    torch.cuda.synchronize()
    ahs.ahs_profile_end()
    prof = ahs.ahs_profile_read()
    out = {"cfg": cfg, "n": n, "strategy": ahs.STRATEGY_NAMES[s]}
    sort_ms = 0.0
    for k, v in prof.items():
        if v["launches"]:
            per = v["ms"] / v["launches"]
            out[k] = round(per * 1e3, 1)
            if not k.startswith("feat"):
                sort_ms += v["ms"] / reps
    passes = ahs.ahs_sort_passes(f, s, dv is not None)
    kvb = (2 * keys.dtype.itemsize) + (8 if dv is not None else 0)
    out["sort_us"] = round(sort_ms * 1e3, 1)
    out["sort_Gkeys"] = round(n / (sort_ms * 1e-3) / 1e9, 1)
    if passes:
        for k in ("onesweep", "onesweep_kv", "count_scatter_kv"):
            if k in out:
                out[k + "_GBps"] = round(kvb * n / (out[k] * 1e-6) / 1e9)
    # correctness spot check
    h = ko.view(torch.int64 if wide else torch.int32).cpu().numpy().view(keys.dtype)
    out["sorted_ok"] = bool(np.array_equal(h, np.sort(keys, kind="stable")))
    return out


if __name__ == "__main__":
    cfgs = sys.argv[1:] or ["cfg2", "cfg2kv", "cfg3", "cfg5_r32"]
    for c in cfgs:
        print(json.dumps(run(c)), flush=True)
