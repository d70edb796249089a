"""Step time vs kernel time of the pipeline (development tool): how much of a step is host round trip.

    python tools/gapbench.py [cfg ...]     (AHS_PDL=0 etc. pass through)
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20677_b200 as ahs  # noqa: E402
import synth  # noqa: E402


def run(cfg, reps=30):
    keys, vals, _ = synth.make(cfg)
    if keys.itemsize == 8:
        dk = torch.from_numpy(keys.view(np.int64)).cuda()
        if keys.dtype == np.uint64:
            dk = dk.view(torch.uint64)
    else:
        dk = torch.from_numpy(keys.view(np.int32)).cuda()
        if keys.dtype == np.uint32:
            dk = dk.view(torch.uint32)
    dv = torch.from_numpy(vals.view(np.int32)).cuda().view(torch.uint32) if vals is not None else None
    ko = torch.empty_like(dk)
    vo = torch.empty_like(dv) if dv is not None else None
    ws = ahs.Workspace(keys.size, dv is not None, key_dtype=keys.dtype)
    st = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        f = ahs.ahs_features(dk, ws)
        s, r = ahs.ahs_select(f)
        ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
    torch.cuda.synchronize()
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    tf, ts, tt = [], [], []
    for _ in range(reps):
        flush.fill_(1)
        a.record(st)
        f = ahs.ahs_features(dk, ws)
        b.record(st)
        s, r = ahs.ahs_select(f)
        ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
        c.record(st)
        torch.cuda.synchronize()
        tf.append(a.elapsed_time(b))
        ts.append(b.elapsed_time(c))
        tt.append(a.elapsed_time(c))
    print(f"{cfg:10s} {ahs.STRATEGY_NAMES[s] if hasattr(ahs, 'STRATEGY_NAMES') else s}: "
          f"features {np.median(tf)*1e3:7.1f} us, sort {np.median(ts)*1e3:7.1f} us, "
          f"step {np.median(tt)*1e3:7.1f} us (min {np.min(tt)*1e3:7.1f}) pdl={os.environ.get('AHS_PDL', '1')}",
          flush=True)


for cfg in (sys.argv[1:] or ["cfg2"]):
    run(cfg)
