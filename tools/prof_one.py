"""One warm-up + one profiled pipeline run of a config (for ncu; development tool).

    python tools/prof_one.py cfg2
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20677_b200 as ahs  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
keys, vals, _ = synth.make(cfg)
dk = torch.from_numpy(keys.view(np.int32)).cuda()
if keys.dtype == np.uint32:
    dk = dk.view(torch.uint32)
dv = torch.from_numpy(vals.view(np.int32)).cuda().view(torch.uint32) if vals is not None else None
ko, vo = torch.empty_like(dk), (torch.empty_like(dv) if dv is not None else None)
ws = ahs.Workspace(keys.size, dv is not None)
for _ in range(2):
    f = ahs.ahs_features(dk, ws)
    s, r = ahs.ahs_select(f)
    ahs.ahs_sort(dk, dv, ko, vo, s, f, ws)
torch.cuda.synchronize()
print(cfg, "ok", ahs.STRATEGY_NAMES[s])
