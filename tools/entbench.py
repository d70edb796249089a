"""K8 (ahs_entropy_sorted) kernel time on sorted outputs of a few configs (development tool)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20677_b200 as ahs  # noqa: E402
import synth  # noqa: E402

for cfg in sys.argv[1:] or ["cfg2", "cfg1", "cfg3"]:
    keys, _, _ = synth.make(cfg)
    ko = torch.from_numpy(np.sort(keys).view(np.int32)).cuda()
    ws = ahs.Workspace(keys.size, False)
    for _ in range(3):
        ahs.ahs_entropy_sorted(ko, ws)
    ahs.ahs_profile_begin()
    for _ in range(20):
        ahs.ahs_entropy_sorted(ko, ws)
    ahs.ahs_profile_end()
    p = ahs.ahs_profile_read()["entropy_sorted"]
    us = p["ms"] / p["launches"] * 1e3
    print(f"{cfg}: n={keys.size} K8 {us:.1f} us = {4 * keys.size / us / 1e3:.0f} GB/s", flush=True)
