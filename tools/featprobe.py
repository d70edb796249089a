"""Runs ahs_features on cfg2's input a few times (ncu target for K1-K3; development tool)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20677_b200 as ahs  # noqa: E402
import synth  # noqa: E402

keys = torch.from_numpy(synth.cfg2().view("int32")).cuda()
ws = ahs.Workspace(keys.numel(), False, keys.device)
for _ in range(int(os.environ.get("REPS", "3"))):
    f = ahs.ahs_features(keys, ws)
torch.cuda.synchronize()
print(f)
