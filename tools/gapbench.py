"""Step time vs kernel time of the pipeline (development tool): how much of a step is host round trip."""
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
ko = torch.empty_like(dk)
ws = ahs.Workspace(keys.size, False)
st = torch.cuda.current_stream()
for _ in range(3):
    f = ahs.ahs_features(dk, ws)
    s, r = ahs.ahs_select(f)
    ahs.ahs_sort(dk, None, ko, None, s, f, ws)
torch.cuda.synchronize()
a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
tf, ts = [], []
ahs.ahs_profile_begin()
for _ in range(20):
    a.record(st)
    f = ahs.ahs_features(dk, ws)
    b.record(st)
    s, r = ahs.ahs_select(f)
    ahs.ahs_sort(dk, None, ko, None, s, f, ws)
    c.record(st)
    torch.cuda.synchronize()
    tf.append(a.elapsed_time(b))
    ts.append(b.elapsed_time(c))
ahs.ahs_profile_end()
prof = ahs.ahs_profile_read()
kf = sum(v["ms"] for k, v in prof.items() if k.startswith("feat")) / 20
ks = sum(v["ms"] for k, v in prof.items() if not k.startswith("feat")) / 20
tf2, ts2 = [], []
for _ in range(20):
    a.record(st)
    f = ahs.ahs_features(dk, ws)
    b.record(st)
    s, r = ahs.ahs_select(f)
    ahs.ahs_sort(dk, None, ko, None, s, f, ws)
    c.record(st)
    torch.cuda.synchronize()
    tf2.append(a.elapsed_time(b))
    ts2.append(b.elapsed_time(c))
print(f"{cfg} (no per-kernel events): features step {np.median(tf2)*1e3:.1f} us, sort step {np.median(ts2)*1e3:.1f} us")
print(f"{cfg}: features step {np.median(tf)*1e3:.1f} us (kernels {kf*1e3:.1f}), "
      f"sort step {np.median(ts)*1e3:.1f} us (kernels {ks*1e3:.1f})")
