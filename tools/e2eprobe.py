"""End-to-end (host buffers) throughput of bench.py's e2e loop against step count, plus pinned
copy bandwidth at the step's buffer size (development tool).

    python tools/e2eprobe.py [cfg] [steps ...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2506_20677_b200 as ahs  # noqa: E402
import synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg5_r32"
steps_list = [int(x) for x in sys.argv[2:]] or [10, 30]
keys, vals, _ = synth.make(cfg)
dev = torch.device("cuda", 0)
n = keys.size
nbytes = keys.nbytes + (vals.nbytes if vals is not None else 0)
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h2.copy_(d2, non_blocking=True))]:
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        fn()
    b.record()
    torch.cuda.synchronize()
    print(f"{name} {3 * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9:.1f} GB/s", flush=True)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
a.record()
for _ in range(3):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
b.record()
torch.cuda.synchronize()
print(f"both at once {3 * nbytes / (a.elapsed_time(b) * 1e-3) / 1e9:.1f} GB/s each way", flush=True)
del h, h2, d, d2
for st in steps_list:
    ms, bi, bo = bench.time_e2e(torch, ahs, keys, vals, st, 2, dev)
    print(f"{cfg} e2e steps={st}: {ms / st:.2f} ms/step, {n * st / (ms * 1e-3) / 1e9:.3f} Gkeys/s, "
          f"{bi * st / (ms * 1e-3) / 1e9:.1f} GB/s each way", flush=True)
