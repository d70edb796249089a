"""Development probe for 64-bit sorts: which sizes / modes disagree with numpy."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_20677_b200 as ahs  # noqa: E402
import synth  # noqa: E402


def run(keys, kv, strategy=None):
    n = keys.size
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    dv = torch.arange(n, dtype=torch.int32, device="cuda").view(torch.uint32) if kv else None
    ws = ahs.Workspace(n, kv, key_dtype=keys.dtype)
    f = ahs.ahs_features(dk.view(torch.uint64) if keys.dtype == np.uint64 else dk, ws)
    s, r = ahs.ahs_select(f)
    if strategy is not None:
        s = strategy
    ko = torch.empty_like(dk)
    vo = torch.empty_like(dv) if kv else None
    kin = dk.view(torch.uint64) if keys.dtype == np.uint64 else dk
    kout = ko.view(torch.uint64) if keys.dtype == np.uint64 else ko
    ahs.ahs_sort(kin, dv, kout, vo, s, f, ws)
    torch.cuda.synchronize()
    got = ko.cpu().numpy().view(keys.dtype)
    want = np.sort(keys, kind="stable")
    bad = np.nonzero(got != want)[0]
    ex = ahs.ahs_sort_executed_passes(ws)
    return s, ex, bad.size, (bad[0] if bad.size else -1)


tag = os.environ.get("TAG", "")
for fam in sys.argv[1:] or ["kmers30"]:
    for n in (100_003, 500_003, 1_000_003, 2_000_003, 3_000_017):
        keys = {"kmers30": lambda: synth.kmers(43, n), "full_u64": lambda: synth.wide_u64(41, n),
                "kmers_top16": lambda: (synth.kmers(43, n) >> np.uint64(56)) << np.uint64(56)}[fam]()
        for kv in (False, True):
            s, ex, nbad, first = run(keys, kv)
            print(f"{tag} {fam} n={n} kv={kv} strategy={s} executed={ex} bad={nbad} first_bad={first}", flush=True)
