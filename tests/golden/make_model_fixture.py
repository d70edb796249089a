"""Writes tests/golden/ahs_model_fixture.json: an "ahs-model/1" tree ensemble (SPEC.md
classifier module) that agrees with the paper's FSM (§III.A; RANGE
normalisation H < 0.7 log2 k, Table II thresholds) on SPEC's 512-point grid:
n in 8 log-spaced values 10^3..10^6, k in 8 log-spaced integers 10..10^7, H = f log2 k for
8 f in 0.1..0.9.  The trained model of the paper is not available; this fixture is
FSM-consistent by construction (SPEC: "fixture is FSM-consistent by construction").

    python tests/golden/make_model_fixture.py
"""
import json
import math
import os

K_COUNTING, K_RADIX, N_INSERTION, COEFF = 1024, 1_000_000, 20, 0.7  # Table II


def grid():
    ns = [round(10 ** (3 + 3 * i / 7)) for i in range(8)]
    ks = [round(10 ** (1 + 6 * i / 7)) for i in range(8)]
    fs = [0.1 + 0.8 * i / 7 for i in range(8)]
    return [(n, k, f * math.log2(k)) for n in ns for k in ks for f in fs]


def build():
    leaf = lambda c: {"leaf": [1.0 if i == c else 0.0 for i in range(4)]}  # classes: ins, cnt, rad, quick
    nodes = [
        {"feature": 0, "threshold": N_INSERTION + 0.5, "left": 1, "right": 2},   # n <= 20 -> insertion
        leaf(0),
        {"feature": 1, "threshold": K_COUNTING + 0.5, "left": 3, "right": 4},    # k <= 1024 -> counting
        leaf(1),
        {"feature": 1, "threshold": K_RADIX + 0.5, "left": 5, "right": 6},       # k <= 10^6 -> quick
        leaf(3),
    ]
    # k > 10^6: one cell per grid k, split on H at 0.7 log2 k (the FSM's threshold there)
    big = sorted({k for _, k, _ in grid() if k > K_RADIX})

    def cells(lo, hi):  # subtree over big[lo:hi], returns its node index
        i = len(nodes)
        if hi - lo == 1:
            k = big[lo]
            nodes.append({"feature": 2, "threshold": COEFF * math.log2(k), "left": i + 1, "right": i + 2})
            nodes.append(leaf(2))
            nodes.append(leaf(3))
            return i
        mid = (lo + hi) // 2
        nodes.append(None)
        left = cells(lo, mid)
        right = cells(mid, hi)
        nodes[i] = {"feature": 1, "threshold": math.sqrt(big[mid - 1] * big[mid]), "left": left, "right": right}
        return i

    assert len(nodes) == 6
    cells(0, len(big))
    tree2 = [{"feature": 1, "threshold": K_COUNTING + 0.5, "left": 1, "right": 2},
             {"leaf": [0.0, 0.25, 0.0, 0.0]}, {"leaf": [0.0, 0.0, 0.0, 0.25]}]
    return {"version": "ahs-model/1", "classes": ["insertion", "counting", "radix", "quick"],
            "feature_names": ["n", "k", "H"], "base_scores": [0.01, 0.02, 0.03, 0.04],
            "trees": [{"nodes": nodes}, {"nodes": tree2}]}


if __name__ == "__main__":
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ahs_model_fixture.json")
    with open(out, "w") as fh:
        json.dump(build(), fh, indent=1)
    print(out)
