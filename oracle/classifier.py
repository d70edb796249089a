"""Plain-Python oracle of the strategy classifier (NEXT-4).

TEST INFRASTRUCTURE ONLY: imported by tests/ (and by the fixture script under
tests/golden/), never by the product.  Shares nothing with
paper_2506_20677_b200/csrc/classifier.hpp.

Follows SPEC.md's classifier module, which makes PAPER.md §III.H
(Listing 5: loadModel / predictStrategy over (n, k, H))
portable:
  load     the "ahs-model/1" JSON schema, validated eagerly: 4 classes naming
           insertion / counting / radix / quick once each, feature_names
           ["n", "k", "H"], 4 finite base scores, trees of nodes that are either
           {"feature", "threshold", "left", "right"} or {"leaf": [4 reals]};
           unknown fields rejected; no node reached twice from the root.
  predict  score_c = base_c + sum over trees of the reached leaf's c-th score,
           going left iff feature value < threshold; argmax, ties to the
           earlier class in `classes`.
"""
from __future__ import annotations

import json
import math

ALGOS = {"insertion": 0, "counting": 1, "radix": 2, "quick": 3}


class ModelError(ValueError):
    """Malformed JSON or a schema violation."""


class VersionError(ModelError):
    """A version other than ahs-model/1."""


def _no_dups(pairs):
    d = {}
    for k, v in pairs:
        if k in d:
            raise ModelError(f"duplicate key {k!r}")
        d[k] = v
    return d


def _reals(v, n, what):
    if not isinstance(v, list) or len(v) != n:
        raise ModelError(f"{what}: expected {n} reals")
    out = []
    for x in v:
        if isinstance(x, bool) or not isinstance(x, (int, float)) or not math.isfinite(float(x)):
            raise ModelError(f"{what}: expected finite reals")
        out.append(float(x))
    return out


def _index(v, hi, what):
    if isinstance(v, bool) or not isinstance(v, int) or not 0 <= v <= hi:
        raise ModelError(f"{what} out of range")
    return v


def load(data) -> dict:
    if isinstance(data, (bytes, bytearray)):
        data = data.decode("utf-8")
    try:
        m = json.loads(data, object_pairs_hook=_no_dups)
    except ModelError:
        raise
    except Exception as e:  # json.JSONDecodeError, empty input
        raise ModelError(f"parse error: {e}") from None
    if not isinstance(m, dict):
        raise ModelError("top level is not an object")
    if set(m) - {"version", "classes", "feature_names", "base_scores", "trees"}:
        raise ModelError("unknown top-level field")
    if m.get("version") != "ahs-model/1":
        if isinstance(m.get("version"), str):
            raise VersionError(f"unsupported version {m['version']!r}")
        raise ModelError("missing version")
    cls = m.get("classes")
    if not isinstance(cls, list) or sorted(cls, key=str) != sorted(ALGOS) or len(set(cls)) != 4:
        raise ModelError("classes must name insertion, counting, radix, quick once each")
    if m.get("feature_names") != ["n", "k", "H"]:
        raise ModelError('feature_names must be ["n","k","H"]')
    base = _reals(m.get("base_scores"), 4, "base_scores")
    trees = m.get("trees")
    if not isinstance(trees, list):
        raise ModelError("trees must be an array")
    out = []
    for t, tv in enumerate(trees):
        if not isinstance(tv, dict) or set(tv) != {"nodes"} or not isinstance(tv["nodes"], list) or not tv["nodes"]:
            raise ModelError(f"tree {t}: expected nodes")
        nodes = []
        for i, nv in enumerate(tv["nodes"]):
            w = f"tree {t} node {i}"
            if not isinstance(nv, dict):
                raise ModelError(f"{w}: not an object")
            if "leaf" in nv:
                if set(nv) != {"leaf"}:
                    raise ModelError(f"{w}: unknown field beside leaf")
                nodes.append(("leaf", _reals(nv["leaf"], 4, w)))
                continue
            if set(nv) - {"feature", "threshold", "left", "right"} or len(nv) != 4:
                raise ModelError(f"{w}: expected feature, threshold, left, right")
            f = _index(nv["feature"], 2, f"{w}: feature index")
            th = nv["threshold"]
            if isinstance(th, bool) or not isinstance(th, (int, float)) or not math.isfinite(float(th)):
                raise ModelError(f"{w}: threshold")
            lo = _index(nv["left"], len(tv["nodes"]) - 1, f"{w}: left child")
            hi = _index(nv["right"], len(tv["nodes"]) - 1, f"{w}: right child")
            nodes.append(("split", f, float(th), lo, hi))
        seen, stack = set(), [0]
        while stack:  # a tree: no node reached twice
            i = stack.pop()
            if i in seen:
                raise ModelError(f"tree {t}: node {i} reached twice")
            seen.add(i)
            if nodes[i][0] == "split":
                stack += [nodes[i][3], nodes[i][4]]
        out.append(nodes)
    return {"classes": [ALGOS[c] for c in cls], "base": base, "trees": out}


def predict(model: dict, n: float, k: float, H: float):
    """Returns (algo4, scores in class order)."""
    x = (float(n), float(k), float(H))
    scores = list(model["base"])
    for nodes in model["trees"]:
        i = 0
        while nodes[i][0] == "split":
            _, f, th, lo, hi = nodes[i]
            i = lo if x[f] < th else hi
        for c in range(4):
            scores[c] += nodes[i][1][c]
    best = 0
    for c in range(1, 4):
        if scores[c] > scores[best]:
            best = c
    return model["classes"][best], scores
