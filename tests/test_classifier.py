"""NEXT-4 strategy classifier (§III.H, Listing 5; SPEC.md classifier
module S:142-193).  Host code only: runs without a GPU.

Oracle pins (oracle/classifier.py against things other than itself): SPEC's worked examples
(a one-leaf model -> insertion with [1,0,0,0]; empty input and an out-of-range feature index
rejected; a foreign version rejected), score additivity when the fixture's trees are split,
and agreement of the FSM-consistent fixture with the paper's FSM (oracle.select, RANGE
normalisation) on SPEC's 512-point grid.  Product parity: libahs's C++ loader / predictor
against the oracle on the fixture, on random ensembles (scores bit-exact: same summation
order) and on a catalogue of malformed models; ahs_select_model's routing.
"""
import json
import os
import random
import sys

import pytest

import oracle
from oracle import classifier as oc

sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
import make_model_fixture as fixture  # noqa: E402

ahs = pytest.importorskip("paper_2506_20677_b200")

FIXTURE = os.path.join(os.path.dirname(__file__), "golden", "ahs_model_fixture.json")


def fixture_text():
    with open(FIXTURE) as fh:
        return fh.read()


def one_leaf(scores, classes=("insertion", "counting", "radix", "quick")):
    return json.dumps({"version": "ahs-model/1", "classes": list(classes), "feature_names": ["n", "k", "H"],
                       "base_scores": [0, 0, 0, 0], "trees": [{"nodes": [{"leaf": scores}]}]})


# ------------------------------------------------------------ oracle pins
def test_fixture_is_what_the_script_writes():
    assert json.loads(fixture_text()) == fixture.build()


def test_spec_constant_model():
    m = oc.load(one_leaf([1, 0, 0, 0]))
    assert oc.predict(m, 100, 10, 1.0) == (0, [1.0, 0.0, 0.0, 0.0])  # S:170 -> (Insertion, [1,0,0,0])


def test_spec_rejections():
    with pytest.raises(oc.ModelError):
        oc.load(b"")  # S:163 empty byte stream -> parse error
    bad = json.loads(one_leaf([1, 0, 0, 0]))
    bad["trees"][0]["nodes"] = [{"feature": 5, "threshold": 1.0, "left": 1, "right": 1}, {"leaf": [0, 0, 0, 0]}]
    with pytest.raises(oc.ModelError):
        oc.load(json.dumps(bad))  # S:164 feature index 5 -> validation error
    v = json.loads(one_leaf([1, 0, 0, 0]))
    v["version"] = "ahs-model/2"
    with pytest.raises(oc.VersionError):
        oc.load(json.dumps(v))


def _fsm(n, k, H):
    f = oracle.Features()
    f.n, f.k, f.entropy, f.nb = n, k, H, min(k, 65536)
    s, _ = oracle.select(f, norm=1)  # RANGE: H < 0.7 log2 k
    return s


def test_fixture_agrees_with_fsm_on_spec_grid():
    m = oc.load(fixture_text())
    g = fixture.grid()
    assert len(g) == 512
    for n, k, H in g:
        assert oc.predict(m, n, k, H)[0] == _fsm(n, k, H), (n, k, H)
    # the grid reaches every branch the FSM has at n >= 1000
    assert {_fsm(n, k, H) for n, k, H in g} == {oracle.COUNTING, oracle.RADIX, oracle.QUICK}


def test_score_additivity():
    full = json.loads(fixture_text())
    a, b = dict(full), dict(full)
    a["trees"], b["trees"] = full["trees"][:1], full["trees"][1:]
    ma, mb, mf = (oc.load(json.dumps(x)) for x in (a, b, full))
    base = full["base_scores"]
    for n, k, H in fixture.grid()[::7]:
        sa, sb, sf = oc.predict(ma, n, k, H)[1], oc.predict(mb, n, k, H)[1], oc.predict(mf, n, k, H)[1]
        for c in range(4):
            assert abs(sf[c] - (sa[c] + sb[c] - base[c])) <= 1e-12


def test_tie_goes_to_the_earlier_class():
    m = oc.load(one_leaf([0, 2, 2, 0], classes=("quick", "radix", "counting", "insertion")))
    assert oc.predict(m, 1, 1, 0)[0] == oc.ALGOS["radix"]


# --------------------------------------------------------- product parity
def random_model(rng: random.Random, ntrees: int):
    classes = ["insertion", "counting", "radix", "quick"]
    rng.shuffle(classes)
    trees = []
    for _ in range(ntrees):
        nodes = [None]

        def grow(i, depth):
            if depth == 0 or rng.random() < 0.25:
                nodes[i] = {"leaf": [rng.uniform(-1, 1) for _ in range(4)]}
                return
            f = rng.randrange(3)
            th = {0: 10 ** rng.uniform(0, 7), 1: 10 ** rng.uniform(0, 9), 2: rng.uniform(0, 30)}[f]
            lo, hi = len(nodes), len(nodes) + 1
            nodes.extend([None, None])
            nodes[i] = {"feature": f, "threshold": th, "left": lo, "right": hi}
            grow(lo, depth - 1)
            grow(hi, depth - 1)

        grow(0, rng.randrange(1, 7))
        trees.append({"nodes": nodes})
    return {"version": "ahs-model/1", "classes": classes, "feature_names": ["n", "k", "H"],
            "base_scores": [rng.uniform(-0.5, 0.5) for _ in range(4)], "trees": trees}


def test_product_matches_oracle_on_fixture_grid():
    txt = fixture_text()
    pm, om = ahs.Model(txt), oc.load(txt)
    for n, k, H in fixture.grid():
        assert pm.predict(n, k, H) == oc.predict(om, n, k, H)


def test_product_matches_oracle_on_random_ensembles():
    rng = random.Random(2506)
    for trial in range(60):
        spec = random_model(rng, rng.randrange(0, 12))
        txt = json.dumps(spec)
        pm, om = ahs.Model(txt), oc.load(txt)
        for _ in range(50):
            n, k, H = 10 ** rng.uniform(0, 8), 10 ** rng.uniform(0, 10), rng.uniform(0, 32)
            assert pm.predict(n, k, H) == oc.predict(om, n, k, H), trial


def _malformed():
    good = json.loads(one_leaf([1, 0, 0, 0]))
    split = {"feature": 0, "threshold": 5.0, "left": 1, "right": 2}
    cases = {
        "empty": "",
        "not_json": "{version: 1}",
        "trailing": one_leaf([1, 0, 0, 0]) + " x",
        "array_top": "[]",
        "unknown_top": dict(good, extra=1),
        "classes_3": dict(good, classes=["insertion", "counting", "radix"]),
        "classes_dup": dict(good, classes=["insertion", "counting", "radix", "radix"]),
        "classes_unknown": dict(good, classes=["insertion", "counting", "radix", "merge"]),
        "features_order": dict(good, feature_names=["k", "n", "H"]),
        "base_3": dict(good, base_scores=[0, 0, 0]),
        "base_str": dict(good, base_scores=[0, 0, "1", 0]),
        "no_trees": {k: v for k, v in good.items() if k != "trees"},
        "tree_no_nodes": dict(good, trees=[{}]),
        "tree_empty": dict(good, trees=[{"nodes": []}]),
        "tree_extra": dict(good, trees=[{"nodes": [{"leaf": [0, 0, 0, 0]}], "x": 1}]),
        "leaf_3": dict(good, trees=[{"nodes": [{"leaf": [0, 0, 0]}]}]),
        "leaf_extra": dict(good, trees=[{"nodes": [{"leaf": [0, 0, 0, 0], "feature": 0}]}]),
        "feature_5": dict(good, trees=[{"nodes": [dict(split, feature=5), {"leaf": [0] * 4}, {"leaf": [0] * 4}]}]),
        "feature_float": dict(good, trees=[{"nodes": [dict(split, feature=1.5), {"leaf": [0] * 4},
                                                      {"leaf": [0] * 4}]}]),
        "child_range": dict(good, trees=[{"nodes": [dict(split, right=3), {"leaf": [0] * 4}, {"leaf": [0] * 4}]}]),
        "child_negative": dict(good, trees=[{"nodes": [dict(split, left=-1), {"leaf": [0] * 4},
                                                       {"leaf": [0] * 4}]}]),
        "cycle": dict(good, trees=[{"nodes": [dict(split, left=0), {"leaf": [0] * 4}, {"leaf": [0] * 4}]}]),
        "shared_child": dict(good, trees=[{"nodes": [dict(split, right=1), {"leaf": [0] * 4}]}]),
        "split_missing_threshold": dict(good, trees=[{"nodes": [{"feature": 0, "left": 1, "right": 2},
                                                                {"leaf": [0] * 4}, {"leaf": [0] * 4}]}]),
        "duplicate_key": '{"version":"ahs-model/1","version":"ahs-model/1"}',
    }
    return {k: (v if isinstance(v, str) else json.dumps(v)) for k, v in cases.items()}


@pytest.mark.parametrize("case", list(_malformed()))
def test_both_reject_malformed(case):
    txt = _malformed()[case]
    with pytest.raises(oc.ModelError):
        oc.load(txt)
    with pytest.raises(ahs.AhsError) as e:
        ahs.Model(txt)
    assert e.value.status == ahs.AHS_EMODEL


def test_product_version_error():
    v = json.loads(one_leaf([1, 0, 0, 0]))
    v["version"] = "ahs-model/0"
    with pytest.raises(ahs.AhsError) as e:
        ahs.Model(json.dumps(v))
    assert e.value.status == ahs.AHS_EMODELVER


def test_select_model_routing():
    model = ahs.Model(fixture_text())
    f = ahs.Features()
    f.n, f.k, f.nbins, f.entropy, f.bits = 10 ** 6, 10 ** 7, 65536, 2.0, 24
    # classifier for n >= ml_min_n: k = 10^7, H = 2 < 0.7 log2 k -> radix
    s, r, src = ahs.ahs_select_model(f, model)
    assert (ahs.STRATEGY_NAMES[s], ahs.RULE_NAMES[r], src) == ("RADIX", "MODEL", 1)
    # below ml_min_n: the rules
    s, r, src = ahs.ahs_select_model(f, model, ml_min_n=10 ** 7)
    assert src == 0 and (s, r) == ahs.ahs_select(f)
    # no model: the rules
    assert ahs.ahs_select_model(f, None)[2] == 0
    # P:411 shortcuts precede the classifier
    f.k = 1
    s, r, src = ahs.ahs_select_model(f, model)
    assert ahs.RULE_NAMES[r] == "CONSTANT" and src == 0
    # (n=10^6, k=500, H=1.1) -> counting, (n=10^6, k=10^8, H=2) -> radix
    assert model.predict(10 ** 6, 500, 1.1)[0] == 1
    assert model.predict(10 ** 6, 10 ** 8, 2.0)[0] == 2
