"""SURVEY §5 Config/flags: environment overrides of the Table II thresholds (SPEC S:534 flag names),
host logic on the CPU: ahs_thresholds_from_env parses them, validates them like ahs_select, and the
FSM decision follows them (missing #5)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, paper_2506_20677_b200 as ahs
try:
    th = ahs.ahs_thresholds_from_env()
    f = ahs.Features(); f.n, f.k, f.nbins, f.entropy, f.dtype = 5000, 1500, 1500, 3.0, 0
    s, r = ahs.ahs_select(f, th)
    print(json.dumps({"ok": True, "n_ins": th.n_insertion, "k_cnt": th.k_counting, "k_rad": th.k_radix,
                      "coeff": th.entropy_coeff, "norm": th.entropy_norm, "strategy": ahs.STRATEGY_NAMES[s]}))
except ahs.AhsError as e:
    print(json.dumps({"ok": False}))
"""


def probe(**env):
    import json
    e = {k: v for k, v in os.environ.items() if not k.startswith("AHS_")}
    e.update(env)
    out = subprocess.run([sys.executable, "-c", PROBE], env=e, cwd=ROOT, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_defaults_without_environment():
    d = probe()
    assert d["ok"] and (d["n_ins"], d["k_cnt"], d["k_rad"], d["coeff"], d["norm"]) == (20, 1024, 1000000, 0.7, 0)
    assert d["strategy"] == "GENERAL"  # k = 1500 > 1024, not > 10^6


def test_overrides_change_the_decision():
    d = probe(AHS_K_COUNTING="2000")
    assert d["ok"] and d["k_cnt"] == 2000 and d["strategy"] == "COUNTING"  # k = 1500 <= 2000
    d = probe(AHS_K_COUNTING="500", AHS_K_RADIX="1000", AHS_ENTROPY_COEFF="0.9", AHS_ENTROPY_NORM="range",
              AHS_N_INSERTION="16")
    assert d["ok"] and (d["k_cnt"], d["k_rad"], d["coeff"], d["norm"], d["n_ins"]) == (500, 1000, 0.9, 1, 16)
    assert d["strategy"] == "RADIX"  # k > 1000 and H = 3 < 0.9 log2 1500


@pytest.mark.parametrize("env", [{"AHS_K_COUNTING": "12x"}, {"AHS_K_RADIX": "-5"}, {"AHS_ENTROPY_NORM": "bins"},
                                 {"AHS_ENTROPY_COEFF": "1.5"}, {"AHS_K_COUNTING": "2000000"}])
def test_malformed_or_invalid_values_are_refused(env):
    assert probe(**env)["ok"] is False
