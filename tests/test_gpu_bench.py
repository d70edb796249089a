"""The driver's bench contract for our own arm, on a B200: `python bench.py` (short run of the
default workload) prints exactly one JSON line with every key the contract asks for, values
consistent with each other (value = keys / step time, roofline frac = achieved / peak, e2e bytes
counted from the copied tensors, launches > 0)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                          "--configs", "cfg1", "--table-steps", "2", "--soak", "0.5", "--cpu-budget", "1"],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
              "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["higher_is_better"] is True
    n = 1 << 28  # cfg5 r=32, the default workload: 2^28 (key, value) pairs, above BASELINE's 2^26 gate
    assert d["config"]["workload"] == "cfg5_r32" and d["config"]["kv"] is True
    assert d["value"] == pytest.approx(n / (d["ms_per_step"] * 1e-3) / 1e9, rel=1e-3)
    hk = d["headline_keys"]  # second headline: keys-only GENERAL at 2^26
    assert hk["workload"] == "cfg4a" and hk["n"] == 1 << 26 and hk["value"] > 0
    assert hk["roofline"]["frac"] == pytest.approx(hk["roofline"]["achieved"] / hk["roofline"]["peak"], rel=1e-3)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert r["frac"] == pytest.approx(r["achieved"] / r["peak"], rel=1e-3)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 8 * n and e["d2h_bytes_per_step"] == 8 * n
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["value"] > 0 and c["cores"] == 1
    assert c["host"]["os_cpu_count"] >= 1 and "pinned" in c["sample"]
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
