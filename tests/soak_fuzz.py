"""Soak run of tests/test_gpu_fuzz.py's generator over many more seeds (a test tool: like
the tests it calls the oracle; not collected by pytest).

    python tests/soak_fuzz.py FIRST LAST [SECONDS]     (env AHS_BL_MIN_KEYS etc. pass through)
    SOAK_LOG2=22,25 python tests/soak_fuzz.py ...      (n log-uniform in [2^22, 2^25] instead of [2, 2^22])

Prints one line per failing seed and a summary; exit code 1 when any seed failed.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))  # test_gpu_fuzz / test_gpu_parity

from test_gpu_fuzz import draw_case  # noqa: E402
from test_gpu_parity import check_pipeline  # noqa: E402

first, last = int(sys.argv[1]), int(sys.argv[2])
budget = float(sys.argv[3]) if len(sys.argv) > 3 else 1e9
t0 = time.time()
bad, done = [], 0
for seed in range(first, last):
    if time.time() - t0 > budget:
        break
    n_big = None
    if os.environ.get("SOAK_LOG2"):
        a, b = (float(v) for v in os.environ["SOAK_LOG2"].split(","))
        n_big = int(2 ** (a + (b - a) * ((seed * 2654435761) % 1000) / 1000.0))
    keys, vals, desc = draw_case(seed, n_big)
    try:
        check_pipeline(keys, vals)
    except Exception as e:  # noqa: BLE001
        bad.append(seed)
        print("FAIL", desc, str(e)[:300], flush=True)
    done += 1
print(f"seeds {first}..{first + done - 1}: {done - len(bad)} passed, {len(bad)} failed, {time.time() - t0:.0f} s "
      f"(AHS_BL_MIN_KEYS={os.environ.get('AHS_BL_MIN_KEYS', 'default')})")
sys.exit(1 if bad else 0)
