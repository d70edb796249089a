"""Per-source-line instruction / shared-wavefront / stall breakdown of an ncu report.

    python tools/ncu_lines.py report.ncu-rep KEYS [min_share]
Numbers are per 32 keys (KEYS = keys processed by the profiled launch).
"""
import csv
import subprocess
import sys


def main():
    rep, keys = sys.argv[1], float(sys.argv[2])
    thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.2
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    per = keys / 32.0
    fname, hdr, res = None, None, []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 10 or r[2] != "-":
            continue
        g = lambda name: float(r[hdr.index(name)] or 0)
        res.append((fname, r[0], r[1].strip()[:80], g("Instructions Executed") / per,
                    g("L1 Wavefronts Shared") / per, g("Warp Stall Sampling (All Samples)")))
    ts = sum(x[5] for x in res) or 1.0
    for x in res:
        if x[3] > thr or x[4] > thr or x[5] / ts > 0.01:
            print(f"{x[3]:6.2f} inst {x[4]:6.2f} wf {100 * x[5] / ts:5.1f}% | {x[0]}:{x[1]} {x[2]}")
    print(f"total (lines, inlined helpers double-count): inst {sum(x[3] for x in res):.1f} "
          f"wf {sum(x[4] for x in res):.1f} per 32 keys")


if __name__ == "__main__":
    main()
