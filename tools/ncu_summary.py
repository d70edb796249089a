"""Per-launch summary of an ncu --set full report (development tool):
duration, DRAM read/write bytes, L1TEX data-pipe utilisation, shared wavefronts and bank
conflicts, global-store sectors per request, issue activity.

    python tools/ncu_summary.py report.ncu-rep [--json]
"""
import csv
import json
import subprocess
import sys

M = {
    "us": "gpu__time_duration.sum",
    "dram_rd": "dram__bytes_read.sum",
    "dram_wr": "dram__bytes_write.sum",
    "lsu_pipe_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "smem_wf": "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smem_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "st_sectors": "l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum",
    "st_requests": "l1tex__t_requests_pipe_lsu_mem_global_op_st.sum",
    "issue_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "inst": "smsp__inst_executed.sum",
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")].split("<")[0].split("(")[0].replace("void ", "")}
        d["name"] = row[hdr.index("Kernel Name")][:120]
        for k, m in M.items():
            if m in hdr:
                v = float(row[hdr.index(m)] or 0)
                u = units[hdr.index(m)]
                v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                      "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
                d[k] = v
        res.append(d)
    return res


def main():
    rep = sys.argv[1]
    rs = rows(rep)
    if "--json" in sys.argv:
        print(json.dumps(rs, indent=1))
        return
    print(f"{'kernel':22s} {'us':>8s} {'DRAM rd MB':>10s} {'DRAM wr MB':>10s} {'LSU pipe%':>9s} "
          f"{'smem wf M':>9s} {'confl M':>8s} {'st sec/req':>10s} {'issue%':>7s}")
    for d in rs:
        spr = d["st_sectors"] / d["st_requests"] if d.get("st_requests") else 0.0
        print(f"{d['kernel']:22s} {d['us']:8.1f} {d['dram_rd'] / 1e6:10.1f} {d['dram_wr'] / 1e6:10.1f} "
              f"{d['lsu_pipe_pct']:9.1f} {d['smem_wf'] / 1e6:9.2f} {d['smem_conflicts'] / 1e6:8.2f} {spr:10.2f} "
              f"{d['issue_pct']:7.1f}")


if __name__ == "__main__":
    main()
