"""Key counters of every kernel in an ncu report (--page raw): duration, DRAM bytes, issue activity and
the per-issue stall breakdown. Run here on the .ncu-rep brought back from the GPU box:

    python tools/ncu_summary.py gpurun_out/x.ncu-rep > profiles/ncu_....json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
STALL = "smsp__average_warps_issue_stalled_"


def main():
    raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = {"kernel": v[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                d[k] = f"{v[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        stalls = {h[len(STALL):].replace("_per_issue_active.ratio", ""): float(v[i])
                  for i, h in enumerate(hdr) if h.startswith(STALL) and h.endswith("_per_issue_active.ratio")
                  and v[i] not in ("", "n/a")}
        d["stalls_per_issue"] = dict(sorted(((k, round(x, 3)) for k, x in stalls.items() if x >= 0.01),
                                            key=lambda kv: -kv[1]))
        out.append(d)
    print(json.dumps({"source": sys.argv[1], "kernels": out}, indent=1))


if __name__ == "__main__":
    main()
