"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel and stream:
launches, total / average microseconds and share of the listed GPU time.

    python tools/launch_summary.py gpurun_out/launches.csv "source command" > profiles/launches_....json
"""
import csv
import io
import json
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = csv.DictReader(io.StringIO("".join(lines)))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", ""))
        key = (r["Kernel Name"].split("(")[0].replace("void ", ""), r["Stream"])
        agg[key][0] += 1
        agg[key][1] += ns / 1e3
    total = sum(v[1] for v in agg.values())
    ks = sorted(agg.items(), key=lambda kv: -kv[1][1])
    out = {"source": sys.argv[2] if len(sys.argv) > 2 else path, "total_us": round(total, 1),
           "kernels": [{"kernel": k, "stream": s, "launches": n, "total_us": round(t, 1),
                        "avg_us": round(t / n, 2), "share": round(t / total, 4)} for (k, s), (n, t) in ks]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
