"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a
per-kernel table: launches, total ms, share of the listed device time, avg us.

python scripts/launch_list_summary.py gpurun_out/launches.csv profiles/r01/launch_list_summary_c.md "<command>"
"""
import csv
import sys
from collections import defaultdict


def main(path, out, cmd):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "ms" else v
        name = r["Kernel Name"].split("(")[0]
        rows.append((name, us))
    agg = defaultdict(lambda: [0, 0.0])
    for name, us in rows:
        agg[name][0] += 1
        agg[name][1] += us
    total = sum(v[1] for v in agg.values())
    lines = ["# ncu launch list summary", "",
             f"Command: `{cmd}`", "",
             "Times are cold-cache and serialised (ncu): compare shares, not absolutes.", "",
             f"Total launches: {len(rows)}; listed device time {total / 1e3:.1f} ms", "",
             "| kernel | launches | total ms | share | avg us |", "|---|---|---|---|---|"]
    for name, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:20]:
        lines.append(f"| `{name}` | {cnt} | {us / 1e3:.2f} | {100 * us / total:.1f}% | {us / cnt:.1f} |")
    with open(out, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3])
