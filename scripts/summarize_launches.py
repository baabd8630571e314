#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, total and average device time, and share of the
library's kernels.  Usage: summarize_launches.py launches.csv [out.md]"""
import collections
import csv
import sys


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    agg = collections.OrderedDict()
    for r in rows:
        name = r[4].split("(")[0].replace("void ", "")[:70]
        a = agg.setdefault(name, [0, 0.0, r[7], r[8]])
        a[0] += 1
        a[1] += float(r[-1])
    ours = sum(v[1] for k, v in agg.items() if k.startswith("sm::"))
    lines = [f"# ncu launch list summary: {path}", "",
             "cold-cache, serialised per-launch device times (gpu__time_duration.sum, --clock-control none);",
             "compare SHARES of the library's step, not absolutes", "",
             "| kernel | launches | total us | avg us | block | grid | share of library step |",
             "|---|---|---|---|---|---|---|"]
    for k, v in agg.items():
        share = f"{v[1] / ours:.3f}" if k.startswith("sm::") and ours else "-"
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e3:.1f} | {v[1] / v[0] / 1e3:.2f} | {v[2]} | {v[3]} | {share} |")
    text = "\n".join(lines) + "\n"
    if out:
        open(out, "w").write(text)
    print(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
