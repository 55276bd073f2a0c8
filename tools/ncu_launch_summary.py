"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list into a markdown table
(per-kernel launches, total/mean device time and share). Usage: python tools/ncu_launch_summary.py CSV [title]"""
import collections
import csv
import re
import sys


def summarise(path):
    rows = [r for r in csv.reader(open(path)) if len(r) >= 15 and r[12] == "gpu__time_duration.sum"]
    agg = collections.OrderedDict()
    for r in rows:
        name = re.sub(r"^void ", "", r[4])
        name = name.replace("maple::<unnamed>::", "").replace("(anonymous namespace)::", "")
        name = re.sub(r"\(.*$", "", name)
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[13], 1e-3)
        agg.setdefault(name, []).append(float(r[14].replace(",", "")) * scale)
    return agg


def table(agg, title=""):
    tot = sum(sum(v) for v in agg.values())
    out = [f"# {title}" if title else "# ncu launch list",
           "cold-cache, serialised per-launch device times (ncu --clock-control none): compare SHARES, not absolutes", "",
           "| kernel | launches | total us | mean us | share |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v) / len(v):.1f} | {sum(v) / tot:.3f} |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    print(table(summarise(sys.argv[1]), sys.argv[2] if len(sys.argv) > 2 else ""))
