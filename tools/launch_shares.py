"""Launch shares from an ncu `--metrics gpu__time_duration.sum --csv` log (dev helper).

usage: python tools/launch_shares.py launches.csv "title line" > profiles/rNN_launch_shares.md
"""
import csv
import re
import sys
from collections import defaultdict


def main(path, title):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr, rows = rows[0], rows[1:]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*", "", r[ki]).split("::")[-1].split("<")[0].strip()
        v = float(r[vi]) * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"# {title}\n")
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches: compare")
    print("shares, not absolutes).\n")
    print("| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"| {k} | {cnt[k]} | {tot[k]:.2f} | {100 * tot[k] / s:.2f}% |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "launch list")
