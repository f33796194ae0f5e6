"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel: share of
the total time, average us per launch, launch count.
Usage: python tools/ncu_launch_summary.py launches.csv [command line for the header]"""
import csv
import sys
from collections import defaultdict


def main(path, cmd=""):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"')) if len(r) > 10]
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[1:]:
        us = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        tot[r[ik]] += us
        cnt[r[ik]] += 1
    all_us = sum(tot.values())
    print("ncu launch list (gpu__time_duration.sum, --clock-control none, -k regex:^k_, cold-cache serialised)")
    if cmd:
        print("command:", cmd)
    print("  share  us/launch  count  kernel")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{100 * tot[k] / all_us:6.2f}%  {tot[k] / cnt[k]:9.1f}  x {cnt[k]:4d}  {k[:120]}")
    print(f"total ms {all_us / 1e3:.3f} launches {sum(cnt.values())}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
