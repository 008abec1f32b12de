#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python tools/launch_summary.py gpurun_out/launches.csv > profiles/launches_rNN.txt

ncu times are cold-cache and serialised: compare each kernel's SHARE of the
step with the in-bench CUDA-event numbers, not the absolute durations.
"""
import collections
import csv
import re
import sys


def main(path):
    agg = collections.OrderedDict()
    for r in csv.reader(open(path)):
        if not r or not r[0].isdigit() or r[12] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\((kpl::SGeo|kpl::CGeo|int, T2).*", "", r[4]).replace("void ", "")[:100]
        a = agg.setdefault(name, [0, 0.0, r[7], r[8]])
        a[0] += 1
        a[1] += float(r[14])
    tot = sum(v[1] for v in agg.values())
    print(f"# {path}: {sum(v[0] for v in agg.values())} launches, {tot/1e6:.3f} ms total")
    print(f"# {'count':>5} {'total_ms':>10} {'share':>7} {'avg_us':>10}  block grid  kernel")
    for k, (c, t, blk, grd) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{c:7d} {t/1e6:10.3f} {100*t/tot:6.2f}% {t/c/1e3:10.1f}  {blk} {grd}  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
