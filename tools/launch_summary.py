"""Summarise an ncu launch list (`--metrics gpu__time_duration.sum --csv`) per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv [header line ...]
"""
import collections
import csv
import sys


def summarise(path):
    hdr = None
    agg = collections.OrderedDict()
    for r in csv.reader(open(path)):
        if len(r) > 10 and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
            name = r[hdr.index("Kernel Name")]
            short = name.split("(")[0][:60] if not name.startswith("void at::") else "torch:" + name[10:40]
            scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(
                r[hdr.index("Metric Unit")], 1e-6)
            a = agg.setdefault(short, [0, 0.0])
            a[0] += 1
            a[1] += float(r[hdr.index("Metric Value")]) * scale
    return agg


if __name__ == "__main__":
    agg = summarise(sys.argv[1])
    for line in sys.argv[2:]:
        print("#", line)
    tot = sum(v[1] for v in agg.values())
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:60s} launches={n:4d} total={t:10.3f} ms share={100 * t / tot:6.2f}%")
