"""Per-kernel summary of an ncu launch list (--metrics gpu__time_duration.sum,
dram bytes; --csv --log-file): launches, total time, share, DRAM bytes per
launch.  Times under ncu are cold-cache and serialized: compare shares only."""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = None
    for i, r in enumerate(rows):
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = r
            rows = rows[i + 1:]
            break
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    idi = hdr.index("ID")
    per = collections.defaultdict(lambda: {"n": set(), "ns": 0.0, "bytes": 0.0})
    scale = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
             "Gbyte": 1e9}
    for r in rows:
        name = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1)
        d = per[name]
        d["n"].add(r[idi])
        if r[mi] == "gpu__time_duration.sum":
            d["ns"] += v
        else:
            d["bytes"] += v
    tot = sum(d["ns"] for d in per.values()) or 1
    print(f"{'kernel':50s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'MB/launch':>10s}")
    for name, d in sorted(per.items(), key=lambda x: -x[1]["ns"]):
        n = len(d["n"])
        print(f"{name[:50]:50s} {n:8d} {d['ns'] / 1e6:9.2f} {d['ns'] / tot * 100:5.1f}% {d['bytes'] / max(n, 1) / 1e6:10.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
