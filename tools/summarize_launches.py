"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list by kernel."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}


def main(path, title=""):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        name = r[ki].split("(")[0].replace("void ", "")
        if name.startswith("at::"):
            name = "torch " + name.split("<")[0] + " (workload generation, untimed)"
        ms = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ms
    tot = sum(v[1] for v in agg.values())
    own = sum(v[1] for k, v in agg.items() if k.startswith("isa::"))
    out = [title, "(ncu launch list: cold-cache, serialised launches -> compare SHARES, not absolutes)", "",
           f"{'kernel':70s} {'launches':>8s} {'ms':>10s} {'share':>7s} {'of isa':>7s}"]
    for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
        share_own = f"{ms / own * 100:6.1f}%" if k.startswith("isa::") and own else ""
        out.append(f"{k:70s} {n:8d} {ms:10.3f} {ms / tot * 100:6.1f}% {share_own:>7s}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
