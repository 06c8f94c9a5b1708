"""Summarise an `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,dram__bytes_write.sum] --csv`
launch list by kernel: launches, device ms, share, DRAM bytes and GB/s (when captured)."""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main(path, title=""):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]
    ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
    per, names = collections.defaultdict(dict), {}
    for r in rows[hi + 1:]:
        per[r[0]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        name = r[ki].split("(")[0].replace("void ", "")
        names[r[0]] = ("torch " + name.split("<")[0] + " (workload generation, untimed)") if name.startswith("at::") else name
    agg = collections.OrderedDict()
    for i, m in per.items():
        a = agg.setdefault(names[i], [0, 0.0, 0.0])
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    own = sum(v[1] for k, v in agg.items() if k.startswith("isa::"))
    out = [title, "(ncu launch list: cold-cache, serialised launches -> compare SHARES, not absolutes)", "",
           f"{'kernel':58s} {'launches':>8s} {'ms':>9s} {'share':>6s} {'of isa':>7s} {'DRAM GB':>8s} {'GB/s':>6s}"]
    for k, (n, ms, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        so = f"{ms / own * 100:6.1f}%" if k.startswith("isa::") and own else ""
        bw = f"{b / 1e9 / (ms / 1e3):6.0f}" if b and ms else ""
        out.append(f"{k[:58]:58s} {n:8d} {ms:9.3f} {ms / tot * 100:5.1f}% {so:>7s} {b / 1e9:8.2f} {bw:>6s}")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
