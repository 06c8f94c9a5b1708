"""One-screen summary of an ncu --set full report's raw CSV (duration, DRAM
bytes and throughput, occupancy, IPC, instructions, top stall reasons)."""
import csv
import sys

WANT = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
        ("dram__bytes_write.sum", "dram write"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
        ("sm__maximum_warps_per_active_cycle_pct", "theoretical occupancy %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
        ("sm__inst_executed.avg.per_cycle_active", "IPC"), ("smsp__inst_executed.sum", "warp instructions"),
        ("launch__registers_per_thread", "registers"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block")]


def main(path):
    r = list(csv.reader(open(path)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        name = row[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name}")
        for key, label in WANT:
            if key in hdr:
                i = hdr.index(key)
                print(f"  {label:26s} {row[i]} {units[i]}")
        st = [(h, row[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h.endswith("not_issued") and row[i]]
        tot = sum(float(v.replace(",", "")) for _, v in st) or 1
        top = sorted(st, key=lambda x: -float(x[1].replace(",", "")))[:6]
        print("  stalls: " + ", ".join(f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} "
                                       f"{float(v.replace(',', '')) / tot * 100:.0f}%" for h, v in top))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
