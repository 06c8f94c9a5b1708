#!/usr/bin/env python
"""Text summary of an .ncu-rep (one block per profiled launch): duration,
DRAM bytes, occupancy, IPC, instruction count, registers, grid and the top
warp-stall reasons -- the lines committed under profiles/.
usage: python tools/ncu_summary.py gpurun_out/x.ncu-rep [...]"""
import csv
import subprocess
import sys

KEYS = [("duration us", "gpu__time_duration.sum"), ("dram read MB", "dram__bytes_read.sum"),
        ("dram write MB", "dram__bytes_write.sum"), ("dram % of peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        ("L2 hit %", "lts__t_sector_hit_rate.pct"),
        ("achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
        ("IPC", "sm__inst_executed.avg.per_cycle_elapsed"), ("warp instructions", "smsp__inst_executed.sum"),
        ("registers", "launch__registers_per_thread"), ("grid", "launch__grid_size"), ("block", "launch__block_size")]


def main():
    for path in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        if len(rows) < 3:
            print(f"# {path}: no launches")
            continue
        h, units = rows[0], rows[1]
        print(f"# {path}")
        for row in rows[2:]:
            print("kernel:", row[h.index("Kernel Name")])
            for label, k in KEYS:
                if k in h:
                    print(f"  {label:<22} {row[h.index(k)]} {units[h.index(k)] if 'bytes' in k else ''}".rstrip())
            st = {}
            for i, k in enumerate(h):
                if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                    try:
                        st[k.split("stalled_")[1].split("_per")[0]] = float(row[i])
                    except ValueError:
                        pass
            tot = sum(st.values()) or 1.0
            top = sorted(st.items(), key=lambda x: -x[1])[:6]
            print("  stalls:", ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))


if __name__ == "__main__":
    main()
