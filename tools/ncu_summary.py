#!/usr/bin/env python
"""Summarise ncu --set full captures (.ncu-rep) into a small CSV of the counters DESIGN.md
cites: per kernel launch, duration, DRAM bytes and throughput, tensor-pipe activity, issue
efficiency, occupancy, registers, instructions.  Runs on the CPU box (ncu -i).

    python tools/ncu_summary.py out.csv capture1.ncu-rep [capture2.ncu-rep ...]
"""
import csv
import subprocess
import sys

METRICS = [
    ("kernel", "Kernel Name"),
    ("time_us", "gpu__time_duration.sum"),
    ("dram_read", "dram__bytes_read.sum"),
    ("dram_write", "dram__bytes_write.sum"),
    ("dram_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
    ("issue_active_pct", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("registers", "launch__registers_per_thread"),
    ("smem_dyn_kb", "launch__shared_mem_per_block_dynamic"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("warp_instructions", "smsp__inst_executed.sum"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
]


def rows_of(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"capture": rep.split("/")[-1]}
        for key, name in METRICS:
            if name in hdr:
                i = hdr.index(name)
                v = r[i]
                u = units[i]
                if key.startswith("dram_") and key != "dram_pct" and v:  # normalise to MB
                    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                    v = "%.2f" % (float(v.replace(",", "")) * scale)
                    key = key + "_mb"
                elif key == "time_us" and v:
                    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
                    v = "%.2f" % (float(v.replace(",", "")) * scale)
                d[key] = v
        yield d


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    allrows = [d for rep in reps for d in rows_of(rep)]
    keys = ["capture"] + sorted({k for d in allrows for k in d if k != "capture"},
                                key=lambda k: [m[0] for m in METRICS].index(k.replace("_mb", "")))
    with open(out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=keys)
        w.writeheader()
        for d in allrows:
            w.writerow(d)
    print("wrote", out, len(allrows), "rows")


if __name__ == "__main__":
    main()
