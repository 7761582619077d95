"""Summarise an ncu --set full capture of one component of the solve (the kernels of one
delayed-CGS2 step, or of one V-cycle) into profiles/r01_ncu_<name>.json, read by bench.py for
roofline.traffic.
  ncu -i <rep> --page raw --csv > raw.csv; python tools/ncu_dcgs_summary.py raw.csv <j> [name]"""
import csv
import json
import os
import sys

rows = list(csv.reader(open(sys.argv[1])))
j = int(sys.argv[2])
name = sys.argv[3] if len(sys.argv) > 3 else f"dcgs_j{j}"
hdr, units = rows[0], rows[1]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
out, total = [], 0.0
for r in rows[2:]:
    d = {k: r[hdr.index(k)] + (" " + units[hdr.index(k)] if units[hdr.index(k)] else "") for k in keys if k in hdr}
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(k)
        total += float(r[i].replace(",", "")) * scale.get(units[i], 1)
    out.append(d)
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"r01_ncu_{name}.json")
json.dump({"source": "ncu --set full --clock-control none, tools/profile_solve.py --workload c1_k400 --graph 0, "
                     f"first inner solve ({name})", "j": j, "dram_bytes_per_step": total, "kernels": out},
          open(path, "w"), indent=1)
print(path, total)
