"""DRAM traffic per launch of the hot kernels from ncu --set full captures (one launch each,
host-loop solve, cold caches): writes profiles/r02_ncu_traffic.json, which bench.py reads for the
roofline's `traffic` field.

  python tools/ncu_traffic.py WORKLOAD COLUMN N1 rep1.ncu-rep [rep2.ncu-rep ...]

Keys: "<workload>:<kernel>" -> {dram_bytes, dram_read, dram_write, us, column, bytes_per_column,
src}.  bytes_per_column: the basis stream of the Gram-Schmidt passes grows by 16 n1 bytes per
column, so bench.py scales the captured traffic to its own mean column.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}


def rows(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = {}
        for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                  "launch__grid_size"):
            i = hdr.index(k)
            d[k] = row[i]
            if k != "Kernel Name":
                d[k] = float(row[i].replace(",", "")) * UNIT.get(units[i], 1.0)
        yield d


def main():
    workload, column, n1 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
    try:
        with open(OUT) as fh:
            out = json.load(fh)
    except (OSError, ValueError):
        out = {}
    for rep in sys.argv[4:]:
        if "=" in rep:   # LABEL=rep.ncu-rep: every launch of the capture summed under one key (a V-cycle)
            label, rep = rep.split("=", 1)
            ds = list(rows(rep))
            key = f"{workload}:{label}"
            out[key] = {"dram_bytes": sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in ds),
                        "dram_read": sum(d["dram__bytes_read.sum"] for d in ds),
                        "dram_write": sum(d["dram__bytes_write.sum"] for d in ds),
                        "us": sum(d["gpu__time_duration.sum"] for d in ds), "launches": len(ds), "column": None,
                        "bytes_per_column": 0.0,
                        "src": os.path.basename(rep) + f" ({len(ds)} launches summed; ncu --set full, cold caches)"}
            print(key, json.dumps(out[key]))
            continue
        for d in rows(rep):
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("helm::", "").replace(" ", "")
            base = name.split("<")[0]
            per_col = 16.0 * n1 if base in ("k_dcgs_update", "k_dcgs_dots", "k_bgs_dots_smem", "k_bgs_update") else 0.0
            key = f"{workload}:{name}"
            out[key] = {"dram_bytes": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
                        "dram_read": d["dram__bytes_read.sum"], "dram_write": d["dram__bytes_write.sum"],
                        "us": d["gpu__time_duration.sum"], "column": column if per_col else None,
                        "bytes_per_column": per_col, "src": os.path.basename(rep) + " (ncu --set full, cold caches)"}
            print(key, json.dumps(out[key]))
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
