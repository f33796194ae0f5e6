"""Extract per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the kernels
in an ncu --set full report and write profiles/ncu_traffic.json for bench.py's roofline.traffic.
Usage: python tools/ncu_traffic.py <report.ncu-rep> <class name> <kernel regex> <nx> <ny> <nz>"""
import csv
import io
import json
import os
import re
import subprocess
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(rep, cls, regex, nx, ny, nz):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    it = hdr.index("gpu__time_duration.sum")
    vals = []
    for r in rows[2:]:
        if not re.search(regex, r[hdr.index("Kernel Name")]):
            continue
        b = float(r[ir].replace(",", "")) * UNITS.get(units[ir], 1) + float(r[iw].replace(",", "")) * UNITS.get(units[iw], 1)
        vals.append((b, float(r[it].replace(",", ""))))
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    data = json.load(open(path)) if os.path.exists(path) else {"classes": {}}
    data["classes"][cls] = {"grid": [int(nx), int(ny), int(nz)], "bytes_per_launch": sum(v[0] for v in vals) / len(vals),
                            "launches_sampled": len(vals), "kernel_regex": regex, "report": os.path.basename(rep)}
    json.dump(data, open(path, "w"), indent=1)
    print(data["classes"][cls])


if __name__ == "__main__":
    main(*sys.argv[1:])
