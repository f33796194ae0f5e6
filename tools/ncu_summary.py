"""Summarise an ncu report (raw page) for the kernels in it: time, DRAM bytes, occupancy,
pipe utilisation and the top stall reasons.  Usage: python tools/ncu_summary.py rep.ncu-rep"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
]


def main(path, top=8):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]  # the raw page's second row holds each metric's unit
    res = []
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        print(name[:110])
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (r[i], units[i])
                print(f"   {k:70s} {r[i]:>16s} {units[i]}")
        st = [(hdr[i], r[i]) for i in range(len(hdr))
              if hdr[i].startswith("smsp__average_warps_issue_stalled_") and hdr[i].endswith("_per_issue_active.ratio")
              and r[i]]
        st = sorted(st, key=lambda x: -float(x[1].replace(",", "")))[:top]
        for s in st:
            nm = s[0].replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")
            print(f"      stall {nm:40s} {s[1]}")
        res.append((name, d))
    return res


if __name__ == "__main__":
    main(sys.argv[1])
