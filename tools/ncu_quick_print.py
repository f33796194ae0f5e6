import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')) if len(r) > 10]
h = rows[0]; ix = {k: i for i, k in enumerate(h)}
by = defaultdict(dict)
for r in rows[1:]:
    key = (r[ix["ID"]], r[ix["Kernel Name"]][:70])
    by[key][r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
short = {"gpu__time_duration.sum": "t", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wf",
         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum": "confl_ld",
         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum": "confl_st", "smsp__inst_executed.sum": "inst",
         "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%", "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue%",
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem%",
         "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma%", "dram__bytes_read.sum": "dram_r",
         "dram__bytes_write.sum": "dram_w", "launch__registers_per_thread": "regs", "launch__occupancy_limit_shared_mem": "blk/sm(smem)",
         "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed": "lsu%"}
for (i, name), m in by.items():
    print(i, name)
    print("   " + "  ".join(f"{short.get(k, k)}={v[0]}{v[1] if v[1] not in ('', 'inst', '%') else ''}" for k, v in m.items()))
