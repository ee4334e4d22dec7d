"""Summarise an ncu report: time, throughputs, stalls, smem wavefronts."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
units = dict(zip(h, rows[1]))
for v in rows[2:]:
    d = dict(zip(h, v))
    print("kernel:", d.get("Kernel Name", "")[:90])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
            "smsp__inst_executed_op_shared_atom.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers"]
    for k in keys:
        print(f"  {k:75s} {d.get(k)} {units.get(k, '')}")
    st = {k: d[k] for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled") and "not_issued" not in k}
    tot = sum(float(x.replace(",", "") or 0) for x in st.values()) or 1
    for k, x in sorted(st.items(), key=lambda kv: -float(kv[1].replace(",", "") or 0))[:10]:
        print(f"  stall {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {float(x.replace(',', '')) / tot:6.1%}")
