"""Summarise an `ncu --page raw --csv` export: time, DRAM bytes, issue, LSU,
shared-memory atomics, instructions, registers, top stall reasons."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "smsp__inst_executed_op_shared_atom.sum",
        "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_shared_st.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smsp__inst_executed_op_branch.sum",
        "smsp__inst_executed_op_global_red.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers",
        "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg"]
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
units = dict(zip(h, rows[1]))
for v in rows[2:]:
    d = dict(zip(h, v))
    print("kernel:", d.get("Kernel Name", "")[:100])
    for k in KEYS:
        if k in d:
            print(f"  {k:70s} {d[k]} {units.get(k, '')}")
    st = {k: d[k] for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled") and "not_issued" not in k}
    tot = sum(float(x.replace(",", "") or 0) for x in st.values()) or 1
    top = sorted(st.items(), key=lambda kv: -float(kv[1].replace(",", "") or 0))[:6]
    print("  stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} "
                                   f"{float(x.replace(',', '')) / tot:.0%}" for k, x in top))
