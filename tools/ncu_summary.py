"""Summarise an ncu report (details page + key raw metrics) as text."""
import csv, io, subprocess, sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
keep = ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
        "Issue Slots Busy", "Executed Ipc Active", "Achieved Occupancy", "Registers Per Thread", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler", "Executed Instructions",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in keep:
        print(f"{d.get('Kernel Name','')[:40]:40s} {d['Metric Name']:40s} {d['Metric Unit']:12s} {d['Metric Value']}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
for line in rr[2:]:
    d = dict(zip(rr[0], line))
    u = dict(zip(rr[0], rr[1]))
    for k in sorted(d):
        if (k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")) or k in (
                "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed_op_global_red.sum",
                "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed", "gpu__time_duration.sum",
                "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
                "smsp__inst_executed_op_shared_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
                "sm__warps_active.avg.pct_of_peak_sustained_active"):
            try:
                if float(d[k]) == 0:
                    continue
            except Exception:
                pass
            print(f"  {k:80s} {u.get(k,''):10s} {d[k]}")
