"""Markdown summary of an exported ncu capture (the details and raw pages as CSV, written by
tools/final_evidence.sh): python tools/evidence_summary.py gpurun_out/ev_det_X.csv gpurun_out/ev_raw_X.csv
[title] > profiles/r02_X.md"""
import csv
import io
import sys

KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "Executed Ipc Active", "Achieved Active Warps Per SM",
        "Registers Per Thread", "L1/TEX Hit Rate", "L2 Hit Rate", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "No Eligible", "Dynamic Shared Memory Per Block",
        "Shared Memory Configuration Size", "Grid Size", "Block Size", "SM Frequency", "DRAM Frequency")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum",
       "smsp__inst_executed_op_global_red.sum", "smsp__inst_executed_op_shared_atom.sum",
       "l1tex__data_pipe_lsu_wavefronts.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
       "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio")


def rows_of(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    return list(csv.reader(io.StringIO(txt[i:] if i >= 0 else txt)))


def main():
    det, raw = sys.argv[1], sys.argv[2]
    title = sys.argv[3] if len(sys.argv) > 3 else det
    print(f"# {title}\n")
    rows = rows_of(det)
    hdr = rows[0]
    kname = ""
    print("| section | metric | unit | value |\n|---|---|---|---|")
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        kname = d.get("Kernel Name", kname)
        if d.get("Metric Name") in KEEP:
            print(f"| {d.get('Section Name', '')} | {d['Metric Name']} | {d.get('Metric Unit', '')} | {d['Metric Value']} |")
    rr = rows_of(raw)
    if len(rr) > 2:
        print("\n| raw metric | unit | value |\n|---|---|---|")
        h, u, v = rr[0], rr[1], rr[2]
        for name in RAW:
            if name in h:
                j = h.index(name)
                print(f"| `{name}` | {u[j]} | {v[j]} |")
    print(f"\nKernel: `{kname[:160]}`")


if __name__ == "__main__":
    main()
