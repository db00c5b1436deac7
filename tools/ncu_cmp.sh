M=gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_red.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__t_sector_hit_rate.pct,dram__bytes_read.sum,smsp__inst_executed.sum,smsp__inst_executed_op_shared_atom.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__issue_active.avg.pct_of_peak_sustained_active
# usage: VARIANTS="3 4" bash tools/ncu_cmp.sh   (GPA_ATTR_VARIANT values; C5 at 1e9 records)
for V in ${VARIANTS:-3 4}; do GPA_ATTR_VARIANT=$V timeout 300 ncu --metrics $M --clock-control none -k regex:k_attr_ -c 1 --csv --log-file gpurun_out/cmp_v$V.csv python tools/prof_attr.py C5 1000000000 1 > /dev/null 2>&1; done
python - <<'P'
import csv
import os
for v in [int(x) for x in os.environ.get('VARIANTS', '3 4').split()]:
    rows=list(csv.reader(open(f"gpurun_out/cmp_v{v}.csv")))
    s=next(i for i,r in enumerate(rows) if r and r[0]=="ID"); h=rows[s]
    for r in rows[s+1:]:
        print(v, r[h.index("Metric Name")], r[h.index("Metric Value")])
P
