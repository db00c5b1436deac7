#!/bin/bash
# Round-end evidence on one GPU box (run from the repo root): bench line, launch list of the bench
# command, ncu --set full of the attribution kernels at their bench / config sizes, the DRAM-traffic
# capture bench.py reads, and the per-config table.  Outputs in gpurun_out/ (copied to profiles/).
set -x
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/ev_bench.log 2>&1
tail -1 gpurun_out/ev_bench.log > gpurun_out/ev_bench_C5.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ev_launches_C5.csv \
  python bench.py --steps 5 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1
for spec in "code32 C5 4000000000" "probe C4 1000000000" "direct C2 10000000"; do
  set -- $spec
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attr_$1 -c 1 -o gpurun_out/ev_$1_$2 -f \
    python tools/prof_attr.py $2 $3 1 > gpurun_out/ev_ncu_$1.log 2>&1
  ncu -i gpurun_out/ev_$1_$2.ncu-rep --page raw --csv > gpurun_out/ev_raw_$1_$2.csv 2>&1
  ncu -i gpurun_out/ev_$1_$2.ncu-rep --page details --csv > gpurun_out/ev_det_$1_$2.csv 2>&1
  [ "$1" = code32 ] && ncu -i gpurun_out/ev_$1_$2.ncu-rep --page source --csv > gpurun_out/ev_src_$1_$2.csv 2>&1
  rm -f gpurun_out/ev_$1_$2.ncu-rep
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attr_prof -c 1 -o gpurun_out/ev_prof_C4 -f \
  python tools/f1_quick.py > gpurun_out/ev_ncu_prof.log 2>&1
ncu -i gpurun_out/ev_prof_C4.ncu-rep --page raw --csv > gpurun_out/ev_raw_prof_C4.csv 2>&1
ncu -i gpurun_out/ev_prof_C4.ncu-rep --page details --csv > gpurun_out/ev_det_prof_C4.csv 2>&1
rm -f gpurun_out/ev_prof_C4.ncu-rep
timeout 900 python tools/capture_traffic.py C5 > gpurun_out/ev_traffic.log 2>&1
timeout 1500 python tools/bench_configs.py > gpurun_out/ev_configs.md 2>&1
timeout 900 python tools/bench_next.py > gpurun_out/ev_next.jsonl 2>&1
ls -la gpurun_out/ev_*
