timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f1i_launch.csv python tools/prof_f1inst.py > /dev/null 2>&1
python tools/launch_table.py gpurun_out/f1i_launch.csv 1.0
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attr_prof_code -c 1 -o gpurun_out/f1i -f python tools/prof_f1inst.py > /dev/null 2>&1
ncu -i gpurun_out/f1i.ncu-rep --page source --csv > gpurun_out/f1i_src.csv 2>&1
ncu -i gpurun_out/f1i.ncu-rep --page details --csv > gpurun_out/f1i_det.csv 2>&1
ncu -i gpurun_out/f1i.ncu-rep --page raw --csv > gpurun_out/f1i_raw.csv 2>&1
rm -f gpurun_out/f1i.ncu-rep
python tools/src_top.py gpurun_out/f1i_src.csv 20
python tools/evidence_summary.py gpurun_out/f1i_det.csv gpurun_out/f1i_raw.csv "f1 inst" | head -40
