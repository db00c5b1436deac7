timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_bt_tile -c 1 -o gpurun_out/bt -f python tools/prof_blame.py 1 > /dev/null 2>&1
ncu -i gpurun_out/bt.ncu-rep --page source --csv > gpurun_out/bt_src.csv 2>&1
ncu -i gpurun_out/bt.ncu-rep --page details --csv > gpurun_out/bt_det.csv 2>&1
ncu -i gpurun_out/bt.ncu-rep --page raw --csv > gpurun_out/bt_raw.csv 2>&1
rm -f gpurun_out/bt.ncu-rep
python tools/src_top.py gpurun_out/bt_src.csv 30
