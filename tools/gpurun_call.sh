timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cctp_ncu.csv python tools/prof_cctp.py 100000000 2 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/cctp_ncu.csv 0.5
