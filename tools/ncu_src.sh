# usage: V=7 CFG=C5 N=1000000000 bash tools/ncu_src.sh  -> gpurun_out/src_v$V.csv (per-instruction stall samples of K_attr)
V=${V:-7}; CFG=${CFG:-C5}; N=${N:-1000000000}; K=${K:-regex:k_attr_}
GPA_ATTR_VARIANT=$V timeout 600 ncu --set full --import-source on --clock-control none -k $K -c 1 -o gpurun_out/src_v$V -f python tools/prof_attr.py $CFG $N 1 > /dev/null 2>&1
ncu -i gpurun_out/src_v$V.ncu-rep --page source --csv > gpurun_out/src_v$V.csv 2>&1
ncu -i gpurun_out/src_v$V.ncu-rep --page raw --csv > gpurun_out/raw_v$V.csv 2>&1
