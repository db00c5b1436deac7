#!/bin/bash
# A/B alternative builds of libgpa.so (tools/alt/libgpa_*.so) for one attribution variant:
#   V=7 CFGS="C5:4000000000 C4:1000000000" bash tools/alt_sweep.sh
cp paper_2109_06931_b200/libgpa.so /tmp/libgpa_default.so
for lib in tools/alt/libgpa_*.so; do
  cp $lib paper_2109_06931_b200/libgpa.so
  for c in ${CFGS:-C5:4000000000 C4:1000000000}; do
    echo "== $(basename $lib) ${c%%:*}: $(timeout 300 python tools/attr_variants.py ${c%%:*} ${c##*:} ${V:-7} | cut -c1-110)"
  done
done
cp /tmp/libgpa_default.so paper_2109_06931_b200/libgpa.so
