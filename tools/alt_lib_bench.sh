#!/bin/bash
# A/B the attribution kernel with alternative builds of libgpa.so (tools/alt/libgpa_*.so)
cp paper_2109_06931_b200/libgpa.so /tmp/libgpa_default.so
for lib in /tmp/libgpa_default.so tools/alt/libgpa_*.so; do
  cp $lib paper_2109_06931_b200/libgpa.so
  echo "== $lib"; timeout 300 python tools/attr_variants.py C5 4000000000 3 | cut -c1-120
  timeout 300 python tools/attr_variants.py C4 1000000000 3 | cut -c1-120
done
cp /tmp/libgpa_default.so paper_2109_06931_b200/libgpa.so
