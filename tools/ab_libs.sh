#!/bin/bash
# A/B alternative builds of libgpa.so (tools/alt/libgpa_<name>.so) against the default build, interleaved
# twice: bash tools/ab_libs.sh "C5" name1 name2 ...   (prints attr_quick lines per build)
cfgs=$1; shift
cp paper_2109_06931_b200/libgpa.so /tmp/libgpa_default.so
for rep in 1 2; do
  for v in default "$@"; do
    if [ "$v" = default ]; then cp /tmp/libgpa_default.so paper_2109_06931_b200/libgpa.so; else cp tools/alt/libgpa_$v.so paper_2109_06931_b200/libgpa.so; fi
    echo "== $v (round $rep)"; timeout 300 python tools/attr_quick.py $cfgs --reps 7 2>&1 | cut -c1-200
  done
done
cp /tmp/libgpa_default.so paper_2109_06931_b200/libgpa.so
