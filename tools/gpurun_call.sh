cp paper_2109_06931_b200/libgpa.so /tmp/d.so
for rep in 1 2; do for v in default m1024; do
  if [ "$v" = default ]; then cp /tmp/d.so paper_2109_06931_b200/libgpa.so; else cp tools/alt/libgpa_$v.so paper_2109_06931_b200/libgpa.so; fi
  echo "== $v"; timeout 200 python tools/bench_next.py f4
done; done
cp /tmp/d.so paper_2109_06931_b200/libgpa.so
