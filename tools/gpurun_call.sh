for i in 1 2 3; do
  GPA_DEBUG_POOL=1 GPA_BENCH_HOSTTIME=1 timeout 300 python bench.py --config C5 --no-cpu-baseline --no-e2e --async-cct > gpurun_out/ht_$i.log 2> gpurun_out/ht_$i.err
  grep -E "^step [0-2]:|pool_alloc" gpurun_out/ht_$i.err | head -12
  echo ---
done
