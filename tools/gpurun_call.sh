timeout 600 python -m pytest tests/test_gpu_cct_async.py -m gpu -x -q > gpurun_out/t7.log 2>&1; echo rc=$? >> gpurun_out/t7.log
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "attr or exact or full or plan or ring" > gpurun_out/t7b.log 2>&1; echo rc=$? >> gpurun_out/t7b.log
for c in C3 C5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/b7_$c.log 2>&1
  timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --sync-cct > gpurun_out/b7s_$c.log 2>&1
done
timeout 300 python tools/attr_quick.py C5 --reps 9 > gpurun_out/aq7.log 2>&1
cp paper_2109_06931_b200/libgpa.so /tmp/libgpa_default.so
cp tools/alt/libgpa_pred0.so paper_2109_06931_b200/libgpa.so
echo "== pred0" >> gpurun_out/aq7.log; timeout 300 python tools/attr_quick.py C5 --reps 9 >> gpurun_out/aq7.log 2>&1
cp /tmp/libgpa_default.so paper_2109_06931_b200/libgpa.so
echo "== pred1 again" >> gpurun_out/aq7.log; timeout 300 python tools/attr_quick.py C5 --reps 9 >> gpurun_out/aq7.log 2>&1
tail -2 gpurun_out/t7.log; tail -2 gpurun_out/t7b.log; cat gpurun_out/aq7.log
for f in gpurun_out/b7*.log; do echo $f; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phases_ms'], d['config']['cct_contexts'])"; done
