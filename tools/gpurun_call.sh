timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/t57.log 2>&1; echo rc=$? >> gpurun_out/t57.log
for i in 1 2 3; do
  timeout 300 python bench.py --config C5 --no-cpu-baseline --no-e2e | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('sync', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), [round(x,1) for x in d['phases_ms']['attr_ms_per_step']])"
  timeout 300 python bench.py --config C5 --no-cpu-baseline --no-e2e --async-cct | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('async', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), [round(x,1) for x in d['phases_ms']['attr_ms_per_step']])"
done
timeout 200 python tools/host_overhead.py C2 10000000 200
timeout 200 python tools/attr_quick.py C2,C3 --reps 9
tail -2 gpurun_out/t57.log
