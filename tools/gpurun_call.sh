for i in 1 2 3; do
  timeout 300 python bench.py --config C5 --no-cpu-baseline --no-e2e | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('serial', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), [round(x,1) for x in d['phases_ms']['attr_ms_per_step']])"
done
timeout 300 python bench.py --config C5 --no-cpu-baseline --no-e2e --pipeline | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pipe', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), [round(x,1) for x in d['phases_ms']['attr_ms_per_step']])"
timeout 300 python bench.py --config C3 --no-cpu-baseline --no-e2e | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 serial', round(d['ms_per_step'],3))"
