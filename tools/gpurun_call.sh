for i in 1 2 3 4 5 6; do
  timeout 300 python bench.py --config C5 --no-cpu-baseline --no-e2e --async-cct | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('async', round(d['ms_per_step'],3), round(d['roofline']['frac'],3), [round(x,1) for x in d['phases_ms']['attr_ms_per_step']])"
done
for c in C3 C4; do for m in "" "--async-cct"; do timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e $m | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $m', round(d['ms_per_step'],4))"; done; done
