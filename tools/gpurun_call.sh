set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t4.log 2>&1; echo rc=$? >> gpurun_out/t4.log
timeout 300 python tools/attr_quick.py C2,C3,C4,C5 > gpurun_out/aq4.log 2>&1
TRACE=1 timeout 200 python tools/prof_cct.py C3 5 > gpurun_out/cct4.log 2>&1
timeout 200 python tools/prof_cct.py C5 5 >> gpurun_out/cct4.log 2>&1
timeout 300 python tools/bench_next.py f2 > gpurun_out/f2_4.log 2>&1
timeout 300 python bench.py > gpurun_out/bench4.log 2>&1
tail -3 gpurun_out/t4.log; cat gpurun_out/aq4.log; grep -v "Warn\|warn_once" gpurun_out/cct4.log; tail -1 gpurun_out/f2_4.log; tail -1 gpurun_out/bench4.log
