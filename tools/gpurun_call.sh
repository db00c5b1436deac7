timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin_gputest.log 2>&1; echo rc=$? >> gpurun_out/fin_gputest.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/fin_bench.log 2>&1
tail -1 gpurun_out/fin_bench.log > gpurun_out/fin_bench_C5.json
tail -2 gpurun_out/fin_gputest.log; tail -1 gpurun_out/fin_smoke.log; cat gpurun_out/fin_bench_C5.json
