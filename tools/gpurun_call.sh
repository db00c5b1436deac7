timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ev_gputest.log 2>&1; echo rc=$? >> gpurun_out/ev_gputest.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ev_smoke.log 2>&1
bash tools/final_evidence.sh > gpurun_out/ev_script.log 2>&1
tail -2 gpurun_out/ev_gputest.log; tail -1 gpurun_out/ev_smoke.log; cat gpurun_out/ev_bench_C5.json; cat gpurun_out/ev_traffic.log | tail -1
