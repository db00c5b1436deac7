timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "profiles_inst" > gpurun_out/t18.log 2>&1; echo rc=$? >> gpurun_out/t18.log
timeout 600 python tools/bench_next.py f1 > gpurun_out/next18.jsonl 2>&1
tail -3 gpurun_out/t18.log; grep -E "Error|assert" gpurun_out/t18.log | head -5; grep "inst" gpurun_out/next18.jsonl
