timeout 300 python -m pytest tests/test_gpu_cct_per_profile.py -m gpu -x -q > gpurun_out/t17.log 2>&1; echo rc=$? >> gpurun_out/t17.log
timeout 600 python tools/bench_next.py f1 > gpurun_out/next17.jsonl 2>&1
bash tools/ab_libs.sh C5 r2s3 nc24r4 look2 pred1 > gpurun_out/ab17.log 2>&1
tail -2 gpurun_out/t17.log; grep call_weights gpurun_out/next17.jsonl; grep -v Warn gpurun_out/ab17.log
