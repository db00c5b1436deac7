timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cct_async.py tests/test_gpu_cct_per_profile.py -m gpu -x -q -k "cct or async" > gpurun_out/t11.log 2>&1; echo rc=$? >> gpurun_out/t11.log
for c in C3 C5; do timeout 200 python tools/prof_cct.py $c 7 >> gpurun_out/cct11.log 2>&1; done
tail -3 gpurun_out/t11.log; grep "rep [456]" gpurun_out/cct11.log
