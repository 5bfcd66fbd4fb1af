timeout 900 python -m pytest tests/test_gpu_strips.py -q -p no:cacheprovider > gpurun_out/r2_dbg2.log 2>&1; echo rc=$? >> gpurun_out/r2_dbg2.log
