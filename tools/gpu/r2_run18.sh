python scratch/dbg_cheb_strip.py > gpurun_out/r2_dbg.log 2>&1
timeout 900 python -m pytest tests/test_gpu_strips.py -x -q -p no:cacheprovider > gpurun_out/r2_t18.log 2>&1; echo rc=$? >> gpurun_out/r2_t18.log
