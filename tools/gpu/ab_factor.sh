timeout 900 python -m pytest tests/test_gpu_ns.py -x -q > gpurun_out/b_nstest.log 2>&1; echo rc=$? >> gpurun_out/b_nstest.log
for rt in 1 4; do echo rt=$rt >> gpurun_out/b_time.log; WRMG_NS_FACTOR_RT=$rt timeout 300 python tools/time_ns_factor.py >> gpurun_out/b_time.log 2>&1; done
