timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_launchpaths.py tests/test_gpu_determinism.py tests/test_gpu_fullsize.py -x -q > gpurun_out/n_test.log 2>&1; echo rc=$? >> gpurun_out/n_test.log
python bench.py --no-cpu-baseline > gpurun_out/n_c2.json 2> gpurun_out/n_c2.err
WRMG_SWEEP_BULK=0 python bench.py --no-cpu-baseline > gpurun_out/n_c2_nobulk.json 2> gpurun_out/n_c2_nobulk.err
