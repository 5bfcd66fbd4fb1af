timeout 900 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_launchpaths.py -x -q -p no:cacheprovider -k "symmetric or coloured or dmma" > gpurun_out/r2_t11.log 2>&1; echo rc=$? >> gpurun_out/r2_t11.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b11.json 2> gpurun_out/r2_b11.err
