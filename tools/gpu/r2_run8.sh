timeout 900 python -m pytest tests/test_gpu_launchpaths.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "sweep or smooth or vcycle or fgmres or C2" > gpurun_out/r2_t8.log 2>&1; echo rc=$? >> gpurun_out/r2_t8.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b8.json 2> gpurun_out/r2_b8.err
WRMG_SWEEP_TILES=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b8_notile.json 2> gpurun_out/r2_b8_notile.err
