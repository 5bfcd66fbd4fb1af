timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=10 > gpurun_out/r2_t13.log 2>&1; echo rc=$? >> gpurun_out/r2_t13.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b13.json 2> gpurun_out/r2_b13.err
