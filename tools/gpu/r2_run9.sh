timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b9.json 2> gpurun_out/r2_b9.err
