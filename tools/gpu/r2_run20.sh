timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b20.json 2> gpurun_out/r2_b20.err
WRMG_MAC_MIN_NODES=10000 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b20m.json 2> gpurun_out/r2_b20m.err
WRMG_MAC_MIN_NODES=2000 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2_b20m2.json 2> gpurun_out/r2_b20m2.err
